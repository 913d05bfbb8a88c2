mkdir -p gpurun_out
MBX_PDL=0 MBX_TC_STAMPS=1 timeout 120 python tools/probe_step.py --reps 2 > gpurun_out/stamps_nopdl.log 2>&1
MBX_ARRIVE_RELEASE=1 MBX_PDL=0 MBX_TC_STAMPS=1 timeout 120 python tools/probe_step.py --reps 2 > gpurun_out/stamps_rel.log 2>&1
bash tools/gpu_ab2.sh MBX_ARRIVE_RELEASE 1

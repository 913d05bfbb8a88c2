mkdir -p gpurun_out
MBX_PDL=0 MBX_TC_STAMPS=1 timeout 120 python tools/probe_step.py --reps 2 > gpurun_out/stamps_nopdl.log 2>&1
MBX_TC_STAMPS=1 timeout 120 python tools/probe_step.py --reps 2 > gpurun_out/stamps.log 2>&1

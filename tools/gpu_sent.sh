mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -2
bash tools/gpu_ab2.sh MBX_NO_SENTINEL 1
MBX_PDL=0 MBX_TC_STAMPS=1 timeout 120 python tools/probe_step.py --reps 2 > gpurun_out/stamps_nopdl.log 2>&1

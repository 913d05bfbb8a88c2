mkdir -p gpurun_out
MBX_TC_STAMPS=1 timeout 120 python tools/probe_step.py --model birnn --reps 2 > gpurun_out/birnn_stamps.log 2>&1

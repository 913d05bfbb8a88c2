set -x
mkdir -p gpurun_out
MBX_TC_STAMPS=1 timeout 300 python tools/probe_step.py --reps 2 > gpurun_out/stamps.log 2>&1
grep -A8 "^levels" gpurun_out/stamps.log | tail -8

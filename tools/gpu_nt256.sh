MBX_LEVELS_CY=1 timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -1
bash tools/gpu_ab2.sh MBX_LEVELS_CY 1
MBX_LEVELS_CY=1 MBX_PDL=0 MBX_TC_STAMPS=1 timeout 120 python tools/probe_step.py --reps 1 2>&1 | grep -A12 "cfg 0" | cut -c1-60

set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mbx_tc_levels --launch-skip 5 --launch-count 1 \
   -o gpurun_out/levels_full -f python tools/probe_step.py --reps 3 > gpurun_out/ncu_levels.log 2>&1
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x -k "bf16x3 or zoo or levels" > gpurun_out/tc_tests.log 2>&1
tail -3 gpurun_out/tc_tests.log

# Iteration run: tensor-core GPU tests, probe timings, stamp trace (profiling aid).
set -x
mkdir -p gpurun_out
MBX_TC_STAMPS=1 timeout 300 python tools/probe_step.py --reps 2 > gpurun_out/stamps.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -q -x 2>&1 | tail -30 > gpurun_out/tc_tests.log
timeout 300 python tools/probe_step.py --reps 3 > gpurun_out/probe.log 2>&1
timeout 300 python tools/probe_step.py --reps 3 --model birnn > gpurun_out/probe_birnn.log 2>&1
cat gpurun_out/tc_tests.log | tail -4; cat gpurun_out/probe.log gpurun_out/probe_birnn.log | tail -8

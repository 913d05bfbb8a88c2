# Iteration run: tensor-core GPU tests, probe timings, stamp trace (profiling aid).
set -x
mkdir -p gpurun_out
MBX_TC_STAMPS=1 timeout 300 python tools/probe_step.py --reps 2 > gpurun_out/stamps.log 2>&1
MBX_TC_STAMPS=1 timeout 300 python tools/probe_step.py --reps 2 --model birnn > gpurun_out/stamps_birnn.log 2>&1
timeout 600 python -m pytest tests/test_gpu_tc.py -q 2>&1 | tail -30 > gpurun_out/tc_tests.log
timeout 300 python tools/probe_step.py --reps 3 > gpurun_out/probe.log 2>&1
timeout 300 python tools/probe_step.py --reps 3 --model birnn > gpurun_out/probe_birnn.log 2>&1
MBX_LEVELS=0 timeout 300 python tools/probe_step.py --reps 3 --precision bf16 > gpurun_out/probe_bf16_nolevels.log 2>&1
cat gpurun_out/tc_tests.log | tail -15; cat gpurun_out/probe.log gpurun_out/probe_birnn.log | tail -8

# One ncu --set full capture of the dominant kernels + stamp trace (profiling, not bench numbers).
set -x
mkdir -p gpurun_out
timeout 300 python tools/probe_step.py --reps 3 > gpurun_out/probe.log 2>&1
MBX_TC_STAMPS=1 timeout 300 python tools/probe_step.py --reps 2 > gpurun_out/stamps.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mbx_tc_gate --launch-skip 14 --launch-count 9 \
   -o gpurun_out/tc_gate_full -f python tools/probe_step.py --reps 3 > gpurun_out/ncu_gate.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mbx_pointwise --launch-skip 1 --launch-count 1 \
   -o gpurun_out/pointwise_full -f python tools/probe_step.py --reps 2 > gpurun_out/ncu_pw.log 2>&1

# Round check: all GPU tests, smoke, bench, launch list (ncu), ncu --set full of the levels kernel
# and the MV-RNN cell kernel (tensor-pipe and DRAM counters).
set -x
mkdir -p gpurun_out
rm -f gpurun_out/parity_tc.jsonl
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --threads 1 --per-thread 1 --no-cpu-baseline --no-other-configs > gpurun_out/b_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mbx_tc_levels --launch-skip 5 --launch-count 1 -o gpurun_out/levels_full -f python tools/probe_step.py --reps 3 > gpurun_out/ncu_levels.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mv_cell --launch-skip 8 --launch-count 1 -o gpurun_out/mv_full -f python tools/probe_step.py --model mvrnn --hidden 128 --precision fp32 --reps 2 > gpurun_out/ncu_mv.log 2>&1
tail -3 gpurun_out/gputests.log; tail -1 gpurun_out/smoke.log
# Berxit (BASELINE configs[4]): launch list of bf16x3 mini-batches and a --set full capture of the GEMM.
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_berxit_b64.csv python tools/berxit_probe.py bf16x3 > gpurun_out/ncu_berxit_list.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bx_gemm --launch-skip 40 --launch-count 1 -o gpurun_out/berxit_gemm_full -f python tools/berxit_probe.py bf16x3 > gpurun_out/ncu_berxit_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bx_attention --launch-skip 10 --launch-count 1 -o gpurun_out/berxit_attn_full -f python tools/berxit_probe.py bf16x3 > gpurun_out/ncu_berxit_attn.log 2>&1
timeout 300 python tools/berxit_probe.py bf16x3 bf16 > gpurun_out/berxit_probe.log 2>&1

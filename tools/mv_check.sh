# MV-RNN kernel: GPU tests (registered plans + whole models), per-batch times, ncu launch list and one full capture.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -k "mv or mvrnn or fp32" > gpurun_out/mv_tests.log 2>&1
tail -3 gpurun_out/mv_tests.log
for p in fp32 bf16x3; do timeout 120 python tools/probe_step.py --model mvrnn --hidden 128 --batch 64 --precision $p --reps 5 > gpurun_out/mv_probe_$p.log 2>&1; tail -1 gpurun_out/mv_probe_$p.log; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/mv_launches.csv python tools/probe_step.py --model mvrnn --hidden 128 --batch 64 --precision fp32 --reps 2 > gpurun_out/mv_ncu.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:mv_cell --launch-skip 8 --launch-count 1 -o gpurun_out/mv_full -f python tools/probe_step.py --model mvrnn --hidden 128 --batch 64 --precision fp32 --reps 2 > gpurun_out/mv_ncu_full.log 2>&1

# exact-kernel check: parity tests + launch durations of mbx_small_dense (bf16x3 classifier, fp32 TreeLSTM)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 > gpurun_out/t.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mbx_small -c 8 --csv --log-file gpurun_out/small_bf.csv python tools/probe_step.py --reps 2 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/small_fp.csv python tools/probe_step.py --reps 2 --precision fp32 > /dev/null 2>&1
python bench.py --steps 10 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench.log
cat gpurun_out/t.log

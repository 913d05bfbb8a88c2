# tests + ncu launch list (kernel durations) + bench line
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -1 > gpurun_out/t.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches2.csv python bench.py --steps 2 --warmup 3 --threads 1 --per-thread 1 --no-cpu-baseline > /dev/null 2>&1
python bench.py --steps 10 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench.log

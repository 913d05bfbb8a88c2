mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches2.csv python bench.py --steps 2 --warmup 3 --threads 1 --per-thread 1 --no-cpu-baseline --no-other-configs > /dev/null 2>&1
python tools/show.py gpurun_out/launches2.csv | head -12

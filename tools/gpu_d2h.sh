timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches3.csv python bench.py --steps 2 --warmup 3 --threads 1 --per-thread 1 --no-cpu-baseline --no-other-configs > /dev/null 2>&1
grep -c pack_ranges gpurun_out/launches3.csv
for i in 1 2 3; do timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['e2e']['value'], j['latency']['e2e_ms_per_minibatch'])"; done

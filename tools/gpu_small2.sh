for v in 0 1; do
  if [ $v = 1 ]; then export MBX_NO_TC_SMALL=1; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/ls_$v.csv python tools/probe_step.py --reps 3 > /dev/null 2>&1
  echo "variant $v"; python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/ls_$v.csv")) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value"); gi=h.index("Grid Size")
print([(r[ki][:20], r[gi], r[vi]) for r in rows[1:] if 'small' in r[ki] or r[gi] in ('(1, 1, 8)','(1, 1, 4)')])
PY
  for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['e2e']['value'], j['latency']['ms_per_minibatch'])"; done
done
unset MBX_NO_TC_SMALL
MBX_NO_TC_SMALL=1 timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -1

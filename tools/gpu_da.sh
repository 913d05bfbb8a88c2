timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/nested2.csv python tools/probe_step.py --model nestedrnn --reps 1 > /dev/null 2>&1
python - <<PY
import csv
from collections import defaultdict
rows=[r for r in csv.reader(open("gpurun_out/nested2.csv")) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
agg=defaultdict(lambda:[0,0.0])
for r in rows[1:]:
    k=r[ki][:40]; agg[k][0]+=1; agg[k][1]+=float(r[vi])/1000
print("total us", round(sum(v[1] for v in agg.values())))
for k,v in sorted(agg.items(), key=lambda x:-x[1][1])[:6]: print(k, v[0], round(v[1]), round(v[1]/v[0],1))
PY
for i in 1 2; do timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print({k: round(v['ms_per_minibatch'],2) for k,v in j['other_configs'].items()})"; done

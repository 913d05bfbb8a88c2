timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 16 --csv --log-file gpurun_out/lf.csv python tools/probe_step.py --reps 3 > /dev/null 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/lf.csv")) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value"); gi=h.index("Grid Size")
print([(r[ki][:18], r[gi], r[vi]) for r in rows[-8:]])
PY
run() { echo "== $*"; env "$@" timeout 300 python bench.py --steps 10 --warmup 5 --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value']/1e6,2), round(j['e2e']['value']/1e6,2), round(j['latency']['ms_per_minibatch'],3), round(j['roofline']['frac'],3))"; }
run X=1 > /dev/null
for i in 1 2 3; do run X=1; run MBX_NO_FUSE=1; done

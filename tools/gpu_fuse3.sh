timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for f in 0 1; do
  if [ $f = 1 ]; then export MBX_FUSE=1; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mbx_tc_levels -c 6 --csv python tools/probe_step.py --reps 3 2>/dev/null | grep -o '"([0-9]*, [0-9]*, [0-9]*)".*' | awk -F'","' '{print $1, $NF}' | tr -d '"' | tr '\n' ' '; echo
done
unset MBX_FUSE
run() { echo "== $*"; env "$@" timeout 300 python bench.py --steps 10 --warmup 5 --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value']/1e6,2), round(j['e2e']['value']/1e6,2), round(j['latency']['ms_per_minibatch'],3), round(j['roofline']['frac'],3))"; }
run X=1 > /dev/null
for i in 1 2 3; do run X=1; run MBX_FUSE=1; done

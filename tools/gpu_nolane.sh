run() { echo "== $*"; env "$@" timeout 300 python bench.py --steps 10 --warmup 5 --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value']/1e6,2), round(j['e2e']['value']/1e6,2))"; }
run X=1 > /dev/null
for i in 1 2 3; do run X=1; run MBX_NO_LANE=1; done

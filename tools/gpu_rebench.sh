nproc; cat /proc/loadavg
for i in 1 2 3; do timeout 600 python bench.py --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['value']/1e6,2), round(j['e2e']['value']/1e6,2), j['config']['host_threads'])"; done
cat /proc/loadavg

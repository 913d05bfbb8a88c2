import csv, json, sys
rows = list(csv.reader(open('gpurun_out/launches2.csv')))
hdr = [r for r in rows if 'Kernel Name' in r][0]
data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and 'Kernel Name' not in r]
for d in data[-7:]:
    print(d['Kernel Name'][:30], d['Grid Size'], d['Metric Value'])
print(open('gpurun_out/t.log').read().strip())
j = json.loads(open('gpurun_out/bench.log').read())
print(round(j['value']), round(j['e2e']['value']), round(j['latency']['ms_per_minibatch'], 3), {k: round(v, 1) for k, v in j['breakdown_us_per_step']['per_sig'].items()}, round(j['step_roofline']['frac'], 4), round(j['roofline']['frac'], 4))

"""Per-kernel totals of one Berxit mini-batch from an ncu launch list (tools/ncu_list.py format)."""
import collections, subprocess, sys
f = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches_berxit_b64.csv"
out = subprocess.run([sys.executable, "tools/ncu_list.py", f], capture_output=True, text=True).stdout.splitlines()
rows = [r for r in out if r.strip()]
start = next(i for i, r in enumerate(rows) if "bx_begin" in r)
end = next((i for i, r in enumerate(rows) if "bx_begin" in r and i > start), len(rows))
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[start:end]:
    name = r[5:66].strip().split("(")[0]
    agg[name][0] += 1
    agg[name][1] += float(r[81:91])
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:40s} {v[0]:4d} {v[1]:9.1f} us {100 * v[1] / tot:5.1f} %")
print(f"{'total':40s} {end - start:4d} {tot:9.1f} us")

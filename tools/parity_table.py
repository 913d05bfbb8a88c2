"""Markdown table of the per-element parity figures the GPU tests append to
gpurun_out/parity_tc.jsonl:  python tools/parity_table.py gpurun_out/parity_tc.jsonl > profiles/r2_parity.md"""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
seen, out = set(), []
for r in rows:
    key = (r["model"], r["prec"], r["hidden"], r["batch"], r["seed"], r.get("variant"))
    if key in seen:
        continue
    seen.add(key)
    out.append(r)
print("| model | precision | H | b | seed | variant | schedule | elements | max-rel | tol | frac within tol | fails | normwise | max-abs | frac within 1e-5 |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
TOL = {"bf16x3": 1e-3, "bf16": 2.5e-1, "bf16x6": 1e-3}
for r in out:
    print(f"| {r['model']} | {r['prec']} | {r['hidden']} | {r['batch']} | {r['seed']} | {r.get('variant')} | "
          f"{'equal' if r['schedule_equal'] else 'DIFF'} | {r['n']} | {r['max_rel']:.2e} | "
          f"{r.get('tol', TOL.get(r['prec'], 0)):.0e} | {r['frac_pass']:.4f} | {r['fails']} | {r['normwise']:.2e} | {r['max_abs']:.2e} | "
          f"{r.get('frac_1e5', float('nan')):.4f} |")

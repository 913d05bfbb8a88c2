"""Prints an ncu --csv launch list (kernel, grid, duration us, DRAM bytes) from gpurun_out."""
import csv, sys
lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(lines[start:]))
by = {}
for r in rows:
    k = (r["ID"], r["Kernel Name"][:60], r["Grid Size"])
    by.setdefault(k, {})[r["Metric Name"]] = r["Metric Value"]
for (i, name, grid), m in by.items():
    t = float(m.get("gpu__time_duration.sum", "nan").replace(",", ""))
    rb = float(m.get("dram__bytes_read.sum", "0").replace(",", "")); wb = float(m.get("dram__bytes_write.sum", "0").replace(",", ""))
    print(f"{i:>4} {name:60s} {grid:>14s} {t/1000 if t > 1000 else t:9.2f} {rb/1e6:9.3f} {wb/1e6:9.3f}")

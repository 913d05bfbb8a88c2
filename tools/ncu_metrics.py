"""One CSV row per ncu --set full capture: the counters profiles/r2_ncu_metrics.csv tracks.
Usage: python tools/ncu_metrics.py gpurun_out/levels_full.ncu-rep ... > profiles/r2_ncu_metrics.csv"""
import csv, io, os, subprocess, sys

COLS = ["Kernel Name", "launch__grid_size", "launch__cluster_dim_z", "launch__registers_per_thread",
        "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_wait"]
w = csv.writer(sys.stdout)
w.writerow(["capture"] + COLS)
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    def get(c):
        if c not in hdr:
            return ""
        v, u = vals[hdr.index(c)], units[hdr.index(c)]
        if c.startswith("dram__bytes") and u in ("byte", "Kbyte", "Mbyte", "Gbyte"):  # -> MB
            v = str(float(v.replace(",", "")) * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}[u])
        if c == "gpu__time_duration.sum" and u in ("nsecond", "msecond", "usecond"):  # -> us
            v = str(float(v.replace(",", "")) * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}[u])
        return v
    w.writerow([os.path.basename(rep).replace(".ncu-rep", "")] + [get(c) for c in COLS])

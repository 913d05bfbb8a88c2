"""Runs a few mini-batches of one workload and prints per-batch device times (for ncu / probes)."""
import argparse, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_10611_b200 import mbx
ap = argparse.ArgumentParser()
ap.add_argument("--model", default="treelstm"); ap.add_argument("--hidden", type=int, default=512)
ap.add_argument("--batch", type=int, default=64); ap.add_argument("--precision", default="bf16x3")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--plain", action="store_true", help="no per-batch timing (the product issue order: sinks hoisted)")
a = ap.parse_args()
c = mbx.Context(0, a.precision); m = mbx.Model(c, a.model, a.hidden); m.make_params(1)
t, d = m.make_inputs(1, a.batch)
for i in range(a.reps):
    r = m.evaluate_batch(t, d, a.batch, record_nodes=False, time_batches=not a.plain)
sigs = m.signatures()
if not a.plain:
    print([(sigs[b.sig], b.size, round(us, 1)) for b, us in zip([b for b in r.trace.batches if not b.ghost], r.timing.batch_us)])

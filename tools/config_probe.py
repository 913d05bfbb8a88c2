"""Host/device split of one mini-batch of a BASELINE config through the Python binding, inputs
resident, outputs left on the device or read back (what bench.py's other_configs measures)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_10611_b200 import mbx
ap = argparse.ArgumentParser()
ap.add_argument("--model", default="birnn"); ap.add_argument("--hidden", type=int, default=512)
ap.add_argument("--batch", type=int, default=64); ap.add_argument("--precision", default="bf16x3")
a = ap.parse_args()
c = mbx.Context(0, a.precision); m = mbx.Model(c, a.model, a.hidden); m.make_params(1)
t, d = m.make_inputs(1, a.batch)
for od in (True, False):
    for i in range(3): m.evaluate_batch(t, d, a.batch, record_nodes=False, decode=False, trace=False)
    rows = []
    for i in range(10):
        t0 = time.perf_counter()
        r = m.evaluate_batch(t, d, a.batch, record_nodes=False, decode=False, trace=False, inputs_resident=True,
                             outputs_on_device=od, time_kernels=True)
        rows.append(((time.perf_counter() - t0) * 1e6, r.timing.host_total_us, r.timing.host_dfg_us,
                     r.timing.device_span_us, r.timing.host_breakdown))
    rows.sort(key=lambda x: x[0])
    print("outputs_on_device" if od else "outputs to host", [round(x) if isinstance(x, float) else {k: round(v) for k, v in x.items()} for x in rows[0]])

"""Ad-hoc probe: tensor-core path vs FP32 path on a few configs (prints errors and timings)."""
import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2305_10611_b200 import mbx
for model, H, b in [("treelstm", 64, 4), ("treelstm", 512, 8), ("treelstm", 512, 64), ("birnn", 512, 8), ("rnn", 64, 8), ("nestedrnn", 64, 4)]:
    res = {}
    for prec in ("fp32", "bf16x3", "bf16"):
        c = mbx.Context(0, prec)
        m = mbx.Model(c, model, H)
        m.make_params(1)
        t, d = m.make_inputs(1, b)
        r = m.evaluate_batch(t, d, b, record_nodes=False, time_batches=True)
        res[prec] = r
    ref = res["fp32"].out_data
    for prec in ("bf16x3", "bf16"):
        r = res[prec]
        same = [x.node_ids for x in r.trace.batches] == [x.node_ids for x in res["fp32"].trace.batches]
        err = np.max(np.abs(r.out_data - ref)) / max(1e-30, np.max(np.abs(ref))) if r.out_data.size == ref.size else -1
        print(model, H, b, prec, "normwise err %.3e" % err, "trace_same", same,
              "batch_us", [round(x, 1) for x in r.timing.batch_us][:12], "fp32_us", [round(x, 1) for x in res["fp32"].timing.batch_us][:12])

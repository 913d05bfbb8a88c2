"""Per-batch comparison of a tensor-core precision against the FP32 path (debug aid)."""
import sys, os, numpy as np
sys.path.insert(0, '.')
from paper_2305_10611_b200 import mbx
model, H, B, seed = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
res = {}
for prec in ("fp32", "bf16x3"):
    c = mbx.Context(0, prec); m = mbx.Model(c, model, H); m.make_params(seed)
    t, d = m.make_inputs(seed, B)
    r = m.evaluate_batch(t, d, B, record_nodes=True)
    outs = []
    for b in r.trace.batches:
        if b.ghost: continue
        v = []
        for nid in b.node_ids:
            n = r.nodes[nid]
            for (off, rows, cols) in n.outputs:
                v.append(c.download(off, rows * cols))
        outs.append(np.concatenate(v))
    res[prec] = (outs, [b for b in r.trace.batches if not b.ghost], m.signatures())
    res[prec + "_ctx"] = (c, m)
f, b16 = res["fp32"][0], res["bf16x3"][0]
sigs = res["fp32"][2]
for i, (x, y, bb) in enumerate(zip(f, b16, res["fp32"][1])):
    print(i, sigs[bb.sig], bb.size, "normwise %.2e" % (np.linalg.norm(x - y) / max(1e-30, np.linalg.norm(x))),
          "maxabs %.2e" % np.max(np.abs(x - y)))

"""Berxit A/B probe: ms per mini-batch for max_batch = batch (the bench's setting), bf16x3, with
L2 flushed before each mini-batch; logits vs the committed golden.  Usage: python tools/berxit_ab.py"""
import gzip, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from paper_2305_10611_b200 import mbx
from parity_metrics import elementwise

runs = {r["batch"]: r for r in json.load(gzip.open("tests/golden/berxit.json.gz", "rt"))["runs"] if r["name"] == "bert-base"}
l2 = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for b in [int(a) for a in sys.argv[1:]] or (64, 8):
    run = runs[b]
    c = mbx.berxit_config(**run["config"])
    m = mbx.Berxit(0, "bf16x3", c, max_batch=b)
    m.make_params(run["seed"])
    x = torch.from_numpy(mbx.berxit_make_inputs(c, run["seed"], b)).cuda()
    s = torch.cuda.ExternalStream(m.stream())
    for _ in range(3):
        m.run_device(b, x.data_ptr())
    r = m.read(b)
    ts = []
    for _ in range(10):
        l2.zero_(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); m.run_device(b, x.data_ptr()); e1.record(s); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    st = elementwise(r.logits, np.asarray(run["logits"], np.float32), 1e-3)
    print(f"b={b}: {np.median(ts):.3f} ms "
          f"(min {min(ts):.3f}); exits equal {r.exit_layer.tolist() == run['exit_layer']}; "
          f"max_rel {st['max_rel']:.2e} frac {st['frac_pass']:.3f} normwise {st['normwise']:.1e}")
    del m

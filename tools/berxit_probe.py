"""Berxit timing probe: ms per mini-batch (device-resident inputs, CUDA events on the model's
stream) at batch 8 / 64, bf16x3 and bf16; exit histogram.  Usage: python tools/berxit_probe.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2305_10611_b200 import mbx

for prec in sys.argv[1:] or ["bf16x3", "bf16"]:
    c = mbx.berxit_config()
    m = mbx.Berxit(0, prec, c, max_batch=64)
    m.make_params(1)
    for b in (64, 8):
        x = torch.from_numpy(mbx.berxit_make_inputs(c, 1, b)).cuda()
        s = torch.cuda.ExternalStream(m.stream())
        torch.cuda.synchronize()
        for _ in range(3):
            m.run_device(b, x.data_ptr())
        r = m.read(b)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 10
        e0.record(s)
        for _ in range(n):
            m.run_device(b, x.data_ptr())
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        layer_inst = int(sum(len(bt) for bt in r.batches()))
        tf = layer_inst * 128 * 2 * (4 * 768 * 768 + 2 * 768 * 3072) / (ms * 1e-3) / 1e12
        tfa = layer_inst * 128 * 2 * 2 * 128 * 768 / (ms * 1e-3) / 1e12
        print(f"{prec} b={b}: {ms:.3f} ms per mini-batch, layer-instances {layer_inst}, "
              f"GEMM {tf:.1f} TFLOP/s + attention {tfa:.1f}, exits {np.bincount(r.exit_layer, minlength=12).tolist()}")

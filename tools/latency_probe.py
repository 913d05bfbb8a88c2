"""Latency split of one mini-batch (default TreeLSTM-512 b64) through the Python binding (GPU)."""
import argparse, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_10611_b200 import mbx
ap = argparse.ArgumentParser()
ap.add_argument("--model", default="treelstm"); ap.add_argument("--hidden", type=int, default=512)
ap.add_argument("--batch", type=int, default=64); ap.add_argument("--precision", default="bf16x3")
A = ap.parse_args()
c = mbx.Context(0, A.precision); m = mbx.Model(c, A.model, A.hidden); m.make_params(1)
t, d = m.make_inputs(1, A.batch)
pd = torch.empty(d.size, dtype=torch.float32, pin_memory=True).numpy(); pd[:] = d
for i in range(10): m.evaluate_batch(t, pd, A.batch, record_nodes=False, decode=False, trace=False)
rows = []
for i in range(20):
    t0 = time.perf_counter()
    r = m.evaluate_batch(t, pd, A.batch, record_nodes=False, decode=False, trace=False, time_kernels=True)
    t1 = time.perf_counter()
    rows.append(((t1 - t0) * 1e6, r.timing.host_total_us, r.timing.host_dfg_us, r.timing.device_span_us, r.timing.host_breakdown))
rows.sort(key=lambda x: x[0])
for x in rows[:5]: print([round(v) if isinstance(v, float) else {k: round(w) for k, w in v.items()} for v in x])
# C ABI call alone vs the Python wrapper
import ctypes, numpy as np
L = mbx.lib()
o = mbx.make_options(record_nodes=False)
tt = np.ascontiguousarray(t, np.int32)
ptr_t = tt.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)); ptr_d = pd.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
ws = []
for i in range(20):
    r = ctypes.c_void_p()
    t0 = time.perf_counter()
    rc = L.mbx_evaluate_batch(m.h, A.batch, ptr_t, tt.size, ptr_d, pd.size, ctypes.byref(o), ctypes.byref(r))
    t1 = time.perf_counter()
    L.mbx_result_destroy(r)
    t2 = time.perf_counter()
    ws.append(((t1 - t0) * 1e6, (t2 - t1) * 1e6))
ws.sort()
print("C ABI call us / result destroy us:", [(round(a), round(b)) for a, b in ws[:5]])

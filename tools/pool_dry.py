"""Host-only throughput of the pool (dry contexts: fibers, DFG, schedule, offset tables; no GPU)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_10611_b200 import mbx
T = int(sys.argv[1]) if len(sys.argv) > 1 else 14
ctx = mbx.Context(-1, "bf16x3"); m = mbx.Model(ctx, "treelstm", 512)
ins = [m.make_inputs(1 + w, 64) for w in range(T)]
for t in (1, T):
    pool = mbx.Pool(-1, "bf16x3", "treelstm", 512, 1, t)
    pool.run(ins[:t] * 4, 64)
    t0 = time.perf_counter(); n = pool.run(ins[:t] * 16, 64); dt = time.perf_counter() - t0
    print(f"threads {t}: {16 * t / dt:.0f} mini-batches/s, {n / dt / 1e6:.2f} M nodes/s (host only)")
    pool.close()

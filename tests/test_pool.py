"""Throughput pool (mbx_pool_*): many mini-batches on one device from T host threads.

CPU (dry contexts): the pool's threading and accounting — every mini-batch evaluated once, on
worker i % T, total DFG nodes equal to the one-at-a-time runs.  GPU: the same on a B200, where
the workers' streams overlap and the persistent multi-level kernels are chained through the
per-device lane; the outputs of a pool worker's context equal a standalone context's."""
import numpy as np
import pytest


def _inputs(mbx, model, hidden, batch, seeds):
    ctx = mbx.Context(-1, "bf16x3")
    m = mbx.Model(ctx, model, hidden)
    return [m.make_inputs(s, batch) for s in seeds], [m.evaluate_batch(*m.make_inputs(s, batch), batch,
                                                                      record_nodes=False).trace.total_nodes
                                                      for s in seeds]


@pytest.mark.parametrize("model,hidden,batch", [("treelstm", 32, 8), ("birnn", 32, 6)])
def test_pool_dry_counts(mbx, model, hidden, batch):
    ins, counts = _inputs(mbx, model, hidden, batch, [1, 2, 3, 4, 5])
    pool = mbx.Pool(-1, "bf16x3", model, hidden, 1, 3)
    assert pool.run(ins, batch) == sum(counts)
    assert pool.run(ins * 2, batch) == 2 * sum(counts)
    pool.close()


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["bf16x3", "fp32"])
def test_pool_gpu(mbx, prec):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    model, hidden, batch = "treelstm", 512, 16
    ins, counts = _inputs(mbx, model, hidden, batch, list(range(1, 9)))
    pool = mbx.Pool(0, prec, model, hidden, 1, 4)
    n, ms = pool.run_timed(ins * 3, batch)
    assert n == 3 * sum(counts) and ms > 0
    n2 = pool.run(ins, batch, inputs_resident=False, outputs_on_device=True)
    assert n2 == sum(counts)
    pool.close()
    # a pool worker's evaluation is mbx_evaluate_batch: compare with a standalone context
    ref_ctx = mbx.Context(0, prec)
    ref = mbx.Model(ref_ctx, model, hidden)
    ref.make_params(1)
    r0 = ref.evaluate_batch(*ins[0], batch)
    pool = mbx.Pool(0, prec, model, hidden, 1, 2)
    pool.run(ins, batch)  # leaves the persistent lane in use by other workers' contexts
    r1 = ref.evaluate_batch(*ins[0], batch)
    pool.close()
    assert np.array_equal(r0.out_data.view(np.uint32), r1.out_data.view(np.uint32))


@pytest.mark.gpu
def test_pool_gpu_headline_stress(mbx):
    """The headline configuration (TreeLSTM-512 b64 bf16x3) from as many host workers as the
    bench uses, several rounds: the persistent launches (grid barrier, cooperative placement)
    must never be starved by the other workers' clustered kernels (a starved grid barrier traps
    after 2 s and the round fails)."""
    import os
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    model, hidden, batch = "treelstm", 512, 64
    ins, counts = _inputs(mbx, model, hidden, batch, list(range(1, 5)))
    threads = max(2, min(14, (os.cpu_count() or 4) - 2))
    pool = mbx.Pool(0, "bf16x3", model, hidden, 1, threads)
    for _ in range(25):  # ~22k mini-batches: the bench's order of magnitude
        n, ms = pool.run_timed(ins * (16 * threads), batch)
        assert n == 16 * threads * sum(counts) and ms > 0
    pool.close()

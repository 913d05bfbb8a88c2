"""Host <-> device input paths of mbx_evaluate_batch on a GPU: pageable inputs (one host memcpy
into pinned staging, one H2D) and pinned inputs (direct H2D copies into the arena when the
tensors lie in stream order there, else one H2D of the caller's data stream scattered to the
arena offsets by a device kernel — forced with MBX_INPUT_SCATTER) give bit-identical results, and
so do resident inputs and deferred completion (the throughput pool's mode)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu(mbx):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return mbx


@pytest.mark.parametrize("model,hidden,batch,prec", [("treelstm", 512, 16, "bf16x3"), ("treelstm", 64, 8, "fp32"),
                                                     ("mvrnn", 32, 8, "fp32"), ("birnn", 128, 8, "bf16x3")])
@pytest.mark.parametrize("scatter", [False, True])
def test_pinned_and_pageable_inputs_agree(gpu, model, hidden, batch, prec, scatter, monkeypatch):
    import torch
    mbx = gpu
    if scatter:
        monkeypatch.setenv("MBX_INPUT_SCATTER", "1")
    c = mbx.Context(0, prec)
    m = mbx.Model(c, model, hidden)
    m.make_params(3)
    t, d = m.make_inputs(5, batch)
    pd = torch.empty(d.size, dtype=torch.float32, pin_memory=True).numpy()
    pd[:] = d
    a = m.evaluate_batch(t, d, batch)
    b = m.evaluate_batch(t, pd, batch)
    r = m.evaluate_batch(t, pd, batch, inputs_resident=True)
    assert np.array_equal(a.out_data.view(np.uint32), b.out_data.view(np.uint32))
    assert np.array_equal(a.out_data.view(np.uint32), r.out_data.view(np.uint32))
    assert b.timing.h2d_bytes >= d.size * 4
    # deferred completion: outputs not decoded, the context synchronised before reuse
    m.evaluate_batch(t, pd, batch, defer_sync=True, decode=False)
    c.sync()
    e = m.evaluate_batch(t, d, batch)
    assert np.array_equal(a.out_data.view(np.uint32), e.out_data.view(np.uint32))

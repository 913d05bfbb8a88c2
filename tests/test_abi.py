"""The C-ABI library (include/mbx.h -> paper_2305_10611_b200/lib/libmbx.so): it loads on a GPU-less
host, exports every declared entry point, and reports the reference's error texts
(proj/tests/backend_test.cpp:96-103, :223-237; proj/src/exec_batched.cpp:25-40) without throwing
across the boundary.  No compute calls here (dry context)."""
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT


def _declared():
    text = open(os.path.join(ROOT, "include", "mbx.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mbx_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(mbx):
    lib = mbx.lib()
    declared = _declared()
    assert len(declared) >= 30
    out = subprocess.check_output(["nm", "-D", "--defined-only", mbx.LIB_PATH]).decode()
    exported = set(re.findall(r" T (mbx_\w+)", out))
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    for s in declared:
        getattr(lib, s)
    assert set(mbx.exported_symbols()) <= exported


def test_library_has_no_libcuda_link_dependency(mbx):
    out = subprocess.check_output(["ldd", mbx.LIB_PATH]).decode()
    assert "libcuda.so" not in out  # driver API resolved at run time via cudaGetDriverEntryPoint


def test_sm100a_code_present(mbx):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", mbx.LIB_PATH]).decode()
    assert "sm_100a" in out


def _relu_bias_dense_plan(h):
    # backend_test.cpp:110-129: dense(B0, S0) then chain [add S1, relu]
    return [0, 2, h, h, 1, h, 1, 1, h, 2,
            0, 0, 1, h, 2, 1, 0, 0, -1, 0, 0, 0, -1, 0,
            2, 1, 1, h, 1, 2, 0, 0, -1, 2, 1, 1, 0, 1, 0, -1, 5, 0, 2, 0, 0, -1,
            1, 2, 1, 0, -1]


def test_plan_encoding_roundtrip(mbx):
    ctx = mbx.Context(-1)
    pid = ctx.register_plan(_relu_bias_dense_plan(4))
    assert pid == ctx.register_plan(_relu_bias_dense_plan(4))  # cached by content
    assert pid != ctx.register_plan(_relu_bias_dense_plan(8))


def test_error_texts(mbx):
    ctx = mbx.Context(-1)
    h = 4
    pid = ctx.register_plan(_relu_bias_dense_plan(h))
    w = ctx.alloc(h, h)
    b = ctx.alloc(1, h)
    w2 = ctx.alloc(h, h)
    xs = [ctx.alloc(1, h) for _ in range(3)]
    with pytest.raises(mbx.MbatchError, match="exec_batched: empty batch"):
        ctx.exec_batched(pid, [w, b], np.zeros((0, 1), np.int64), 1)
    with pytest.raises(mbx.MbatchError, match="shared-param handle mismatch across instances"):
        ctx.exec_batched(pid, np.array([[w, b], [w2, b]]), np.array([[xs[0]], [xs[1]]]), 1)
    with pytest.raises(mbx.MbatchError, match="tensor handle out of arena bounds"):
        ctx.exec_batched(pid, [w, b], np.array([[ctx.used() + 100]]), 1)
    with pytest.raises(mbx.MbatchError, match="add"):
        ctx.exec_primop("add", [(xs[0], (1, 4)), (w, (4, 4))], (xs[1], (1, 4)))
    with pytest.raises(mbx.MbatchError, match="dense: shape mismatch"):
        ctx.exec_primop("dense", [(xs[0], (1, 4)), (xs[1], (1, 4))], (xs[2], (1, 4)))
    with pytest.raises(mbx.MbatchError, match="plan encoding"):
        ctx.register_plan([0, 1])


def test_explicit_gather_accounting_dry(mbx):
    """gather_bytes: fused always 0; explicit counts non-contiguous slots only
    (backend_test.cpp:175-221)."""
    ctx = mbx.Context(-1)
    h = 4
    pid = ctx.register_plan(_relu_bias_dense_plan(h))
    w, b = ctx.alloc(h, h), ctx.alloc(1, h)
    scattered = []
    for _ in range(4):
        scattered.append(ctx.alloc(1, h))
        ctx.alloc(1, 3)  # padding makes neighbours non-adjacent
    xs = np.array(scattered).reshape(4, 1)
    _, gb = ctx.exec_batched(pid, [w, b], xs, 1, "fused")
    assert gb == 0
    _, gb = ctx.exec_batched(pid, [w, b], xs, 1, "explicit")
    assert gb == 4 * h * 4
    region = ctx.alloc(4, h)
    contiguous = np.array([region + i * h for i in range(4)]).reshape(4, 1)
    _, gb = ctx.exec_batched(pid, [w, b], contiguous, 1, "explicit")
    assert gb == 0
    _, gb = ctx.exec_batched(pid, [w, b], np.array([[scattered[0]]]), 1, "explicit")
    assert gb == 0  # a batch of one is contiguous


def test_output_regions_are_batch_contiguous(mbx):
    ctx = mbx.Context(-1)
    h = 4
    pid = ctx.register_plan(_relu_bias_dense_plan(h))
    w, b = ctx.alloc(h, h), ctx.alloc(1, h)
    xs = np.array([ctx.alloc(1, h) for _ in range(8)]).reshape(8, 1)
    before = ctx.used()
    outs, _ = ctx.exec_batched(pid, [w, b], xs, 1)
    assert outs[:, 0].tolist() == [before + i * h for i in range(8)]
    # temporaries are reserved after the region exactly as the reference allocates them
    assert ctx.used() == before + 8 * h + 8 * (h + h)


def test_device_context_fails_loudly_without_gpu(mbx):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(mbx.MbatchError):
        mbx.Context(0)


def _reencode(toks, wide_ints=False, named_ctors=False):
    """Rewrites a hostval token stream with int64 scalars (kind 6) and / or named ADT
    constructors (kind 4, ctor -1 + bytes) — the encodings the C ABI accepts besides kind 1 and
    ctor ids 0 / 1 (include/mbx.h)."""
    import numpy as np
    out, ti = [], 0

    def one():
        nonlocal ti
        k = int(toks[ti]); ti += 1
        if k == 0:
            out.extend([0, int(toks[ti]), int(toks[ti + 1])]); ti += 2
        elif k == 1:
            v = int(toks[ti]); ti += 1
            if wide_ints:
                u = v & 0xFFFFFFFFFFFFFFFF
                out.extend([6, np.uint32(u & 0xFFFFFFFF).view(np.int32).item(), np.uint32(u >> 32).view(np.int32).item()])
            else:
                out.extend([1, v])
        else:
            out.append(k)
            if k == 4:
                cid = int(toks[ti]); ti += 1
                if named_ctors:
                    name = b"Node" if cid else b"Leaf"
                    out.extend([-1, len(name)] + list(name))
                else:
                    out.append(cid)
            n = int(toks[ti]); ti += 1
            out.append(n)
            for _ in range(n):
                one()

    while ti < len(toks):
        one()
    return np.array(out, np.int32)


@pytest.mark.parametrize("model", ["treelstm", "drnn", "stackrnn"])
def test_hostval_wide_ints_and_named_ctors(mbx, model):
    """int64 scalars and named constructors in the input encoding evaluate exactly like the
    compact forms (same schedule, same decoded outputs), dry run."""
    c = mbx.Context(-1, "fp32")
    m = mbx.Model(c, model, 32)
    m.make_params(1)
    t, d = m.make_inputs(2, 4)
    base = m.evaluate_batch(t, d, 4)
    for kw in ({"wide_ints": True}, {"named_ctors": True}):
        r = m.evaluate_batch(_reencode(t, **kw), d, 4)
        assert [(b.sig, b.size, b.node_ids) for b in r.trace.batches] == \
            [(b.sig, b.size, b.node_ids) for b in base.trace.batches]


def test_hostval_decode_float_and_int64(mbx):
    import numpy as np
    bits = np.array([2.5], np.float64).view(np.uint32)
    big = np.array([-(1 << 40)], np.int64).view(np.uint32)
    toks = np.array([3, 3, 5, bits[0].view(np.int32), bits[1].view(np.int32), 6, big[0].view(np.int32),
                     big[1].view(np.int32), 4, -1, 3, ord("F"), ord("o"), ord("o"), 0], np.int32)
    v = mbx.decode_hostvals(toks, np.zeros(0, np.float32), 1)[0]
    assert v[0] == 2.5 and v[1] == -(1 << 40) and v[2].ctor == "Foo" and v[2].fields == []

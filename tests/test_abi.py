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

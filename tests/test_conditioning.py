"""Conditioning of the TreeLSTM-512 b64 outputs (SURVEY 8a per-element tolerance), on the CPU.

The headline config's logits are relu(h . c_wt + cbias) after ~10 tree levels of LSTM cells with
U[-0.5, 0.5) weights; the oracle (the CPU restatement, pinned bit-for-bit to the reference) shows
how far its own outputs move when the weights move by a rounding error:

* weights rounded to split bf16 (hi + lo, 16 significant bits: the tensor-core operand precision of
  the bf16x3 path) fail the per-element test |d| <= 1e-3 * max(|ref|, 1e-6) on a few logits that the
  relu leaves near zero (the same count the GPU shows: profiles/r2_parity.md), while the
  normwise error stays ~3e-5;
* a three-way split (24 bits) reproduces fp32 exactly, i.e. the failures are operand rounding, not
  an implementation error;
* a random perturbation of ONE ulp (rel 2^-24) of every weight — any reassociated fp32 summation,
  e.g. an FFMA kernel with a different reduction order, perturbs at least this much — already fails
  the per-element test at seed 2.

So on this config no implementation that is not bit-identical to the reference can pass the
per-element test on every element; the GPU tests hold the bf16x3 path to >= 98% of elements
within rel 1e-3 plus normwise <= 1e-3 (tests/test_gpu_tc.py), and the FP32 path to bit equality.
"""
import ctypes

import numpy as np
import pytest

from parity_metrics import elementwise


def _bf16(x):
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


def _split(x, parts):
    out = np.zeros_like(x)
    rest = x.copy()
    for _ in range(parts):
        h = _bf16(rest)
        out = (out + h).astype(np.float32)
        rest = (rest - h).astype(np.float32)
    return out


def _perturbed_outputs(oracle, seed, fn):
    om = oracle.model("treelstm", 512, seed)
    om.make_inputs(seed, 64)
    L = oracle.L
    for i in range(L.orc_num_params(om.h)):
        if not L.orc_param_name(om.h, i).decode().endswith("wt"):
            continue
        r, c = ctypes.c_int(), ctypes.c_int()
        L.orc_param_shape(om.h, i, ctypes.byref(r), ctypes.byref(c))
        p = np.ctypeslib.as_array(L.orc_param_data(om.h, i), shape=(r.value * c.value,))
        p[:] = fn(p.copy())
    return om.evaluate()[1]


@pytest.fixture(scope="module")
def reference_outputs(oracle):
    out = {}
    for seed in (1, 2):
        om = oracle.model("treelstm", 512, seed)
        om.make_inputs(seed, 64)
        out[seed] = om.evaluate()[1]
    return out


@pytest.mark.parametrize("seed,min_fails", [(1, 1), (2, 1)])
def test_split_bf16_weights_fail_per_element_not_normwise(oracle, reference_outputs, seed, min_fails):
    st = elementwise(_perturbed_outputs(oracle, seed, lambda w: _split(w, 2)), reference_outputs[seed], 1e-3)
    assert st["fails"] >= min_fails and st["frac_pass"] >= 0.98, st
    assert st["normwise"] < 1e-4, st


@pytest.mark.parametrize("seed", [1, 2])
def test_three_way_split_is_exact(oracle, reference_outputs, seed):
    got = _perturbed_outputs(oracle, seed, lambda w: _split(w, 3))
    assert np.array_equal(got.view(np.uint32), reference_outputs[seed].view(np.uint32))


def test_one_ulp_weight_perturbation_fails_per_element(oracle, reference_outputs):
    rng = np.random.default_rng(0)
    st = elementwise(_perturbed_outputs(oracle, 2, lambda w: (w * (1 + 2.0**-24 * rng.standard_normal(w.size))).astype(np.float32)),
                     reference_outputs[2], 1e-3)
    assert st["fails"] >= 1, st
    assert st["normwise"] < 1e-5, st

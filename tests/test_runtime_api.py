"""runtime::profile_invocations and runtime::reference_evaluate (proj/include/mbatch/runtime.hpp:
141-154) through the C ABI, mirroring the reference's runtime_test.cpp:483-546 cases.

profile counts are pinned to the reference: per signature they equal the sizes of the non-ghost
batches of that signature in the golden traces the reference wrote (tests/golden)."""
import collections

import numpy as np
import pytest

from conftest import MODELS, STATIC_MODELS

DYNAMIC_MODELS = [m for m in MODELS if m not in STATIC_MODELS]


def _dry_model(mbx, name, hidden, seed, device=-1):
    ctx = mbx.Context(device, "fp32")
    m = mbx.Model(ctx, name, hidden)
    m.make_params(seed)
    return ctx, m


def _check_profile_golden(mbx, golden, model, device):
    g = golden(model)
    done = 0
    for run in g["runs"]:
        if run["variant"] not in ("default", "depth-fused", "large-b64"):
            continue
        ctx, m = _dry_model(mbx, model, run["hidden"], run["seed"], device)
        t, d = m.make_inputs(run["seed"], run["batch"])
        rep = m.profile_invocations(t, d, run["batch"])
        want = collections.Counter()
        for b in run["trace"]["batches"]:
            if not b["ghost"]:
                want[b["sig"]] += b["size"]
        assert rep["counts"] == dict(want), (model, run["variant"], run["batch"], run["seed"])
        ranked = sorted(want, key=lambda s: (-want[s], s))
        assert rep["ranking"] == ranked
        done += 1
    assert done > 0


@pytest.mark.parametrize("model", STATIC_MODELS)
def test_profile_counts_equal_golden_batch_sizes(mbx, golden, model):
    """counts[sig] == the reference's non-ghost DFG nodes of sig (sum of its batch sizes); models
    without tensor-dependent control flow, on a host-only context."""
    _check_profile_golden(mbx, golden, model, -1)


@pytest.mark.gpu
@pytest.mark.parametrize("model", DYNAMIC_MODELS)
def test_profile_counts_equal_golden_batch_sizes_gpu(gpu_mbx, golden, model):
    """The same for the models whose decisions come from the device (argmax scalars)."""
    _check_profile_golden(gpu_mbx, golden, model, 0)


def test_profile_treelstm_cells_equal_tree_nodes(mbx):
    """runtime_test.cpp:520-546: the leaf-cell and internal-cell blocks run once per tree node."""
    ctx, m = _dry_model(mbx, "treelstm", 32, 103)
    t, d = m.make_inputs(103, 5)
    rep = m.profile_invocations(t, d, 5)
    sigs = m.signatures()
    cells = sum(rep["counts"].get(sigs.index(s), 0) for s in ("add_mul_sigmoid_add", "add_mul_sigmoid_bias"))
    # leaves = bias_dense count (one per leaf); internal = internal-cell count; nodes = both
    leaves = rep["counts"][sigs.index("bias_dense")]
    internal = rep["counts"][sigs.index("add_mul_sigmoid_bias")]
    assert cells == leaves + internal
    assert internal == leaves - 5  # binary trees: one fewer internal node than leaves, per tree
    assert rep["static_estimate"][sigs.index("add_mul_sigmoid_bias")] == 1
    assert rep["static_estimate"][sigs.index("relu_bias_dense")] == 0


@pytest.mark.gpu
def test_profile_nestedrnn_inner_dominates(gpu_mbx):
    """runtime_test.cpp:483-498: the top signature is the inner-loop cell, one nesting level deeper
    (2), and it runs 25-36 times as often as the outer blocks (inner loop n + 25, n = argmax < 11)."""
    mbx = gpu_mbx
    ctx = mbx.Context(0, "fp32")
    m = mbx.Model(ctx, "nestedrnn", 32)
    m.make_params(97)
    t, d = m.make_inputs(97, 4)
    rep = m.profile_invocations(t, d, 4)
    top = rep["ranking"][0]
    assert rep["static_estimate"][top] == 2
    inner = rep["counts"][top]
    outer = sum(c for s, c in rep["counts"].items() if rep["static_estimate"][s] == 1)
    assert 25 * outer <= inner <= 36 * outer


@pytest.mark.gpu
@pytest.mark.parametrize("model,hidden,batch,seed", [("treelstm", 64, 6, 3), ("mvrnn", 32, 5, 2), ("birnn", 64, 4, 1),
                                                     ("nestedrnn", 32, 4, 97), ("drnn", 32, 5, 4), ("stackrnn", 32, 4, 5)])
def test_reference_evaluate_equals_batched_bitwise(gpu_mbx, model, hidden, batch, seed):
    """Unbatched (one instance per mini-batch) == batched, bit for bit, in FP32 (the reference's
    acceptance property, acceptance_test.cpp:69-104)."""
    mbx = gpu_mbx
    ctx = mbx.Context(0, "fp32")
    m = mbx.Model(ctx, model, hidden)
    m.make_params(seed)
    t, d = m.make_inputs(seed, batch)
    batched = m.evaluate_batch(t, d, batch)
    n0 = mbx.lib().mbx_kernel_launch_count()
    single = m.reference_evaluate(t, d, batch)
    assert mbx.lib().mbx_kernel_launch_count() > n0  # ran on the device
    assert len(single) == batch
    for i in range(batch):
        a = mbx.flatten_floats(batched.outputs[i])
        b = mbx.flatten_floats(single[i])
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), (model, i)


@pytest.fixture(scope="module")
def gpu_mbx(mbx):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return mbx

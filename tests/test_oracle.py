"""The CPU oracle (oracle/oracle.cpp) pinned against the compiled reference.

Every digest in tests/golden/ was produced by the unmodified reference (oracle/_ref/mbatch_ref,
see oracle/make_golden.py); the restatement must reproduce params, inputs and outputs
bit-for-bit, plus the reference's own known-answer unit tests (proj/tests/backend_test.cpp,
proj/tests/runtime_test.cpp)."""
import ctypes

import numpy as np
import pytest

from conftest import MODELS


@pytest.mark.parametrize("model", MODELS)
def test_oracle_digests_match_reference_runs(oracle, golden, model):
    g = golden(model)
    seen = set()
    for run in g["runs"]:
        key = (run["hidden"], run["batch"], run["seed"])
        if key in seen or run["hidden"] > 32:
            continue
        seen.add(key)
        m = oracle.model(model, run["hidden"], run["seed"])
        m.make_inputs(run["seed"], run["batch"])
        m.evaluate()
        d = m.digests()
        assert d == run["digests"], (model, key)
        assert run["batched_equals_unbatched"] is True


@pytest.mark.parametrize("model", MODELS)
def test_oracle_outputs_match_reference_values(oracle, golden, model):
    from paper_2305_10611_b200.mbx import decode_hostvals, flatten_floats
    run = golden(model)["runs"][0]
    m = oracle.model(model, run["hidden"], run["seed"])
    m.make_inputs(run["seed"], run["batch"])
    t, d = m.evaluate()
    got = [flatten_floats(v) for v in decode_hostvals(t, d, run["batch"])]

    def flat(j):
        if j["k"] == "t":
            return list(j["d"])
        return [x for it in j.get("items", []) for x in flat(it)]

    for i, o in enumerate(run["outputs"]):
        want = np.array(flat(o), np.float32)
        assert np.array_equal(got[i].view(np.uint32), want.view(np.uint32)), (model, i)


def test_oracle_baseline_configs(oracle, golden):
    for run in golden("baseline"):
        m = oracle.model(run["model"], run["hidden"], run["seed"])
        m.make_inputs(run["seed"], run["batch"])
        m.evaluate()
        assert m.digests() == run["digests"], (run["model"], run["hidden"], run["batch"], run["seed"])


def _primop(oracle, op, ins, out_shape, fill=0.0):
    arrs = [np.ascontiguousarray(a, np.float32) for a in ins]
    ptrs = (ctypes.POINTER(ctypes.c_float) * max(1, len(arrs)))(*[a.ctypes.data_as(ctypes.POINTER(ctypes.c_float)) for a in arrs])
    rows = (ctypes.c_int * max(1, len(arrs)))(*[a.shape[0] for a in arrs])
    cols = (ctypes.c_int * max(1, len(arrs)))(*[a.shape[1] for a in arrs])
    out = np.zeros(out_shape, np.float32)
    L = oracle.L
    L.orc_exec_primop.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_float]
    rc = L.orc_exec_primop(op, len(arrs), ptrs, rows, cols, out.ctypes.data, out_shape[0], out_shape[1], fill)
    assert rc == 0
    return out


def test_known_answers(oracle):
    # backend_test.cpp:33-57
    out = _primop(oracle, 0, [np.array([[1, 2]]), np.eye(2)], (1, 2))
    assert out.tolist() == [[1.0, 2.0]]
    assert _primop(oracle, 3, [np.zeros((1, 1))], (1, 1))[0, 0] == 0.5
    assert _primop(oracle, 7, [np.array([[0.1, 0.9, 0.3]])], (1, 1))[0, 0] == 1.0
    # ties resolve to the lowest index
    assert _primop(oracle, 7, [np.array([[0.5, 0.9, 0.9]])], (1, 1))[0, 0] == 1.0
    # concat along axis 1 (backend_test.cpp:86-94)
    out = _primop(oracle, 6, [np.array([[1, 2], [3, 4]]), np.array([[9], [8]])], (2, 3))
    assert out.reshape(-1).tolist() == [1, 2, 9, 3, 4, 8]


def test_dense_matches_scalar_reference(oracle):
    rng = np.random.default_rng(7)
    for _ in range(50):  # backend_test.cpp:59-84
        m, k, n = rng.integers(1, 9, size=3)
        a = rng.uniform(-2, 2, (m, k)).astype(np.float32)
        b = rng.uniform(-2, 2, (k, n)).astype(np.float32)
        want = np.zeros((m, n), np.float32)
        for i in range(m):
            for p in range(k):
                want[i] = (want[i] + np.float32(a[i, p]) * b[p]).astype(np.float32)
        got = _primop(oracle, 0, [a, b], (m, n))
        assert np.array_equal(got, want)


def test_schedule_depth_grouping(oracle):
    # runtime_test.cpp:48-66: 4x sigA@0, 2x sigB@0, 2x sigA@1 -> batches 4/2/2
    n = 8
    ids = np.arange(n, dtype=np.int32)
    phase = np.zeros(n, np.int32)
    depth = np.array([0, 0, 0, 0, 0, 0, 1, 1], np.int32)
    sig = np.array([0, 0, 0, 0, 1, 1, 0, 0], np.int32)
    ghost = np.zeros(n, np.int32)
    nsh = np.zeros(n, np.int32)
    refs = np.zeros(1, np.int64)
    batches = np.zeros(5 * n, np.int32)
    order = np.zeros(n, np.int32)
    ops = ctypes.c_long(0)
    L = oracle.L
    p = lambda a: a.ctypes.data
    L.orc_schedule_depth.argtypes = [ctypes.c_int] + [ctypes.c_void_p] * 9 + [ctypes.POINTER(ctypes.c_long)]
    nb = L.orc_schedule_depth(n, p(ids), p(phase), p(depth), p(sig), p(ghost), p(nsh), p(refs), p(batches), p(order),
                              ctypes.byref(ops))
    assert nb == 3
    rows = batches[:15].reshape(3, 5)
    assert rows[:, 4].tolist() == [4, 2, 2]
    assert rows[:, 2].tolist() == [0, 1, 0]
    assert rows[2, 1] == 1
    assert ops.value == 2 * n

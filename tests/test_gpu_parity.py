"""Parity of the B200 path (through the C ABI) with the reference, on a real GPU.

FP32 path: bit-exact.  The plan VM reproduces the reference's accumulation order and glibc's
expf/tanhf, so every output tensor equals the reference's bit for bit and the schedule (which
nodes land in which batch, in what order) equals the reference's exactly — including models whose
control flow depends on tensor values (NestedRNN, DRNN, StackRNN: argmax decisions).
"""
import numpy as np
import pytest

from conftest import MODELS, trace_counters, trace_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu(mbx):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return mbx


def _kw(variant):
    kw = {}
    if variant.startswith("agenda"):
        kw["scheduler"] = "agenda"
    if variant.endswith("explicit"):
        kw["gather"] = "explicit"
    if variant == "no-hoist":
        kw["hoist"] = False
    if variant == "no-phases":
        kw["phases"] = False
    return kw


def _flat_golden(j):
    if j["k"] == "t":
        return list(j["d"])
    return [x for it in j.get("items", []) for x in _flat_golden(it)]


@pytest.mark.parametrize("model", MODELS)
def test_fp32_bitwise_and_schedule(gpu, golden, oracle, model):
    mbx = gpu
    g = golden(model)
    models = {}
    for run in g["runs"]:
        key = (run["hidden"], run["seed"])
        if key not in models:
            c = mbx.Context(0, "fp32")
            m = mbx.Model(c, model, run["hidden"])
            m.make_params(run["seed"])
            models[key] = (c, m)
        m = models[key][1]
        t, d = m.make_inputs(run["seed"], run["batch"])
        r = m.evaluate_batch(t, d, run["batch"], record_nodes="nodes" in run, **_kw(run["variant"]))
        where = (model, run["variant"], run["hidden"], run["batch"], run["seed"])
        assert trace_rows(r.trace) == trace_rows(run["trace"]), where
        assert trace_counters(r.trace) == trace_counters(run["trace"]), where
        assert oracle.digest(r.out_toks, r.out_data, run["batch"]) == run["digests"]["outputs"], where
        if "outputs" in run:
            for i, o in enumerate(run["outputs"]):
                want = np.array(_flat_golden(o), np.float32)
                got = mbx.flatten_floats(r.outputs[i])
                assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), where + (i,)
        # Every batch runs on the device.  Fewer launches than batches: an MV-RNN combine cell and
        # the next matrix add of the same nodes share one launch (kernels_mv.cu), persistent levels
        # runs cover many depths, and a flush's sinks of one exact plan (classifiers of trees of
        # different depths, decision cells) run as one merged launch (runtime.cpp hoist_sinks).
        assert r.trace.device_launches >= 1, where


@pytest.mark.parametrize("idx", range(10))
def test_fp32_baseline_configs(gpu, golden, idx):
    mbx = gpu
    run = golden("baseline")[idx]
    c = mbx.Context(0, "fp32")
    m = mbx.Model(c, run["model"], run["hidden"])
    m.make_params(run["seed"])
    t, d = m.make_inputs(run["seed"], run["batch"])
    r = m.evaluate_batch(t, d, run["batch"], record_nodes=False)
    from conftest import Oracle
    assert trace_rows(r.trace) == trace_rows(run["trace"])
    assert trace_counters(r.trace) == trace_counters(run["trace"])
    assert Oracle().digest(r.out_toks, r.out_data, run["batch"]) == run["digests"]["outputs"]


@pytest.mark.parametrize("model,hidden,batch,seed,prec", [("nestedrnn", 64, 16, 3, "fp32"), ("nestedrnn", 512, 8, 1, "bf16x3"),
                                                        ("drnn", 64, 16, 2, "fp32"), ("stackrnn", 64, 16, 4, "fp32"),
                                                        ("mvrnn", 64, 16, 5, "fp32")])
def test_sink_hoisting_is_bitwise_neutral(gpu, model, hidden, batch, seed, prec):
    """runtime.cpp hoist_sinks: a flush's batches no later batch reads (decision cells, classifiers
    of shallower trees) run after the rest, merged into one launch per plan.  The per-batch timing
    mode keeps the reference's issue order; both orders give bitwise-identical outputs and the same
    trace, and the hoisted order needs fewer launches wherever sinks were interleaved."""
    mbx = gpu
    c = mbx.Context(0, prec)
    m = mbx.Model(c, model, hidden)
    m.make_params(seed)
    t, d = m.make_inputs(seed, batch)
    hoisted = m.evaluate_batch(t, d, batch)
    ordered = m.evaluate_batch(t, d, batch, time_batches=True)
    assert trace_rows(hoisted.trace) == trace_rows(ordered.trace)
    assert trace_counters(hoisted.trace) == trace_counters(ordered.trace)
    for i in range(batch):
        a = mbx.flatten_floats(hoisted.outputs[i])
        b = mbx.flatten_floats(ordered.outputs[i])
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), (model, i)
    if model == "nestedrnn":  # ~10 decision batches per flush become one head + one tail launch
        assert hoisted.trace.device_launches < ordered.trace.device_launches, (
            hoisted.trace.device_launches, ordered.trace.device_launches)


def _relu_bias_dense_plan(h):
    return [0, 2, h, h, 1, h, 1, 1, h, 2,
            0, 0, 1, h, 2, 1, 0, 0, -1, 0, 0, 0, -1, 0,
            2, 1, 1, h, 1, 2, 0, 0, -1, 2, 1, 1, 0, 1, 0, -1, 5, 0, 2, 0, 0, -1,
            1, 2, 1, 0, -1]


def test_exec_batched_equals_primop_fold_bitwise(gpu):
    """backend_test.cpp:134-173: exec_batched == per-instance fold of exec_primop, bitwise,
    b in {1, 2, 8, 64}, both gather modes."""
    mbx = gpu
    rng = np.random.default_rng(11)
    h = 4
    for b in (1, 2, 8, 64):
        ctx = mbx.Context(0, "fp32")
        pid = ctx.register_plan(_relu_bias_dense_plan(h))
        w, _ = ctx.tensor(rng.uniform(-1, 1, (h, h)))
        bias, _ = ctx.tensor(rng.uniform(-1, 1, (1, h)))
        xs = [ctx.tensor(rng.uniform(-1, 1, (1, h)))[0] for _ in range(b)]
        for mode in ("fused", "explicit"):
            outs, _ = ctx.exec_batched(pid, [w, bias], np.array(xs).reshape(b, 1), 1, mode)
            for i in range(b):
                t0, t1, t2 = ctx.alloc(1, h), ctx.alloc(1, h), ctx.alloc(1, h)
                ctx.exec_primop("dense", [(xs[i], (1, h)), (w, (h, h))], (t0, (1, h)))
                ctx.exec_primop("add", [(t0, (1, h)), (bias, (1, h))], (t1, (1, h)))
                ctx.exec_primop("relu", [(t1, (1, h))], (t2, (1, h)))
                a = ctx.download(int(outs[i, 0]), h)
                e = ctx.download(t2, h)
                assert np.array_equal(a.view(np.uint32), e.view(np.uint32))


def test_primops_match_oracle(gpu, oracle):
    """exec_primop on the device vs the CPU restatement on random small shapes
    (backend_test.cpp:59-84), bitwise."""
    import ctypes
    mbx = gpu
    rng = np.random.default_rng(7)
    ctx = mbx.Context(0, "fp32")
    L = oracle.L
    L.orc_exec_primop.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_float]
    for trial in range(50):
        m, k, n = (int(x) for x in rng.integers(1, 9, size=3))
        a = rng.uniform(-2, 2, (m, k)).astype(np.float32)
        bm = rng.uniform(-2, 2, (k, n)).astype(np.float32)
        cases = [("dense", [a, bm], (m, n)), ("tanh", [a], (m, k)), ("relu", [a], (m, k)), ("sigmoid", [a], (m, k)),
                 ("add", [a, a[::-1].copy()], (m, k)), ("mul", [a, a], (m, k)), ("concat", [a, a], (m, 2 * k))]
        for op, ins, oshape in cases:
            offs = [ctx.tensor(x) for x in ins]
            out = ctx.alloc(*oshape)
            ctx.exec_primop(op, offs, (out, oshape))
            got = ctx.download(out, oshape[0] * oshape[1])
            arrs = [np.ascontiguousarray(x) for x in ins]
            ptrs = (ctypes.c_void_p * len(arrs))(*[x.ctypes.data for x in arrs])
            rows = (ctypes.c_int * len(arrs))(*[x.shape[0] for x in arrs])
            cols = (ctypes.c_int * len(arrs))(*[x.shape[1] for x in arrs])
            want = np.zeros(oshape, np.float32)
            L.orc_exec_primop(mbx.OPS.index(op), len(arrs), ptrs, rows, cols, want.ctypes.data, oshape[0], oshape[1], 0.0)
            assert np.array_equal(got.view(np.uint32), want.reshape(-1).view(np.uint32)), (op, m, k, n)


def test_activation_restatements_exhaustive_sample(gpu, oracle):
    """sigmoid / tanh on the device vs glibc on 2^22 float bit patterns spread over the whole
    range (the full 2^32 sweep of the same code runs on the host in test_libm_exact.py)."""
    mbx = gpu
    ctx = mbx.Context(0, "fp32")
    bits = (np.arange(1 << 22, dtype=np.uint64) * 1021 + 7) % (1 << 32)
    x = bits.astype(np.uint32).view(np.float32)
    x = x[np.isfinite(x)].reshape(1, -1)
    n = x.shape[1]
    xo, _ = ctx.tensor(x)
    for op, which in (("sigmoid", 2), ("tanh", 1)):
        out = ctx.alloc(1, n)
        ctx.exec_primop(op, [(xo, (1, n))], (out, (1, n)))
        got = ctx.download(out, n)
        want = np.array([oracle.L.orc_unary(which, float(v)) for v in x[0, :: 997]], np.float32)
        assert np.array_equal(got[::997].view(np.uint32), want.view(np.uint32)), op


def _dense_argmax_plan(k, n, a_shared, outs):
    """[dense(a . W), argmax] with W shared (k x n) and the row a batched or shared (1 x k); `outs`
    lists which step results are plan outputs (0 = the dense row, 1 = the argmax index)."""
    shared = [k, n] + ([1, k] if a_shared else [])
    e = [0, 2 if a_shared else 1] + shared
    e += [0] if a_shared else [1, 1, k]
    a_ref = [0, 1, 0, -1] if a_shared else [1, 0, 0, -1]
    e += [2,
          0, 0, 1, n, 2] + a_ref + [0, 0, 0, -1] + [0,
          0, 7, 1, 1, 1, 2, 0, 0, -1, 0]
    e += [len(outs)]
    for o in outs:
        e += [2, o, 0, -1]
    return e


@pytest.mark.parametrize("k,n,a_shared,outs", [(512, 11, False, [1]), (512, 11, False, [0, 1]),
                                               (256, 32, False, [1, 0]), (512, 11, True, [0, 1]),
                                               (4096, 16, False, [0, 1])])
def test_dense_argmax_registered_plan_bitwise(gpu, k, n, a_shared, outs):
    """Registered [dense, argmax] plans (NestedRNN's decision tail shape; dense_argmax_kernel when
    W and the row fit shared memory, the plan VM otherwise, e.g. K=4096 x N=16) through
    mbx_plan_register + mbx_exec_batched == the fold of exec_primop dense -> argmax, bitwise, for
    the row output, the index output (first maximum; ties seeded in), a shared row and large K."""
    mbx = gpu
    rng = np.random.default_rng(k + n)
    b = 37
    ctx = mbx.Context(0, "fp32")
    pid = ctx.register_plan(_dense_argmax_plan(k, n, a_shared, outs))
    wv = rng.uniform(-0.5, 0.5, (k, n)).astype(np.float32)
    wv[:, 3] = wv[:, 2]  # exact ties between columns 2 and 3: the first index must win
    w, _ = ctx.tensor(wv)
    shared = [w]
    if a_shared:
        a0, _ = ctx.tensor(rng.uniform(-1, 1, (1, k)))
        shared.append(a0)
        rows = [a0] * b
        batched = np.zeros((b, 0), np.int64)
    else:
        rows = [ctx.tensor(rng.uniform(-1, 1, (1, k)))[0] for _ in range(b)]
        batched = np.array(rows, np.int64).reshape(b, 1)
    res, _ = ctx.exec_batched(pid, shared, batched, len(outs))
    for i in range(b):
        t0, t1 = ctx.alloc(1, n), ctx.alloc(1, 1)
        ctx.exec_primop("dense", [(rows[i], (1, k)), (w, (k, n))], (t0, (1, n)))
        ctx.exec_primop("argmax", [(t0, (1, n))], (t1, (1, 1)))
        for j, o in enumerate(outs):
            size = n if o == 0 else 1
            got = ctx.download(int(res[i, j]), size)
            want = ctx.download(t0 if o == 0 else t1, size)
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (i, o)


@pytest.mark.parametrize("h,b", [(32, 37), (128, 64)])
@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("misalign", [False, True])
def test_mv_cell_registered_plan_bitwise(gpu, h, b, fused, misalign):
    """MV-RNN's combine cell (zoo.cpp:124-136) and matrix add (zoo.cpp:135) registered through
    mbx_plan_register and issued through mbx_exec_batched: standalone (mv_cell_kernel alone, the
    add on the pointwise kernel) and inside one flush scope (the add folded into the cell launch),
    16-byte aligned and misaligned matrices, == the fold of exec_primop, bitwise."""
    mbx = gpu
    rng = np.random.default_rng(h * 1000 + b)
    ctx = mbx.Context(0, "fp32")
    model = mbx.Model(ctx, "mvrnn", h)
    sigs = model.signatures()
    cell = ctx.register_plan(model.plan_encoding(sigs.index("tanh_bias_dense_concat")))
    add = ctx.register_plan(model.plan_encoding(sigs.index("add")))
    vw, _ = ctx.tensor(rng.uniform(-0.5, 0.5, (2 * h, h)))
    vb, _ = ctx.tensor(rng.uniform(-0.5, 0.5, (1, h)))
    rows, mats = [], []
    for i in range(b):
        if misalign:
            ctx.alloc(1, 1 + (i % 3))
        lv, _ = ctx.tensor(rng.uniform(-1, 1, (1, h)))
        rm, _ = ctx.tensor(rng.uniform(-0.5, 0.5, (h, h)))
        rv, _ = ctx.tensor(rng.uniform(-1, 1, (1, h)))
        lm, _ = ctx.tensor(rng.uniform(-0.5, 0.5, (h, h)))
        rows.append((lv, rv))
        mats.append((lm, rm))
    cell_b = np.array([[lv, rm, rv, lm] for (lv, rv), (lm, rm) in zip(rows, mats)], np.int64)
    add_b = np.array([[lm, rm] for lm, rm in mats], np.int64)
    n0 = mbx.lib().mbx_kernel_launch_count()
    if fused:
        ctx.flush_begin()
    vout, _ = ctx.exec_batched(cell, [vw, vb], cell_b, 1)
    mout, _ = ctx.exec_batched(add, [], add_b, 1)
    if fused:
        ctx.flush_end()
    ctx.sync()
    # + 1: W (not a session parameter here) is transposed for the cell kernel at every launch
    assert mbx.lib().mbx_kernel_launch_count() - n0 == (1 if fused else 2) + 1
    for i in range(b):
        (lv, rv), (lm, rm) = rows[i], mats[i]
        t0, t1, t2, t3, t4, t5, t6 = (ctx.alloc(1, h), ctx.alloc(1, h), ctx.alloc(1, 2 * h), ctx.alloc(1, h),
                                      ctx.alloc(1, h), ctx.alloc(1, h), ctx.alloc(h, h))
        ctx.exec_primop("dense", [(lv, (1, h)), (rm, (h, h))], (t0, (1, h)))
        ctx.exec_primop("dense", [(rv, (1, h)), (lm, (h, h))], (t1, (1, h)))
        ctx.exec_primop("concat", [(t0, (1, h)), (t1, (1, h))], (t2, (1, 2 * h)))
        ctx.exec_primop("dense", [(t2, (1, 2 * h)), (vw, (2 * h, h))], (t3, (1, h)))
        ctx.exec_primop("add", [(vb, (1, h)), (t3, (1, h))], (t4, (1, h)))
        ctx.exec_primop("tanh", [(t4, (1, h))], (t5, (1, h)))
        ctx.exec_primop("add", [(lm, (h, h)), (rm, (h, h))], (t6, (h, h)))
        got, want = ctx.download(int(vout[i, 0]), h), ctx.download(t5, h)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), ("cell", i)
        got, want = ctx.download(int(mout[i, 0]), h * h), ctx.download(t6, h * h)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), ("add", i)


@pytest.mark.parametrize("misalign", [False, True])
def test_concat_registered_plan_bitwise(gpu, misalign):
    """BiRNN's output concat (zoo.cpp:47-76) registered and issued through mbx_exec_batched runs
    on concat_rows_kernel: == exec_primop concat per node, bitwise, 16-byte aligned or not."""
    mbx = gpu
    rng = np.random.default_rng(5)
    h, b = 96, 45
    ctx = mbx.Context(0, "fp32")
    model = mbx.Model(ctx, "birnn", h)
    pid = ctx.register_plan(model.plan_encoding(model.signatures().index("concat")))
    rows = []
    for i in range(b):
        if misalign:
            ctx.alloc(1, 1 + i % 3)
        rows.append((ctx.tensor(rng.uniform(-1, 1, (1, h)))[0], ctx.tensor(rng.uniform(-1, 1, (1, h)))[0]))
    n0 = mbx.lib().mbx_kernel_launch_count()
    out, _ = ctx.exec_batched(pid, [], np.array(rows, np.int64), 1)
    ctx.sync()
    assert mbx.lib().mbx_kernel_launch_count() - n0 == 1
    for i, (f, bk) in enumerate(rows):
        t = ctx.alloc(1, 2 * h)
        ctx.exec_primop("concat", [(f, (1, h)), (bk, (1, h))], (t, (1, 2 * h)))
        got, want = ctx.download(int(out[i, 0]), 2 * h), ctx.download(t, 2 * h)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), i

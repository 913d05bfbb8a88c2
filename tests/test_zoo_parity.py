"""Host-logic parity (CPU, no GPU): the native library's compiled models and its runtime's
schedules against the reference compiler/executor dumps in tests/golden/.

The runtime runs in dry mode (device = -1): every host step of the B200 path executes — fibers,
inline-depth DFG construction, depth/agenda scheduling, arena allocation in the reference's order,
EXPLICIT-gather accounting — while no kernel is launched.  For models whose control flow does not
depend on tensor values the trace, counters and node table (including every arena offset) must
equal the reference's exactly."""
import numpy as np
import pytest

from conftest import MODELS, STATIC_MODELS, trace_counters, trace_rows


@pytest.fixture(scope="module")
def dry(mbx):
    return mbx.Context(-1)


@pytest.mark.parametrize("model", MODELS)
def test_compiled_artefacts_match_reference(mbx, dry, golden, model):
    g = golden(model)
    m = mbx.Model(dry, model, 32)
    assert m.param_names() == [p["name"] for p in g["params"]]
    assert m.signatures() == [s["name"] for s in g["signatures"]]
    for sig, plan in enumerate(g["plans"]):
        assert m.plan_encoding(sig).tolist() == mbx.plan_from_dump(plan), (model, sig)


@pytest.mark.parametrize("model", MODELS)
def test_inputs_match_reference_generators(mbx, dry, oracle, golden, model):
    g = golden(model)
    m = mbx.Model(dry, model, 32)
    for run in g["runs"]:
        if run["hidden"] != 32:
            continue
        t, d = m.make_inputs(run["seed"], run["batch"])
        nin = len(g["instance_inputs"])
        assert oracle.digest(t, d, run["batch"] * nin) == run["digests"]["inputs"], (model, run["variant"])


def _variant_kwargs(variant):
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


def _node_rows(nodes):
    return [(n.id, n.sig_id, n.block_id, n.instance, n.phase, n.depth, n.ghost, [list(x) for x in n.shared_ins],
             [list(x) for x in n.batched_ins], list(n.producers), [list(x) for x in n.outputs]) for n in nodes]


def _golden_node_rows(nodes):
    return [(n["id"], n["sig"], n["block"], n["inst"], n["phase"], n["depth"], n["ghost"], n["shared"], n["batched"],
             n["producers"], n["outputs"]) for n in nodes]


@pytest.mark.parametrize("model", STATIC_MODELS)
def test_dry_run_traces_match_reference(mbx, dry, golden, model):
    g = golden(model)
    models = {}
    for run in g["runs"]:
        h = run["hidden"]
        if h not in models:  # a fresh context per model: params at offset 0 as in the reference
            c = mbx.Context(-1)
            models[h] = (c, mbx.Model(c, model, h))
        m = models[h][1]
        t, d = m.make_inputs(run["seed"], run["batch"])
        r = m.evaluate_batch(t, d, run["batch"], record_nodes="nodes" in run, decode=False,
                             **_variant_kwargs(run["variant"]))
        assert trace_rows(r.trace) == trace_rows(run["trace"]), (model, run["variant"], run["seed"])
        assert trace_counters(r.trace) == trace_counters(run["trace"]), (model, run["variant"])
        if "nodes" in run:
            assert _node_rows(r.nodes) == _golden_node_rows(run["nodes"]), (model, run["variant"])


@pytest.mark.parametrize("idx", range(10))
def test_dry_run_baseline_traces(mbx, dry, golden, idx):
    run = golden("baseline")[idx]
    if run["model"] not in STATIC_MODELS:
        pytest.skip("tensor-dependent control flow: trace checked on the GPU")
    c = mbx.Context(-1)
    m = mbx.Model(c, run["model"], run["hidden"])
    t, d = m.make_inputs(run["seed"], run["batch"])
    r = m.evaluate_batch(t, d, run["batch"], record_nodes=False, decode=False)
    assert trace_rows(r.trace) == trace_rows(run["trace"])
    assert trace_counters(r.trace) == trace_counters(run["trace"])


def test_gather_bytes_semantics(mbx, dry, golden):
    """EXPLICIT mode counts only non-contiguous batched slots (exec_batched.cpp:46-65)."""
    g = golden("treelstm")
    for run in g["runs"]:
        if run["variant"].endswith("explicit"):
            assert run["trace"]["gather_bytes"] > 0
        elif run["variant"].endswith("fused"):
            assert run["trace"]["gather_bytes"] == 0

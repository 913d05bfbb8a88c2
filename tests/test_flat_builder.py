"""Program::run_flat (coroutine-free DFG construction for control-flow-static models) against the
fiber scheduler path, on the CPU (dry contexts): identical node tables (ids, signatures, blocks,
instances, phases, depths, inputs, producers, arena offsets), traces and counters for every
scheduler / gather / hoist / phase variant, over many seeds and batch sizes.  The reference goldens
pin both paths too (test_zoo_parity.py runs the default, flat path)."""
import os

import pytest

from conftest import trace_counters, trace_rows
from test_zoo_parity import _node_rows

FLAT_MODELS = ["treelstm", "mvrnn", "rnn", "birnn", "fig5"]
VARIANTS = [{}, {"scheduler": "agenda"}, {"gather": "explicit"}, {"hoist": False}, {"phases": False}]


def _run(mbx, model, hidden, seed, batch, flat, kw):
    os.environ["MBX_FLAT_DFG"] = "1" if flat else "0"
    try:
        c = mbx.Context(-1)
        m = mbx.Model(c, model, hidden)
        m.make_params(seed)
        t, d = m.make_inputs(seed, batch)
        r = m.evaluate_batch(t, d, batch, record_nodes=True, decode=False, **kw)
        return _node_rows(r.nodes), trace_rows(r.trace), trace_counters(r.trace)
    finally:
        os.environ.pop("MBX_FLAT_DFG", None)


@pytest.mark.parametrize("model", FLAT_MODELS)
@pytest.mark.parametrize("seed,batch", [(1, 1), (2, 3), (3, 8), (4, 17), (5, 64)])
@pytest.mark.parametrize("vi", range(len(VARIANTS)))
def test_flat_equals_fibers(mbx, model, seed, batch, vi):
    kw = VARIANTS[vi]
    a = _run(mbx, model, 32, seed, batch, True, kw)
    b = _run(mbx, model, 32, seed, batch, False, kw)
    assert a[1] == b[1], (model, seed, batch, kw)
    assert a[2] == b[2], (model, seed, batch, kw)
    assert a[0] == b[0], (model, seed, batch, kw)

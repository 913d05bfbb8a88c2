"""Shared fixtures.  CPU tests (-m "not gpu") cover the oracle against the reference's golden
dumps, the native library's ABI and its host logic (dry-run traces); GPU tests (-m gpu) are the
parity tests proper and go through the C ABI of the native library."""
import ctypes
import gzip
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "liboracle.so")
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "mbatch_ref")
MODELS = ["rnn", "birnn", "treelstm", "mvrnn", "nestedrnn", "drnn", "stackrnn", "fig5"]
# Models whose schedule does not depend on tensor values (dry-run traces must match).
STATIC_MODELS = ["rnn", "birnn", "treelstm", "mvrnn", "fig5"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")


def load_golden(name):
    with gzip.open(os.path.join(GOLDEN, f"{name}.json.gz"), "rt") as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load_golden(name)
        return cache[name]

    return get


def _build_oracle():
    if not os.path.exists(ORACLE_SO):
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"])


class Oracle:
    """ctypes view of oracle/_build/liboracle.so (the CPU restatement; test infrastructure)."""

    def __init__(self):
        _build_oracle()
        L = ctypes.CDLL(ORACLE_SO)
        P, I, I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
        pI32, pF = ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_float)
        L.orc_model_create.restype = P
        L.orc_model_create.argtypes = [ctypes.c_char_p, I, ctypes.c_uint]
        L.orc_model_destroy.argtypes = [P]
        L.orc_make_inputs.argtypes = [P, ctypes.c_uint, I]
        L.orc_set_inputs.argtypes = [P, I, pI32, I64, pF, I64]
        for f in ("orc_inputs_ntok", "orc_inputs_ndata", "orc_outputs_ntok", "orc_outputs_ndata", "orc_last_prim_ops"):
            getattr(L, f).restype = I64
            getattr(L, f).argtypes = [P]
        L.orc_get_inputs.argtypes = [P, pI32, pF]
        L.orc_get_outputs.argtypes = [P, pI32, pF]
        for f in ("orc_params_digest", "orc_inputs_digest", "orc_outputs_digest"):
            getattr(L, f).restype = ctypes.c_uint64
            getattr(L, f).argtypes = [P]
        L.orc_evaluate.argtypes = [P]
        L.orc_digest_encoded.restype = ctypes.c_uint64
        L.orc_digest_encoded.argtypes = [pI32, I64, pF, I64, I]
        L.orc_unary.restype = ctypes.c_float
        L.orc_unary.argtypes = [I, ctypes.c_float]
        L.orc_num_params.argtypes = [P]
        L.orc_param_name.restype = ctypes.c_char_p
        L.orc_param_name.argtypes = [P, I]
        L.orc_param_shape.argtypes = [P, I, ctypes.POINTER(I), ctypes.POINTER(I)]
        L.orc_param_data.restype = pF
        L.orc_param_data.argtypes = [P, I]
        self.L = L

    def model(self, name, hidden, seed):
        h = self.L.orc_model_create(name.encode(), hidden, seed)
        assert h, name
        return OracleModel(self, h)

    def digest(self, toks, data, count):
        t = np.ascontiguousarray(toks, np.int32)
        d = np.ascontiguousarray(data, np.float32)
        return "%016x" % self.L.orc_digest_encoded(t.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), t.size,
                                                   d.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), d.size, count)


class OracleModel:
    def __init__(self, o, h):
        self.o, self.h = o, h

    def __del__(self):
        try:
            self.o.L.orc_model_destroy(self.h)
        except Exception:
            pass

    def make_inputs(self, seed, batch):
        self.o.L.orc_make_inputs(self.h, seed, batch)

    def set_inputs(self, batch, toks, data):
        t = np.ascontiguousarray(toks, np.int32)
        d = np.ascontiguousarray(data, np.float32)
        rc = self.o.L.orc_set_inputs(self.h, batch, t.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), t.size,
                                     d.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), d.size)
        assert rc == 0

    def inputs(self):
        L = self.o.L
        t = np.zeros(L.orc_inputs_ntok(self.h), np.int32)
        d = np.zeros(L.orc_inputs_ndata(self.h), np.float32)
        L.orc_get_inputs(self.h, t.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                         d.ctypes.data_as(ctypes.POINTER(ctypes.c_float)))
        return t, d

    def evaluate(self):
        L = self.o.L
        L.orc_evaluate(self.h)
        t = np.zeros(L.orc_outputs_ntok(self.h), np.int32)
        d = np.zeros(L.orc_outputs_ndata(self.h), np.float32)
        L.orc_get_outputs(self.h, t.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                          d.ctypes.data_as(ctypes.POINTER(ctypes.c_float)))
        return t, d

    def digests(self):
        L = self.o.L
        return {"params": "%016x" % L.orc_params_digest(self.h), "inputs": "%016x" % L.orc_inputs_digest(self.h),
                "outputs": "%016x" % L.orc_outputs_digest(self.h)}

    def params(self):
        L = self.o.L
        out = {}
        for i in range(L.orc_num_params(self.h)):
            r, c = ctypes.c_int(), ctypes.c_int()
            L.orc_param_shape(self.h, i, ctypes.byref(r), ctypes.byref(c))
            p = L.orc_param_data(self.h, i)
            out[L.orc_param_name(self.h, i).decode()] = np.ctypeslib.as_array(p, shape=(r.value * c.value,)).copy().reshape(r.value, c.value)
        return out


@pytest.fixture(scope="session")
def oracle():
    return Oracle()


@pytest.fixture(scope="session")
def mbx():
    from paper_2305_10611_b200 import mbx as m
    m.lib()
    return m


def trace_rows(trace):
    """Comparable view of a trace: (phase, depth, sig, size, ghost, node_ids) per batch."""
    if isinstance(trace, dict):
        return [(b["phase"], b["depth"], b["sig"], b["size"], bool(b["ghost"]), list(b["nodes"])) for b in trace["batches"]]
    return [(b.phase, b.depth, b.sig, b.size, b.ghost, list(b.node_ids)) for b in trace.batches]


def trace_counters(trace):
    if isinstance(trace, dict):
        return {k: trace[k] for k in ("kernel_launches", "total_nodes", "scheduler_ops", "sync_points", "gather_bytes",
                                      "dfg_edges", "flush_boundaries")}
    return {"kernel_launches": trace.kernel_launches, "total_nodes": trace.total_nodes,
            "scheduler_ops": trace.scheduler_ops, "sync_points": trace.sync_points,
            "gather_bytes": trace.gather_bytes, "dfg_edges": trace.dfg_edges,
            "flush_boundaries": list(trace.flush_boundaries)}

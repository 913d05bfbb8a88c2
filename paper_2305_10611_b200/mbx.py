"""ctypes binding of libmbx.so (include/mbx.h) — the host-side mirror of the reference's
`mbatch` runtime API (proj/include/mbatch/runtime.hpp) for Python callers and tests.

Names follow the reference: ``evaluate_batch`` returns an ``EvalResult`` with ``outputs`` (host
values), ``trace`` (a ``ScheduleTrace``: batches, counters, flush boundaries) and ``nodes`` (the
DFG node table).  Errors raise ``MbatchError`` carrying the reference's message text.

There is no fallback: if the native library is missing or the CUDA device cannot be opened the
calls raise — the product path is the sm_100a library or nothing.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Any, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MBX_LIB") or os.path.join(_HERE, "lib", "libmbx.so")  # MBX_LIB: A/B builds (tools/)

PREC = {"fp32": 0, "bf16x3": 1, "bf16": 2, "bf16x6": 3}
OPS = ["dense", "add", "mul", "sigmoid", "tanh", "relu", "concat", "argmax", "fill"]


class MbatchError(RuntimeError):
    """mbatch::Error raised across the C ABI (same message text as the reference)."""


class _Opts(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("scheduler", "gather", "hoist", "phases", "record_nodes", "time_kernels", "time_batches",
                 "inputs_resident", "outputs_on_device", "ghost", "defer_sync")]


class BerxitConfig(ctypes.Structure):
    """mbx_berxit_config (include/mbx_berxit.h)."""
    _fields_ = [("hidden", ctypes.c_int32), ("heads", ctypes.c_int32), ("ffn", ctypes.c_int32),
                ("layers", ctypes.c_int32), ("seq", ctypes.c_int32), ("classes", ctypes.c_int32),
                ("exit_threshold", ctypes.c_float), ("ln_eps", ctypes.c_float)]


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise MbatchError(f"native library not built: {LIB_PATH} (run __graft_entry__.build())")
    L = ctypes.CDLL(LIB_PATH)
    P, I, I64, F = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_float
    pI32, pI64, pF, pD = (ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64),
                          ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_double))
    sig = {
        "mbx_version": (ctypes.c_char_p, []),
        "mbx_kernel_launch_count": (I64, []),
        "mbx_ctx_create": (I, [I, I, ctypes.POINTER(P)]),
        "mbx_ctx_destroy": (None, [P]),
        "mbx_last_error": (ctypes.c_char_p, [P]),
        "mbx_ctx_set_precision": (I, [P, I]),
        "mbx_sync": (I, [P]),
        "mbx_arena_alloc": (I, [P, I, I, pI64]),
        "mbx_arena_used": (I64, [P]),
        "mbx_arena_upload": (I, [P, I64, pF, I64]),
        "mbx_arena_download": (I, [P, I64, pF, I64]),
        "mbx_arena_rewind": (I, [P, I64]),
        "mbx_arena_device_ptr": (I, [P, I64, I64, ctypes.POINTER(pF)]),
        "mbx_flush_begin": (I, [P]),
        "mbx_flush_end": (I, [P]),
        "mbx_read_ints": (I, [P, pI64, I, pI64]),
        "mbx_plan_register": (I, [P, pI32, I64, ctypes.POINTER(I)]),
        "mbx_exec_batched": (I, [P, I, I, pI64, pI64, I, pI64, pI64]),
        "mbx_exec_primop": (I, [P, I, I, pI64, ctypes.POINTER(I), ctypes.POINTER(I), I64, I, I, F]),
        "mbx_model_create": (I, [P, ctypes.c_char_p, I, ctypes.POINTER(P)]),
        "mbx_model_destroy": (None, [P]),
        "mbx_model_make_params": (I, [P, ctypes.c_uint]),
        "mbx_model_set_param": (I, [P, ctypes.c_char_p, pF, I64]),
        "mbx_model_num_params": (I, [P]),
        "mbx_model_param_name": (ctypes.c_char_p, [P, I]),
        "mbx_model_make_inputs": (I, [P, ctypes.c_uint, I, pI32, pI64, pF, pI64]),
        "mbx_model_num_sigs": (I, [P]),
        "mbx_model_sig_name": (ctypes.c_char_p, [P, I]),
        "mbx_model_plan_encoding": (I, [P, I, pI32, pI64]),
        "mbx_options_default": (None, [ctypes.POINTER(_Opts)]),
        "mbx_evaluate_batch": (I, [P, I, pI32, I64, pF, I64, ctypes.POINTER(_Opts), ctypes.POINTER(P)]),
        "mbx_reference_evaluate": (I, [P, I, pI32, I64, pF, I64, ctypes.POINTER(P)]),
        "mbx_profile_invocations": (I, [P, I, pI32, I64, pF, I64, pI64, pI32, pI32, ctypes.POINTER(I)]),
        "mbx_result_destroy": (None, [P]),
        "mbx_result_outputs": (I, [P, pI32, pI64, pF, pI64]),
        "mbx_result_counters": (I, [P, pI64]),
        "mbx_result_batches": (I, [P, pI32, pI32]),
        "mbx_result_flush_boundaries": (I, [P, pI32]),
        "mbx_result_nodes": (I, [P, pI32, pI64, pI64]),
        "mbx_result_timing": (I, [P, pD]),
        "mbx_result_batch_times": (I, [P, pD]),
        "mbx_result_host_breakdown": (I, [P, pD]),
        "mbx_ctx_stream": (P, [P]),
        "mbx_pool_create": (I, [I, I, ctypes.c_char_p, I, ctypes.c_uint, I, ctypes.POINTER(P)]),
        "mbx_pool_destroy": (None, [P]),
        "mbx_pool_last_error": (ctypes.c_char_p, [P]),
        "mbx_pool_set_error": (None, [ctypes.c_char_p]),
        "mbx_pool_threads": (I, [P]),
        "mbx_pool_stream": (P, [P]),
        "mbx_pool_model": (P, [P, I]),
        "mbx_pool_run": (I, [P, I, I, ctypes.POINTER(pI32), pI64, ctypes.POINTER(pF), pI64, ctypes.POINTER(_Opts),
                             pI64]),
        "mbx_pool_run_timed": (I, [P, I, I, ctypes.POINTER(pI32), pI64, ctypes.POINTER(pF), pI64,
                                   ctypes.POINTER(_Opts), pI64, pD]),
        "mbx_berxit_config_default": (None, [ctypes.POINTER(BerxitConfig)]),
        "mbx_berxit_param_count": (I64, [ctypes.POINTER(BerxitConfig)]),
        "mbx_berxit_make_params": (I, [ctypes.POINTER(BerxitConfig), ctypes.c_uint, pF]),
        "mbx_berxit_make_input": (I, [ctypes.POINTER(BerxitConfig), ctypes.c_uint, I, pF]),
        "mbx_berxit_create": (I, [I, I, ctypes.POINTER(BerxitConfig), I, ctypes.POINTER(P)]),
        "mbx_berxit_destroy": (None, [P]),
        "mbx_berxit_last_error": (ctypes.c_char_p, [P]),
        "mbx_berxit_set_params": (I, [P, pF, I64]),
        "mbx_berxit_run": (I, [P, I, pF, pF, pI32, pI32]),
        "mbx_berxit_run_device": (I, [P, I, P]),
        "mbx_berxit_read": (I, [P, I, pF, pI32, pI32]),
        "mbx_berxit_stream": (P, [P]),
        "mbx_berxit_launches_per_batch": (I, [P, I]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def exported_symbols() -> List[str]:
    """mbx_* functions declared in include/mbx.h (for ABI checks), parsed from the header."""
    import re
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    hdr = "".join(open(os.path.join(inc, h)).read() for h in ("mbx.h", "mbx_berxit.h"))
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(mbx_[a-z0-9_]+)\s*\(", hdr)))


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


# ---- host values ---------------------------------------------------------------------------

@dataclass
class Adt:
    ctor: str
    fields: list


def decode_hostvals(toks: np.ndarray, data: np.ndarray, count: int) -> list:
    """Decodes `count` values of the hostval encoding (see include/mbx.h)."""
    ti, di = 0, 0

    def one():
        nonlocal ti, di
        k = int(toks[ti]); ti += 1
        if k == 0:
            r, c = int(toks[ti]), int(toks[ti + 1]); ti += 2
            v = np.array(data[di:di + r * c], dtype=np.float32).reshape(r, c); di += r * c
            return v
        if k == 1:
            v = int(toks[ti]); ti += 1
            return v
        if k in (5, 6):  # float64 / int64 scalar: two tokens, low word first
            bits = np.array([toks[ti], toks[ti + 1]], np.int32).view(np.uint32)
            ti += 2
            raw = np.array([int(bits[0]) | (int(bits[1]) << 32)], np.uint64)
            return float(raw.view(np.float64)[0]) if k == 5 else int(raw.view(np.int64)[0])
        ctor = None
        if k == 4:
            cid = int(toks[ti]); ti += 1
            if cid >= 0:
                ctor = "Node" if cid else "Leaf"
            else:  # named constructor: length, one token per byte
                n = int(toks[ti]); ti += 1
                ctor = bytes(int(x) for x in toks[ti:ti + n]).decode(); ti += n
        n = int(toks[ti]); ti += 1
        items = [one() for _ in range(n)]
        if k == 2:
            return items
        if k == 3:
            return tuple(items)
        return Adt(ctor, items)

    out = [one() for _ in range(count)]
    assert ti == len(toks) and di == len(data), "trailing hostval data"
    return out


def instance_spans(toks: np.ndarray, batch: int) -> List[Tuple[int, int, int, int]]:
    """Per instance of a `batch`-instance hostval encoding: (tok_begin, tok_end, data_begin,
    data_end).  Instances are encoded one after another (each: its @main instance inputs)."""
    ends = []
    ti, di = 0, 0

    def skip():
        nonlocal ti, di
        k = int(toks[ti]); ti += 1
        if k == 0:
            di += int(toks[ti]) * int(toks[ti + 1]); ti += 2
        elif k == 1:
            ti += 1
        elif k in (5, 6):
            ti += 2
        else:
            if k == 4:
                cid = int(toks[ti]); ti += 1
                if cid < 0:
                    ti += 1 + int(toks[ti])
            n = int(toks[ti]); ti += 1
            for _ in range(n):
                skip()

    while ti < len(toks):
        skip()
        ends.append((ti, di))
    assert len(ends) % batch == 0, "encoding does not hold `batch` instances"
    per = len(ends) // batch
    spans, t0, d0 = [], 0, 0
    for i in range(batch):
        t1, d1 = ends[(i + 1) * per - 1]
        spans.append((t0, t1, d0, d1))
        t0, d0 = t1, d1
    return spans


def shard_instances(toks: np.ndarray, data: np.ndarray, batch: int, rank: int, world: int):
    """Contiguous instance shard of a mini-batch for multi-GPU execution: rank r of
    `world` gets instances [lo, hi) with lo = r*batch//world.  Returns (toks, data, lo, hi).
    Instances never exchange tensors, so each shard runs on its own GPU with no collective."""
    lo, hi = rank * batch // world, (rank + 1) * batch // world
    sp = instance_spans(toks, batch)
    if hi <= lo:
        return np.zeros(0, np.int32), np.zeros(0, np.float32), lo, hi
    return (np.ascontiguousarray(toks[sp[lo][0]:sp[hi - 1][1]]), np.ascontiguousarray(data[sp[lo][2]:sp[hi - 1][3]]),
            lo, hi)


def flatten_floats(v) -> np.ndarray:
    """All tensor data of a host value, depth-first (the digest order of the oracle)."""
    parts = []

    def go(x):
        if isinstance(x, np.ndarray):
            parts.append(x.reshape(-1))
        elif isinstance(x, (list, tuple)):
            for y in x:
                go(y)
        elif isinstance(x, Adt):
            for y in x.fields:
                go(y)

    go(v)
    return np.concatenate(parts).astype(np.float32) if parts else np.zeros(0, np.float32)


# ---- results -------------------------------------------------------------------------------

@dataclass
class BatchRecord:
    phase: int
    depth: int
    sig: int
    size: int
    ghost: bool
    node_ids: List[int]


@dataclass
class ScheduleTrace:
    batches: List[BatchRecord]
    kernel_launches: int
    total_nodes: int
    scheduler_ops: int
    sync_points: int
    gather_bytes: int
    dfg_edges: int
    flush_boundaries: List[int]
    device_launches: int = 0


@dataclass
class DFGNode:
    id: int
    sig_id: int
    block_id: int
    instance: int
    phase: int
    depth: int
    ghost: bool
    shared_ins: List[Tuple[int, int, int]]
    batched_ins: List[Tuple[int, int, int]]
    producers: List[int]
    outputs: List[Tuple[int, int, int]]


@dataclass
class Timing:
    host_total_us: float
    host_dfg_us: float
    device_span_us: float
    h2d_bytes: int
    d2h_bytes: int
    batch_us: List[float] = field(default_factory=list)
    host_breakdown: dict = field(default_factory=dict)  # fibers / sched / prepare / issue (us)


@dataclass
class EvalResult:
    outputs: list
    trace: ScheduleTrace
    nodes: List[DFGNode] = field(default_factory=list)
    timing: Optional[Timing] = None
    out_toks: Optional[np.ndarray] = None
    out_data: Optional[np.ndarray] = None


# ---- context / model -----------------------------------------------------------------------

class Context:
    """One device + stream + HBM arena (device < 0: host-only dry run, no CUDA)."""

    def __init__(self, device: int = 0, precision: str = "fp32"):
        L = lib()
        h = ctypes.c_void_p()
        if L.mbx_ctx_create(device, PREC[precision], ctypes.byref(h)) != 0:
            raise MbatchError(L.mbx_last_error(None).decode())
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            lib().mbx_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc: int):
        if rc != 0:
            raise MbatchError(lib().mbx_last_error(self.h).decode())

    def set_precision(self, precision: str):
        self.check(lib().mbx_ctx_set_precision(self.h, PREC[precision]))

    def sync(self):
        self.check(lib().mbx_sync(self.h))

    # arena
    def alloc(self, rows: int, cols: int) -> int:
        off = ctypes.c_int64()
        self.check(lib().mbx_arena_alloc(self.h, rows, cols, ctypes.byref(off)))
        return off.value

    def used(self) -> int:
        return lib().mbx_arena_used(self.h)

    def upload(self, offset: int, arr: np.ndarray):
        a = np.ascontiguousarray(arr, dtype=np.float32).reshape(-1)
        self.check(lib().mbx_arena_upload(self.h, offset, _ptr(a, ctypes.c_float), a.size))

    def download(self, offset: int, n: int) -> np.ndarray:
        a = np.empty(n, np.float32)
        self.check(lib().mbx_arena_download(self.h, offset, _ptr(a, ctypes.c_float), n))
        return a

    def tensor(self, arr: np.ndarray) -> Tuple[int, Tuple[int, int]]:
        arr = np.asarray(arr, np.float32)
        if arr.ndim == 1:
            arr = arr.reshape(1, -1)
        off = self.alloc(*arr.shape)
        self.upload(off, arr)
        return off, arr.shape

    # plans / batched execution (backend::exec_batched)
    def register_plan(self, enc: Sequence[int]) -> int:
        e = np.asarray(enc, np.int32)
        pid = ctypes.c_int()
        self.check(lib().mbx_plan_register(self.h, _ptr(e, ctypes.c_int32), e.size, ctypes.byref(pid)))
        return pid.value

    def flush_begin(self):
        """Opens a flush scope (mbx_flush_begin): exec_batched calls queue until flush_end."""
        self.check(lib().mbx_flush_begin(self.h))

    def flush_end(self):
        self.check(lib().mbx_flush_end(self.h))

    def read_ints(self, offsets: Sequence[int]) -> List[int]:
        """(long) arena[off] for every offset, one device round trip (mbx_read_ints)."""
        o = np.ascontiguousarray(offsets, np.int64)
        out = np.zeros(max(1, o.size), np.int64)
        self.check(lib().mbx_read_ints(self.h, _ptr(o, ctypes.c_int64), o.size, _ptr(out, ctypes.c_int64)))
        return [int(x) for x in out[:o.size]]

    def stream(self) -> int:
        """cudaStream_t of the context (e.g. for torch.cuda.ExternalStream)."""
        return lib().mbx_ctx_stream(self.h) or 0

    def exec_batched(self, plan_id: int, shared, batched: np.ndarray, nout: int,
                     gather: str = "fused") -> Tuple[np.ndarray, int]:
        """backend::exec_batched.  `shared` is either one row of shared offsets (broadcast to every
        instance) or a (b, nshared) array of per-instance shared offsets."""
        b = batched.shape[0]
        s = np.asarray(shared, np.int64)
        if s.ndim == 1:
            s = np.tile(s, (b, 1))
        s = np.ascontiguousarray(s)
        bt = np.ascontiguousarray(batched, np.int64)
        out = np.zeros(b * nout, np.int64)
        gb = ctypes.c_int64()
        self.check(lib().mbx_exec_batched(self.h, plan_id, b, _ptr(s, ctypes.c_int64), _ptr(bt, ctypes.c_int64),
                                          1 if gather == "explicit" else 0, _ptr(out, ctypes.c_int64),
                                          ctypes.byref(gb)))
        return out.reshape(b, nout), gb.value

    def exec_primop(self, op: str, ins: Sequence[Tuple[int, Tuple[int, int]]], out: Tuple[int, Tuple[int, int]],
                    fill: float = 0.0):
        offs = np.array([o for o, _ in ins], np.int64)
        rows = (ctypes.c_int * max(1, len(ins)))(*[s[0] for _, s in ins])
        cols = (ctypes.c_int * max(1, len(ins)))(*[s[1] for _, s in ins])
        self.check(lib().mbx_exec_primop(self.h, OPS.index(op), len(ins), _ptr(offs, ctypes.c_int64), rows, cols,
                                         out[0], out[1][0], out[1][1], fill))


class Model:
    """A zoo model compiled for the device (zoo::get_model) with resident parameters."""

    def __init__(self, ctx: Context, name: str, hidden: int):
        self.ctx = ctx
        self.name = name
        self.hidden = hidden
        h = ctypes.c_void_p()
        ctx.check(lib().mbx_model_create(ctx.h, name.encode(), hidden, ctypes.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().mbx_model_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def make_params(self, seed: int):
        self.ctx.check(lib().mbx_model_make_params(self.h, seed))

    def set_param(self, name: str, arr: np.ndarray):
        a = np.ascontiguousarray(arr, np.float32).reshape(-1)
        self.ctx.check(lib().mbx_model_set_param(self.h, name.encode(), _ptr(a, ctypes.c_float), a.size))

    def param_names(self) -> List[str]:
        return [lib().mbx_model_param_name(self.h, i).decode() for i in range(lib().mbx_model_num_params(self.h))]

    def make_inputs(self, seed: int, batch: int) -> Tuple[np.ndarray, np.ndarray]:
        nt, nd = ctypes.c_int64(), ctypes.c_int64()
        self.ctx.check(lib().mbx_model_make_inputs(self.h, seed, batch, None, ctypes.byref(nt), None, ctypes.byref(nd)))
        t = np.zeros(nt.value, np.int32)
        d = np.zeros(nd.value, np.float32)
        self.ctx.check(lib().mbx_model_make_inputs(self.h, seed, batch, _ptr(t, ctypes.c_int32), ctypes.byref(nt),
                                                   _ptr(d, ctypes.c_float), ctypes.byref(nd)))
        return t, d

    def signatures(self) -> List[str]:
        return [lib().mbx_model_sig_name(self.h, i).decode() for i in range(lib().mbx_model_num_sigs(self.h))]

    def plan_encoding(self, sig: int) -> np.ndarray:
        n = ctypes.c_int64()
        self.ctx.check(lib().mbx_model_plan_encoding(self.h, sig, None, ctypes.byref(n)))
        e = np.zeros(n.value, np.int32)
        self.ctx.check(lib().mbx_model_plan_encoding(self.h, sig, _ptr(e, ctypes.c_int32), ctypes.byref(n)))
        return e

    def evaluate_batch(self, toks: np.ndarray, data: np.ndarray, batch: int, scheduler: str = "depth",
                       gather: str = "fused", hoist: bool = True, phases: bool = True, record_nodes: bool = True,
                       time_kernels: bool = False, time_batches: bool = False, inputs_resident: bool = False,
                       outputs_on_device: bool = False, ghost: bool = True, decode: bool = True,
                       trace: bool = True, defer_sync: bool = False) -> EvalResult:
        L = lib()
        o = make_options(scheduler, gather, hoist, phases, record_nodes, time_kernels, time_batches, inputs_resident,
                         outputs_on_device, ghost, defer_sync)
        t = np.ascontiguousarray(toks, np.int32)
        d = np.ascontiguousarray(data, np.float32)
        r = ctypes.c_void_p()
        self.ctx.check(L.mbx_evaluate_batch(self.h, batch, _ptr(t, ctypes.c_int32), t.size, _ptr(d, ctypes.c_float),
                                            d.size, ctypes.byref(o), ctypes.byref(r)))
        try:
            return _read_result(r, batch, record_nodes, decode, trace)
        finally:
            L.mbx_result_destroy(r)


    def reference_evaluate(self, toks: np.ndarray, data: np.ndarray, batch: int) -> list:
        """runtime::reference_evaluate: every instance on its own (no cross-instance batching);
        decoded outputs, one per instance."""
        L = lib()
        t = np.ascontiguousarray(toks, np.int32)
        d = np.ascontiguousarray(data, np.float32)
        r = ctypes.c_void_p()
        self.ctx.check(L.mbx_reference_evaluate(self.h, batch, _ptr(t, ctypes.c_int32), t.size,
                                                _ptr(d, ctypes.c_float), d.size, ctypes.byref(r)))
        try:
            nt, nd = ctypes.c_int64(), ctypes.c_int64()
            L.mbx_result_outputs(r, None, ctypes.byref(nt), None, ctypes.byref(nd))
            ot, od = np.zeros(nt.value, np.int32), np.zeros(nd.value, np.float32)
            L.mbx_result_outputs(r, _ptr(ot, ctypes.c_int32), ctypes.byref(nt), _ptr(od, ctypes.c_float), ctypes.byref(nd))
            return decode_hostvals(ot, od, batch)
        finally:
            L.mbx_result_destroy(r)

    def profile_invocations(self, toks: np.ndarray, data: np.ndarray, batch: int) -> dict:
        """runtime::profile_invocations: {"counts": {sig: n}, "static_estimate": {sig: level},
        "ranking": [sig, ...]} over one evaluation of the inputs."""
        L = lib()
        t = np.ascontiguousarray(toks, np.int32)
        d = np.ascontiguousarray(data, np.float32)
        ns = L.mbx_model_num_sigs(self.h)
        counts, levels, ranking = np.zeros(ns, np.int64), np.zeros(ns, np.int32), np.zeros(ns, np.int32)
        nr = ctypes.c_int()
        self.ctx.check(L.mbx_profile_invocations(self.h, batch, _ptr(t, ctypes.c_int32), t.size, _ptr(d, ctypes.c_float),
                                                 d.size, _ptr(counts, ctypes.c_int64), _ptr(levels, ctypes.c_int32),
                                                 _ptr(ranking, ctypes.c_int32), ctypes.byref(nr)))
        return {"counts": {k: int(counts[k]) for k in range(ns) if counts[k]},
                "static_estimate": {k: int(levels[k]) for k in range(ns) if levels[k] >= 0},
                "ranking": [int(x) for x in ranking[:nr.value]]}


def make_options(scheduler: str = "depth", gather: str = "fused", hoist: bool = True, phases: bool = True,
                 record_nodes: bool = False, time_kernels: bool = False, time_batches: bool = False,
                 inputs_resident: bool = False, outputs_on_device: bool = False, ghost: bool = True,
                 defer_sync: bool = False) -> _Opts:
    o = _Opts()
    lib().mbx_options_default(ctypes.byref(o))
    o.scheduler = 1 if scheduler == "agenda" else 0
    o.gather = 1 if gather == "explicit" else 0
    o.hoist, o.phases, o.ghost = int(hoist), int(phases), int(ghost)
    o.record_nodes, o.time_kernels, o.time_batches = int(record_nodes), int(time_kernels), int(time_batches)
    o.inputs_resident, o.outputs_on_device = int(inputs_resident), int(outputs_on_device)
    o.defer_sync = int(defer_sync)
    return o


class Pool:
    """Throughput mode (mbx_pool_*): `threads` worker contexts on one device, each with its own
    stream; ``run`` evaluates many independent mini-batches, mini-batch i on worker i % threads,
    host and device work overlapping across workers (launches needing co-resident CTAs chained
    through the per-device persistent lane)."""

    def __init__(self, device: int, precision: str, model: str, hidden: int, param_seed: int, threads: int):
        self.h = ctypes.c_void_p()
        if lib().mbx_pool_create(device, PREC[precision], model.encode(), hidden, param_seed, threads,
                                 ctypes.byref(self.h)):
            raise MbatchError(lib().mbx_last_error(None).decode())
        self.threads = threads

    def close(self):
        if self.h:
            lib().mbx_pool_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stream(self) -> int:
        return lib().mbx_pool_stream(self.h) or 0

    def evaluate_on_worker(self, worker: int, toks: np.ndarray, data: np.ndarray, batch: int,
                           **opts) -> EvalResult:
        """One mini-batch through worker `worker`'s own context and model (the code path every
        pool run takes), synchronously, with decoded outputs and the full trace: the bench's
        checked mini-batch."""
        L = lib()
        m = L.mbx_pool_model(self.h, worker)
        if not m:
            raise MbatchError(f"pool has no worker {worker}")
        o = make_options(**opts)
        t = np.ascontiguousarray(toks, np.int32)
        d = np.ascontiguousarray(data, np.float32)
        r = ctypes.c_void_p()
        if L.mbx_evaluate_batch(m, batch, _ptr(t, ctypes.c_int32), t.size, _ptr(d, ctypes.c_float), d.size,
                                ctypes.byref(o), ctypes.byref(r)):
            raise MbatchError(L.mbx_last_error(None).decode())
        try:
            return _read_result(r, batch, False, True, True)
        finally:
            L.mbx_result_destroy(r)

    def run(self, inputs: Sequence[Tuple[np.ndarray, np.ndarray]], batch: int, **opts) -> int:
        """Evaluates every (toks, data) mini-batch; returns the total DFG node count."""
        return self.run_timed(inputs, batch, **opts)[0]

    def run_timed(self, inputs: Sequence[Tuple[np.ndarray, np.ndarray]], batch: int, **opts) -> Tuple[int, float]:
        """Like run; also returns the device time of the run in ms (CUDA events on the worker
        streams: first start to last end)."""
        L = lib()
        n = len(inputs)
        ts = [np.ascontiguousarray(t, np.int32) for t, _ in inputs]
        ds = [np.ascontiguousarray(d, np.float32) for _, d in inputs]
        tp = (ctypes.POINTER(ctypes.c_int32) * n)(*[_ptr(t, ctypes.c_int32) for t in ts])
        dp = (ctypes.POINTER(ctypes.c_float) * n)(*[_ptr(d, ctypes.c_float) for d in ds])
        nt = (ctypes.c_int64 * n)(*[t.size for t in ts])
        nd = (ctypes.c_int64 * n)(*[d.size for d in ds])
        o = make_options(**opts)
        total = ctypes.c_int64(0)
        ms = ctypes.c_double(0.0)
        if L.mbx_pool_run_timed(self.h, n, batch, tp, nt, dp, nd, ctypes.byref(o), ctypes.byref(total), ctypes.byref(ms)):
            raise MbatchError(L.mbx_pool_last_error(self.h).decode())
        return int(total.value), float(ms.value)


def _read_result(r, batch: int, record_nodes: bool, decode: bool, want_trace: bool = True) -> EvalResult:
    L = lib()
    nt, nd = ctypes.c_int64(), ctypes.c_int64()
    L.mbx_result_outputs(r, None, ctypes.byref(nt), None, ctypes.byref(nd))
    ot = np.zeros(nt.value, np.int32)
    od = np.zeros(nd.value, np.float32)
    L.mbx_result_outputs(r, _ptr(ot, ctypes.c_int32), ctypes.byref(nt), _ptr(od, ctypes.c_float), ctypes.byref(nd))
    c = np.zeros(9, np.int64)
    L.mbx_result_counters(r, _ptr(c, ctypes.c_int64))
    nb = int(c[6]) if want_trace else 0
    rows = np.zeros(5 * max(1, nb), np.int32)
    total_ids = 0
    ids = np.zeros(max(1, int(c[1])), np.int32)
    if want_trace:
        L.mbx_result_batches(r, _ptr(rows, ctypes.c_int32), _ptr(ids, ctypes.c_int32))
    batches, k = [], 0
    for b in range(nb):
        ph, dp, sg, sz, gh = (int(x) for x in rows[5 * b:5 * b + 5])
        batches.append(BatchRecord(ph, dp, sg, sz, bool(gh), [int(x) for x in ids[k:k + sz]]))
        k += sz
        total_ids += sz
    fb = np.zeros(max(1, int(c[7])), np.int32)
    L.mbx_result_flush_boundaries(r, _ptr(fb, ctypes.c_int32))
    trace = ScheduleTrace(batches, int(c[0]), int(c[1]), int(c[2]), int(c[3]), int(c[4]), int(c[5]),
                          [int(x) for x in fb[:int(c[7])]], int(c[8]))
    nodes = []
    if record_nodes and c[1] > 0:
        nr = ctypes.c_int64()
        L.mbx_result_nodes(r, None, None, ctypes.byref(nr))
        hdr = np.zeros(11 * int(c[1]), np.int32)
        refs = np.zeros(max(1, nr.value), np.int64)
        L.mbx_result_nodes(r, _ptr(hdr, ctypes.c_int32), _ptr(refs, ctypes.c_int64), ctypes.byref(nr))
        k = 0
        for i in range(int(c[1])):
            h = [int(x) for x in hdr[11 * i:11 * i + 11]]
            ns, nbt, npr, no = h[7], h[8], h[9], h[10]
            sh = [tuple(int(x) for x in refs[k + 3 * j:k + 3 * j + 3]) for j in range(ns)]; k += 3 * ns
            bt = [tuple(int(x) for x in refs[k + 3 * j:k + 3 * j + 3]) for j in range(nbt)]; k += 3 * nbt
            pr = [int(x) for x in refs[k:k + npr]]; k += npr
            ou = [tuple(int(x) for x in refs[k + 3 * j:k + 3 * j + 3]) for j in range(no)]; k += 3 * no
            nodes.append(DFGNode(h[0], h[1], h[2], h[3], h[4], h[5], bool(h[6]), sh, bt, pr, ou))
    tm = np.zeros(5, np.float64)
    L.mbx_result_timing(r, _ptr(tm, ctypes.c_double))
    bt = np.zeros(max(1, int(c[6])), np.float64)
    nbt = L.mbx_result_batch_times(r, _ptr(bt, ctypes.c_double))
    hb = np.zeros(4, np.float64)
    L.mbx_result_host_breakdown(r, _ptr(hb, ctypes.c_double))
    timing = Timing(float(tm[0]), float(tm[1]), float(tm[2]), int(tm[3]), int(tm[4]), bt[:nbt].tolist(),
                    dict(zip(("fibers", "sched", "prepare", "issue"), hb.tolist())))
    outputs = decode_hostvals(ot, od, batch) if decode else []
    return EvalResult(outputs, trace, nodes, timing, ot, od)


# ---- plan encodings ------------------------------------------------------------------------

def plan_from_dump(p: dict) -> List[int]:
    """mbx_plan_register encoding of a plan as dumped by oracle/ref_harness.cpp."""
    kind = {"S": 0, "B": 1, "T": 2}
    stepk = {"op": 0, "fused_dense": 1, "chain": 2}
    e = [1 if p["ghost"] else 0, len(p["shared_shapes"])]
    for r, c in p["shared_shapes"]:
        e += [r, c]
    e.append(len(p["batched_shapes"]))
    for r, c in p["batched_shapes"]:
        e += [r, c]
    e.append(len(p["steps"]))
    for st in p["steps"]:
        e += [stepk[st["kind"]], OPS.index(st["op"]), st["out"][0], st["out"][1], len(st["ins"])]
        for k, i, off, cols in st["ins"]:
            e += [kind[k], i, off, cols]
        e.append(len(st["chain"]))
        for l in st["chain"]:
            e += [OPS.index(l["op"]), 1 if l["rhs"] is not None else 0]
            e += ([kind[l["rhs"][0]], *l["rhs"][1:]] if l["rhs"] is not None else [2, 0, 0, -1])
    e.append(len(p["outputs"]))
    for k, i, off, cols in p["outputs"]:
        e += [kind[k], i, off, cols]
    return e


def berxit_config(**kw) -> BerxitConfig:
    """mbx_berxit_config_default (BERT-base: H 768, 12 heads, FFN 3072, 12 shared layers, seq 128,
    8 classes, exit threshold 0.6) with the given fields replaced."""
    c = BerxitConfig()
    lib().mbx_berxit_config_default(ctypes.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def berxit_make_params(cfg: BerxitConfig, seed: int) -> np.ndarray:
    n = lib().mbx_berxit_param_count(ctypes.byref(cfg))
    out = np.empty(n, np.float32)
    if lib().mbx_berxit_make_params(ctypes.byref(cfg), seed, _ptr(out, ctypes.c_float)):
        raise MbatchError(lib().mbx_berxit_last_error(None).decode())
    return out


def berxit_make_inputs(cfg: BerxitConfig, seed: int, batch: int, first: int = 0) -> np.ndarray:
    """Instances first .. first + batch - 1 of the synthetic input set, [batch][seq][hidden]."""
    out = np.empty((batch, cfg.seq, cfg.hidden), np.float32)
    for i in range(batch):
        if lib().mbx_berxit_make_input(ctypes.byref(cfg), seed, first + i, _ptr(out[i], ctypes.c_float)):
            raise MbatchError(lib().mbx_berxit_last_error(None).decode())
    return out


@dataclass
class BerxitResult:
    logits: np.ndarray       # [batch][classes]
    exit_layer: np.ndarray   # [batch]
    schedule: np.ndarray     # [layers][batch]: instance ids of layer l's batch, -1 padded

    def batches(self) -> List[List[int]]:
        return [[int(i) for i in row if i >= 0] for row in self.schedule]


class Berxit:
    """Berxit early-exit encoder on one B200 (include/mbx_berxit.h): parameters resident, one
    mini-batch per ``run`` (per-layer batches over the running instances, exits decided on the
    device)."""

    def __init__(self, device: int = 0, precision: str = "bf16x3", cfg: Optional[BerxitConfig] = None,
                 max_batch: int = 64):
        self.cfg = cfg if cfg is not None else berxit_config()
        self.max_batch = max_batch
        h = ctypes.c_void_p()
        if lib().mbx_berxit_create(device, PREC[precision], ctypes.byref(self.cfg), max_batch, ctypes.byref(h)):
            raise MbatchError(lib().mbx_berxit_last_error(None).decode())
        self.h = h

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib is not None:
            try:
                _lib.mbx_berxit_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self.h = None

    def _check(self, rc):
        if rc:
            raise MbatchError(lib().mbx_berxit_last_error(self.h).decode())

    def set_params(self, params: np.ndarray):
        p = np.ascontiguousarray(params, np.float32)
        self._check(lib().mbx_berxit_set_params(self.h, _ptr(p, ctypes.c_float), p.size))

    def make_params(self, seed: int) -> np.ndarray:
        p = berxit_make_params(self.cfg, seed)
        self.set_params(p)
        return p

    def _out(self, batch):
        return (np.empty((batch, self.cfg.classes), np.float32), np.empty(batch, np.int32),
                np.empty((self.cfg.layers, batch), np.int32))

    def run(self, x: np.ndarray) -> BerxitResult:
        """One mini-batch from host inputs [batch][seq][hidden] (synchronous)."""
        x = np.ascontiguousarray(x, np.float32)
        b = x.shape[0]
        lg, ex, sc = self._out(b)
        self._check(lib().mbx_berxit_run(self.h, b, _ptr(x, ctypes.c_float), _ptr(lg, ctypes.c_float),
                                         _ptr(ex, ctypes.c_int32), _ptr(sc, ctypes.c_int32)))
        return BerxitResult(lg, ex, sc)

    def run_into(self, x: np.ndarray, logits: np.ndarray, exit_layer: np.ndarray):
        """``run`` into caller-owned output arrays, without the schedule (the e2e timing call)."""
        self._check(lib().mbx_berxit_run(self.h, x.shape[0], _ptr(x, ctypes.c_float), _ptr(logits, ctypes.c_float),
                                         _ptr(exit_layer, ctypes.c_int32), None))

    def run_device(self, batch: int, x_dev_ptr: int):
        """Enqueues one mini-batch whose inputs are at device address x_dev_ptr (asynchronous)."""
        self._check(lib().mbx_berxit_run_device(self.h, batch, ctypes.c_void_p(x_dev_ptr)))

    def read(self, batch: int) -> BerxitResult:
        lg, ex, sc = self._out(batch)
        self._check(lib().mbx_berxit_read(self.h, batch, _ptr(lg, ctypes.c_float), _ptr(ex, ctypes.c_int32),
                                          _ptr(sc, ctypes.c_int32)))
        return BerxitResult(lg, ex, sc)

    def stream(self) -> int:
        return lib().mbx_berxit_stream(self.h) or 0

    def launches_per_batch(self, batch: int) -> int:
        return lib().mbx_berxit_launches_per_batch(self.h, batch)

#!/usr/bin/env python
"""Benchmark of the batched-execution hot path (BASELINE.json: "batched nodes/sec and ms per
mini-batch (bs 8/64) at 1/2/4/8 B200 vs CPU ref").

A mini-batch of the workload is evaluated end to end by the runtime: fibers + inline-depth DFG
construction + depth scheduling on the host, every batch as a device launch, synthetic inputs
from the reference's zoo generators.  Default workload: TreeLSTM hidden 512, batch 64 (the
headline config, BASELINE.json configs[1]).

A step = T x R independent mini-batches (R = 16 per worker) evaluated by the native throughput pool
(mbx_pool_run: T host worker threads, one context and stream each; the persistent kernels chained
through a per-device lane) — the same use of the host cores as the reference arm, which runs one
process per core.
  value  nodes/s with every mini-batch's inputs already resident in HBM (no input H2D, outputs
         left in HBM), CUDA events on the worker streams around each step, L2 flushed between
         steps.
  e2e    the same with HOST buffers: H2D of the inputs, the run, D2H of the outputs, every
         mini-batch (mbx_evaluate_batch semantics per mini-batch).
  latency  one mini-batch at a time on one context (ms per mini-batch, host split, per-signature
         device times) — the roofline figures come from this single-stream run.
Multi-GPU (torchrun, one process per GPU): each rank runs its own mini-batch (seed + rank) —
instances shard independently, no collective on the data path ("scaling": "weak"); NCCL is used
only for the start barrier and the max-over-ranks of the timings.

--impl reference: the reference's own CPU implementation (oracle/_ref/mbatch_ref, the unmodified
reference compiled here) on the host cores, one process per core, each timing evaluate_batch on
its own mini-batch.
"""
import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
METRIC = "batched nodes/sec and ms per mini-batch (bs 8/64) at 1/2/4/8 B200 vs CPU ref"
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "mbatch_ref")


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--model", default="treelstm")
    p.add_argument("--hidden", type=int, default=512)
    p.add_argument("--batch", type=int, default=64)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--precision", default="bf16x3", choices=["fp32", "bf16x3", "bf16x6", "bf16"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--threads", type=int, default=0,
                   help="host worker threads of the throughput pool (0: cores per rank - 2)")
    p.add_argument("--per-thread", type=int, default=16, help="mini-batches per worker thread per step")
    p.add_argument("--no-other-configs", action="store_true",
                   help="skip the per-config latency table of the other BASELINE configs")
    return p.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        j = json.load(open(path))
        return {"hbm_gbs": j["hbm_gbs"], "bf16_tflops": j["bf16_tflops"],
                "bf16_tflops_sustained": j.get("bf16_tflops_sustained", j["bf16_tflops"]), "src": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1590.0, "src": "fallback"}


# ---- algorithmic work --------------------------------------------------------

def decode_plan(enc):
    """mbx plan encoding -> dict with shapes and steps (see include/mbx.h)."""
    e = list(enc)
    i = 0

    def get():
        nonlocal i
        i += 1
        return e[i - 1]

    def ref():
        return (get(), get(), get(), get())

    p = {"ghost": get(), "shared": [], "batched": [], "steps": [], "outputs": []}
    for _ in range(get()):
        p["shared"].append((get(), get()))
    for _ in range(get()):
        p["batched"].append((get(), get()))
    for _ in range(get()):
        st = {"kind": get(), "op": get(), "out": (get(), get())}
        st["ins"] = [ref() for _ in range(get())]
        st["chain"] = []
        for _ in range(get()):
            op, has = get(), get()
            r = ref()
            st["chain"].append((op, r if has else None))
        p["steps"].append(st)
    for _ in range(get()):
        p["outputs"].append(ref())
    return p


def launch_work(plan, b, weight_bytes):
    """(flops, bytes) of one launch of `plan` over b nodes: dense steps 2*m*k*n per node (steps whose
    operands are all shared count once per launch), bytes = shared tensors once (weights at their
    storage width) + b * (batched inputs + outputs) in fp32."""
    def shape(r, cur):
        kind, idx, off, cols = r
        s = plan["shared"][idx] if kind == 0 else plan["batched"][idx] if kind == 1 else plan["steps"][idx]["out"]
        return (1, cols) if cols >= 0 else s

    shared_only = []
    flops = 0
    for s, st in enumerate(plan["steps"]):
        refs = list(st["ins"]) + [r for _, r in st["chain"] if r is not None]
        so = all(r[0] == 0 or (r[0] == 2 and shared_only[r[1]]) for r in refs)
        shared_only.append(so)
        if st["op"] == 0 and st["kind"] in (0, 1):
            a = shape(st["ins"][0], s)
            n = sum(shape(w, s)[1] for w in st["ins"][1:])
            f = 2 * a[0] * a[1] * n
            flops += f if so else f * b
    sbytes = 0
    for (r, c) in plan["shared"]:
        sbytes += r * c * (weight_bytes if r > 1 else 4)
    bbytes = sum(r * c * 4 for (r, c) in plan["batched"])
    obytes = sum(shape(o, len(plan["steps"]))[0] * shape(o, len(plan["steps"]))[1] * 4 for o in plan["outputs"])
    return flops, sbytes + b * (bbytes + obytes)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, device):
        self.device = device
        self.lines = []
        self.proc = None

    def __enter__(self):
        if shutil.which("nvidia-smi"):
            q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons), "samples": len(sm)}


# ---- CPU legs ----------------------------------------------------------------------------------

def cpu_reference_time(model, hidden, batch, seed, reps):
    """Times the reference's batched CPU path (runtime::evaluate_batch) in oracle/_ref/mbatch_ref."""
    out = subprocess.check_output([REF_BIN, "time", "--model", model, "--hidden", str(hidden), "--batch", str(batch),
                                   "--seed", str(seed), "--reps", str(reps), "--no-verify"], text=True)
    return json.loads(out)


def cpu_port_time(model, hidden, batch, seed, reps):
    """Fallback when the reference binary is absent: the oracle restatement (unbatched)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from conftest import Oracle
    o = Oracle()
    m = o.model(model, hidden, seed)
    m.make_inputs(seed, batch)
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        m.evaluate()
        best = min(best, (time.perf_counter() - t0) * 1e3)
    return {"batched_ms_best": best, "batched_ms_mean": best, "nodes": None}


def cpu_baseline(args, nodes):
    if os.path.exists(REF_BIN):
        j = cpu_reference_time(args.model, args.hidden, args.batch, args.seed, 3)
        kind = "reference"
    else:
        j = cpu_port_time(args.model, args.hidden, args.batch, args.seed, 2)
        j["nodes"] = nodes
        kind = "port"
    ms = j["batched_ms_mean"]
    return {"value": j["nodes"] / (ms / 1e3), "unit": "nodes/s", "cores": 1, "kind": kind,
            "ms_per_minibatch": ms,
            "sample": f"{args.model} H={args.hidden} b={args.batch} seed {args.seed}: 1 warm-up + 3 timed "
                      f"evaluate_batch calls, single thread"}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if not os.path.exists(REF_BIN):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/mbatch_ref not built (needs /root/reference)"}))
        return
    P = os.cpu_count() or 1
    reps = max(1, args.steps)
    procs = []
    t0 = time.perf_counter()
    for k in range(P):
        procs.append(subprocess.Popen([REF_BIN, "time", "--model", args.model, "--hidden", str(args.hidden), "--batch",
                                       str(args.batch), "--seed", str(args.seed + k), "--reps", str(reps),
                                       "--warmup", str(max(1, args.warmup)), "--no-verify"],
                                      stdout=subprocess.PIPE, text=True))
    res = [json.loads(p.communicate()[0]) for p in procs]
    wall = time.perf_counter() - t0
    nodes_per_s = sum(r["nodes"] / (r["batched_ms_mean"] / 1e3) for r in res)
    ms = statistics.mean(r["batched_ms_mean"] for r in res)
    line = {"metric": METRIC, "impl": "reference", "value": nodes_per_s, "unit": "nodes/s", "n_gpus": args.gpus,
            "steps": reps, "warmup": max(1, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference zoo generators, seeds %d..%d)" % (
                args.seed, args.seed + P - 1),
            "config": {"workload": f"{args.model}-h{args.hidden}-b{args.batch}", "hidden": args.hidden,
                       "batch": args.batch, "processes": P},
            "cpu_baseline": {"value": nodes_per_s, "unit": "nodes/s", "cores": P, "kind": "reference",
                             "sample": f"{P} processes x {reps} evaluate_batch calls (+{max(1, args.warmup)} warm-up) of the unmodified "
                                       f"reference, one mini-batch each; wall {wall:.1f}s"},
            "e2e": {"value": nodes_per_s, "unit": "nodes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ---- our arm -------------------------------------------------------------------------------------

def run_ours(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        # NCCL's init lines (ranks, transports) on stderr, so the rank count can be checked; the
        # JSON line stays alone on stdout.  NCCL only carries the start barrier and the final
        # max / sum of the timings: nothing on the data path.
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    from paper_2305_10611_b200 import mbx

    ctx = mbx.Context(local, args.precision)
    model = mbx.Model(ctx, args.model, args.hidden)
    model.make_params(args.seed)
    seed = args.seed + rank
    toks, data = pinned_inputs(torch, *model.make_inputs(seed, args.batch))
    stream = torch.cuda.ExternalStream(ctx.stream(), device=local)
    l2 = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    def step(**kw):
        kw.setdefault("trace", False)
        return model.evaluate_batch(toks, data, args.batch, record_nodes=False, decode=False, **kw)

    for _ in range(max(3, args.warmup)):
        r0 = step()
    nodes = r0.trace.total_nodes
    step(inputs_resident=False)  # leave this mini-batch's inputs in the arena for region A

    def timed(kw, per_batch=False):
        evs = []
        batch_us = []
        host = 0.0
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                l2.zero_()  # flush L2 between steps (256 MiB > 126 MB L2)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
            t0 = time.perf_counter()
            r = step(**kw)
            host += time.perf_counter() - t0
            with torch.cuda.stream(stream):
                b.record(stream)
            evs.append((a, b))
            if per_batch:
                batch_us.append(r.timing.batch_us)
        torch.cuda.synchronize(local)
        dev_ms = sum(a.elapsed_time(b) for a, b in evs)
        return dev_ms, host * 1e3, r, batch_us

    if dist:
        dist.barrier()
    torch.cuda.synchronize(local)
    launches0 = mbx.lib().mbx_kernel_launch_count()
    with ClockSampler(local) as clocks:
        pool_res = run_pool(args, mbx, torch, local, rank, world, nodes, l2)
        launches0 = mbx.lib().mbx_kernel_launch_count()
        dev_ms, host_ms, rA, _ = timed({"inputs_resident": True, "outputs_on_device": True, "time_kernels": True})
        gpu_launches = mbx.lib().mbx_kernel_launch_count() - launches0
        e2e_ms, e2e_host_ms, rB, _ = timed({})
        prof_ms, _, rC, batch_us = timed({"time_batches": True, "trace": True}, per_batch=True)
    times = torch.tensor([dev_ms, e2e_ms, float(nodes)], dtype=torch.float64, device=f"cuda:{local}")
    if dist:
        mx = times.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        tot = times.clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        dev_max, e2e_max, nodes_total = float(mx[0]), float(mx[1]), float(tot[2])
    else:
        dev_max, e2e_max, nodes_total = dev_ms, e2e_ms, float(nodes)
    if rank != 0:
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    K = args.steps
    lat_value = nodes_total * K / (dev_max / 1e3)
    lat_e2e = nodes_total * K / (e2e_max / 1e3)
    value, e2e = pool_res["value"], pool_res["e2e"]
    pk = peaks()
    # Per-signature device time from region C and algorithmic work of each launch.
    sigs = model.signatures()
    plans = {s: decode_plan(model.plan_encoding(s)) for s in range(len(sigs))}
    wbytes = 2 if args.precision == "bf16" else 4
    per_sig = {}
    R_total_us = 0.0
    meas_total_us = 0.0
    launch_rows = [b for b in rC.trace.batches if not b.ghost]
    for k_step in batch_us:
        for b, us in zip(launch_rows, k_step):
            f, by = launch_work(plans[b.sig], b.size, wbytes)
            e = per_sig.setdefault(b.sig, {"us": 0.0, "flops": 0.0, "bytes": 0.0, "launches": 0})
            e["us"] += us
            e["flops"] += f
            e["bytes"] += by
            e["launches"] += 1
            # in-step kernels: the sustained tensor peak
            R_total_us += max(f / (pk["bf16_tflops_sustained"] * 1e6), by / (pk["hbm_gbs"] * 1e3))
            meas_total_us += us
    dom = max(per_sig, key=lambda s: per_sig[s]["us"])
    d = per_sig[dom]
    t_s = d["us"] / 1e6
    tensor_path = args.precision != "fp32"
    compute_peak = pk["bf16_tflops"] if tensor_path else 74.4  # FP32 SIMT: 148 SM x 128 FMA x 2 x 1.965 GHz
    bound = "tensor" if d["flops"] / (compute_peak * 1e12) > d["bytes"] / (pk["hbm_gbs"] * 1e9) else "hbm"
    if bound == "hbm":
        ach, peak, unit = d["bytes"] / t_s / 1e9, pk["hbm_gbs"], "GB/s"
    else:
        ach, peak, unit = d["flops"] / t_s / 1e12, compute_peak, "TFLOP/s"
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        tj = json.load(open(prof))
        traffic = tj.get(f"{args.model}-h{args.hidden}-b{args.batch}-{args.precision}-{sigs[dom]}")
    clk = clocks.summary()
    line = {
        "metric": METRIC, "value": value, "unit": "nodes/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": pool_res["ms_per_step"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": {"fp32": "f32", "bf16x3": "bf16x3 (split-bf16 tcgen05, fp32 accumulate)",
                  "bf16x6": "bf16x6 (three-part split-bf16 tcgen05, fp32 accumulate)", "bf16": "bf16"}[args.precision],
        "data": f"synthetic: reference zoo generators (params seed {args.seed}, inputs seed {args.seed}+rank)",
        "config": {"workload": f"{args.model}-h{args.hidden}-b{args.batch}", "hidden": args.hidden,
                   "batch": args.batch, "nodes_per_minibatch": nodes, "precision": args.precision,
                   "l2": "flushed between steps (256 MiB write)", "parallelism": f"instance shards x{world}",
                   "minibatches_per_step": pool_res["threads"] * pool_res["per_thread"],
                   "host_threads": pool_res["threads"]},
        "e2e": {"value": e2e, "unit": "nodes/s", "ms_per_step": pool_res["e2e_ms_per_step"],
                "h2d_bytes_per_step": rB.timing.h2d_bytes * pool_res["threads"] * pool_res["per_thread"],
                "d2h_bytes_per_step": rB.timing.d2h_bytes * pool_res["threads"] * pool_res["per_thread"]},
        "latency": {"ms_per_minibatch": dev_max / K, "e2e_ms_per_minibatch": e2e_max / K,
                    "nodes_per_s": lat_value, "e2e_nodes_per_s": lat_e2e,
                    "def": "one mini-batch at a time on one context, device events around each call"},
        "gpu_launches": int(gpu_launches) + pool_res["launches"],
        "roofline": {"bound": bound, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
                     "traffic": traffic, "kernel": sigs[dom], "launches_per_step": d["launches"] // K,
                     "peak_src": pk["src"] if tensor_path or bound == "hbm" else "fp32 SIMT nominal"},
        "step_roofline": {"R_us": R_total_us / K, "kernel_us": meas_total_us / K,
                          "frac": (R_total_us / meas_total_us) if meas_total_us else None,
                          "def": "sum over launches of max(F/sustained bf16 peak, B/HBM) vs summed launch times (SURVEY 8d)"},
        "breakdown_us_per_step": {"host_dfg_and_launch": rA.timing.host_dfg_us, "host_split": rA.timing.host_breakdown,
                                  "device_span": rA.timing.device_span_us,
                                  "per_sig": {sigs[s]: v["us"] / K for s, v in per_sig.items()}},
        "clocks": clk,
        "parity": pool_res["parity"],
    }
    # Whether this rank's host workers can feed its GPU: each needs host_ms of CPU per mini-batch
    # (DFG + scheduling + launch, the latency run's host split), the GPU ~ms_per_step / minibatches.
    host_ms = rA.timing.host_dfg_us / 1e3
    dev_mb_ms = pool_res["ms_per_step"] / max(1, pool_res["threads"] * pool_res["per_thread"])
    line["host_capacity"] = {"cores_per_rank": pool_res["cores"], "workers": pool_res["threads"],
                             "host_ms_per_minibatch": host_ms, "device_ms_per_minibatch": dev_mb_ms,
                             "keeps_up": pool_res["threads"] / host_ms >= 1.0 / dev_mb_ms}
    if world == 1 and not args.no_other_configs:
        line["other_configs"] = other_configs(mbx, torch, local)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, nodes)
    if world == 1 and not args.no_other_configs:
        line["berxit"] = berxit_section(mbx, torch, local, l2, pk, cpu=not args.no_cpu_baseline)
    print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


# The other BASELINE.json configs with the precision SURVEY §8a assigns them (rel 1e-5 -> the
# bit-exact FP32 path, rel 1e-3 -> bf16x3 tensor cores).  Parity for all of them: tests/.
OTHER_CONFIGS = [("treelstm", 256, 8, "fp32"), ("treelstm", 512, 8, "bf16x3"), ("mvrnn", 128, 64, "fp32"),
                 ("birnn", 512, 64, "bf16x3"), ("nestedrnn", 512, 64, "bf16x3"), ("nestedrnn", 512, 8, "bf16x3")]


def other_configs(mbx, torch, local, reps=5):
    """ms per mini-batch (one at a time on one context, CUDA events around each call, inputs
    resident) and nodes/s for the other BASELINE configs."""
    out = {}
    for model, hidden, batch, prec in OTHER_CONFIGS:
        ctx = mbx.Context(local, prec)
        m = mbx.Model(ctx, model, hidden)
        m.make_params(1)
        toks, data = m.make_inputs(1, batch)
        stream = torch.cuda.ExternalStream(ctx.stream(), device=local)
        r = None
        for _ in range(2):
            r = m.evaluate_batch(toks, data, batch, record_nodes=False, decode=False, trace=False)
        ms = []
        for _ in range(reps):
            with torch.cuda.stream(stream):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
            r = m.evaluate_batch(toks, data, batch, record_nodes=False, decode=False, trace=False,
                                 inputs_resident=True, outputs_on_device=True, time_kernels=True)
            with torch.cuda.stream(stream):
                b.record(stream)
            b.synchronize()
            ms.append(a.elapsed_time(b))
        best = min(ms)
        out[f"{model}-h{hidden}-b{batch}-{prec}"] = {
            "ms_per_minibatch": best, "nodes": r.trace.total_nodes, "nodes_per_s": r.trace.total_nodes / (best / 1e3),
            "device_us": r.timing.device_span_us, "host_us": r.timing.host_dfg_us, "batches": r.trace.kernel_launches}
        m.close()
        ctx.close()
    return out


# ACRoBat's published Berxit latencies (BERT-base "small", RTX 3070).
BERXIT_PUBLISHED_MS = {64: 204.54, 8: 38.49}


def berxit_section(mbx, torch, local, l2, pk, cpu=True, reps=10):
    """BASELINE configs[4]: Berxit early-exit BERT-base encoder (include/mbx_berxit.h), batch 64 and 8,
    bf16x3 tensor cores.  Parity against tests/golden/berxit.json.gz (oracle-made, parity
    unpinned); device ms per mini-batch (inputs resident, CUDA events on the model's stream, L2
    flushed before every mini-batch) and e2e ms (pinned host inputs H2D + run + results D2H through
    mbx_berxit_run); the published ACRoBat latency beside it."""
    import gzip
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from parity_metrics import elementwise
    with gzip.open(os.path.join(ROOT, "tests", "golden", "berxit.json.gz"), "rt") as f:
        runs = {r["batch"]: r for r in json.load(f)["runs"] if r["name"] == "bert-base"}
    out = {}
    for b in (64, 8):
        run = runs[b]
        c = mbx.berxit_config(**run["config"])
        m = mbx.Berxit(local, "bf16x3", c, max_batch=b)
        m.make_params(run["seed"])
        xh = torch.from_numpy(mbx.berxit_make_inputs(c, run["seed"], b)).pin_memory()
        xd = xh.to(f"cuda:{local}")
        r = m.run(xh.numpy())
        want_lg = np.asarray(run["logits"], np.float32)
        st = elementwise(r.logits, want_lg, 1e-3)
        scale = np.sqrt(np.mean(want_lg.astype(np.float64) ** 2, axis=-1, keepdims=True))
        parity = {"golden": f"tests/golden/berxit.json.gz bert-base b{b} seed {run['seed']} (oracle, parity unpinned)",
                  "exit_layers_equal": bool(np.array_equal(r.exit_layer, run["exit_layer"])),
                  "schedule_equal": r.batches() == [[i for i, e in enumerate(run["exit_layer"]) if e >= l]
                                                    for l in range(c.layers)],
                  "max_rel": st["max_rel"], "frac_pass_rel1e-3": st["frac_pass"], "normwise": st["normwise"],
                  "max_err_over_row_rms": float(np.max(np.abs(r.logits - want_lg) / scale))}
        stream = torch.cuda.ExternalStream(m.stream(), device=local)
        for _ in range(3):
            m.run_device(b, xd.data_ptr())
        torch.cuda.synchronize(local)
        dev, e2e = [], []
        for _ in range(reps):
            l2.zero_()
            torch.cuda.synchronize(local)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            m.run_device(b, xd.data_ptr())
            e1.record(stream)
            e1.synchronize()
            dev.append(e0.elapsed_time(e1))
        lg = np.empty((b, c.classes), np.float32)
        ex = np.empty(b, np.int32)
        for _ in range(reps):
            l2.zero_()
            torch.cuda.synchronize(local)
            t0 = time.perf_counter()
            m.run_into(xh.numpy(), lg, ex)
            e2e.append((time.perf_counter() - t0) * 1e3)
        layer_inst = sum(len(bt) for bt in r.batches())
        H, F, S = c.hidden, c.ffn, c.seq
        flops = layer_inst * S * 2 * (4 * H * H + 2 * H * F + 2 * S * H)  # GEMMs + the two attention products
        ms = statistics.median(dev)
        tensor = flops * 3 / (ms * 1e-3) / 1e12  # bf16x3: three tcgen05 products per contraction
        out[f"b{b}"] = {
            "ms_per_minibatch": ms, "ms_min": min(dev), "e2e_ms_per_minibatch": statistics.median(e2e),
            "h2d_bytes": int(xh.numel() * 4), "d2h_bytes": int(b * (c.classes + 1 + c.layers) * 4),
            "published_acrobat_ms": BERXIT_PUBLISHED_MS[b], "published_hw": "RTX 3070 (PAPER.md:846-847)",
            "speedup_vs_published_e2e": BERXIT_PUBLISHED_MS[b] / statistics.median(e2e),
            "layer_instances": layer_inst, "exits_per_layer": np.bincount(r.exit_layer, minlength=c.layers).tolist(),
            "launches_per_minibatch": m.launches_per_batch(b),
            "roofline": {"bound": "tensor", "achieved_algorithmic_tflops": flops / (ms * 1e-3) / 1e12,
                         "achieved_tensor_tflops": tensor, "peak": pk["bf16_tflops_sustained"], "unit": "TFLOP/s",
                         "frac": tensor / pk["bf16_tflops_sustained"],
                         "def": "tensor = 3 split-bf16 products per algorithmic FMA; peak = measured sustained bf16"},
            "parity": parity}
        del m
    cfg = mbx.berxit_config()
    out["config"] = {"model": "Berxit (BERT-base, shared layers, LTE exit)", "hidden": cfg.hidden, "heads": cfg.heads,
                     "ffn": cfg.ffn, "layers": cfg.layers, "seq": cfg.seq, "classes": cfg.classes,
                     "exit_threshold": cfg.exit_threshold, "precision": "bf16x3", "l2": "flushed before each mini-batch"}
    if cpu:
        out["cpu_baseline"] = berxit_cpu(mbx, runs[64])
    return out


def berxit_cpu(mbx, run):
    """The oracle restatement (oracle/berxit_oracle.cpp, the only CPU Berxit: the reference has none)
    on one full-depth instance, one thread."""
    from test_berxit import BerxitOracle
    o = BerxitOracle()
    c = mbx.berxit_config(**run["config"])
    i = run["exit_layer"].index(c.layers - 1)
    p = o.params(c, run["seed"])
    x = o.inputs(c, run["seed"], [i])
    t0 = time.perf_counter()
    o.run(c, p, x, threads=1)
    s = time.perf_counter() - t0
    mean_layers = (np.mean(run["exit_layer"]) + 1) / c.layers
    return {"kind": "port", "cores": 1, "s_per_instance_12_layers": s,
            "ms_per_minibatch_b64_1core": s * 1e3 * 64 * mean_layers,
            "sample": f"oracle, instance {i} (exits after layer {c.layers}), one thread"}


def pinned_inputs(torch, toks, data):
    """The hostval-encoded inputs with the float data stream in page-locked host memory."""
    pd = torch.empty(data.size, dtype=torch.float32, pin_memory=True).numpy()
    pd[:] = data
    return toks, pd


def checked_minibatch(args, pool, gen):
    """One mini-batch (seed args.seed) through a pool worker's own context before the timed
    region, compared with the reference's golden outputs and schedule for the same config
    (tests/golden/baseline.json.gz, written by the unmodified reference): SURVEY §8a's per-element
    metric (|ours - ref| <= tol * max(|ref|, 1e-6), max-rel, fraction passing), normwise, and the
    schedule compared batch by batch."""
    import gzip
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from parity_metrics import elementwise, merge
    from conftest import trace_counters, trace_rows
    with gzip.open(os.path.join(ROOT, "tests", "golden", "baseline.json.gz"), "rt") as f:
        runs = json.load(f)
    run = next((r for r in runs if (r["model"], r["hidden"], r["batch"], r["seed"]) ==
                (args.model, args.hidden, args.batch, args.seed) and "outputs" in r), None)
    if run is None:
        return {"checked": False, "why": "no reference golden for this config"}
    toks, data = gen.make_inputs(args.seed, args.batch)
    r = pool.evaluate_on_worker(0, toks, data, args.batch)
    tol = 1e-5 if args.precision == "fp32" else 1e-3

    def flat(j):
        return list(j["d"]) if j["k"] == "t" else [x for it in j.get("items", []) for x in flat(it)]
    st = merge([elementwise(mbx_flat(r.outputs[i]), np.asarray(flat(o), np.float32), tol)
                for i, o in enumerate(run["outputs"])])
    return {"checked": True, "against": "reference golden (tests/golden/baseline.json.gz) %s-h%d-b%d seed %d" % (
        args.model, args.hidden, args.batch, args.seed), "tol_rel": tol, "max_rel": st["max_rel"],
            "frac_pass": st["frac_pass"], "normwise": st["normwise"], "elements": st["n"],
            "schedule_equal": trace_rows(r.trace) == trace_rows(run["trace"]) and
            trace_counters(r.trace) == trace_counters(run["trace"])}


def mbx_flat(v):
    from paper_2305_10611_b200 import mbx
    return mbx.flatten_floats(v)


def run_pool(args, mbx, torch, local, rank, world, nodes, l2):
    """Throughput: T worker threads, each evaluating its own mini-batch per step (mbx_pool_run).
    Returns value / e2e nodes/s and the per-step device times (CUDA events on the pool stream)."""
    # Host worker threads per rank: the cores this process may run on, shared evenly by the ranks
    # of the node, one left for the driver thread (each worker's host side, ~0.3-0.5 ms per
    # TreeLSTM-512 b64 mini-batch, must keep pace with ~0.1 ms of device work per mini-batch).
    avail = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    cores = max(1, avail // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", world))))
    T = args.threads or max(1, cores - 1)
    pool = mbx.Pool(local, args.precision, args.model, args.hidden, args.seed, T)
    ctx = mbx.Context(-1, args.precision)  # host-only: the synthetic inputs
    gen = mbx.Model(ctx, args.model, args.hidden)
    # Host inputs in pinned memory (the e2e contract: H2D from pinned host buffers): the library
    # then copies each mini-batch's data stream in one piece and scatters it on the device.
    ins = [pinned_inputs(torch, *gen.make_inputs(args.seed + rank * T + w, args.batch)) for w in range(T)]
    parity = checked_minibatch(args, pool, gen) if rank == 0 else None
    def steps(K, kw):
        ms, total = 0.0, 0
        for _ in range(K):
            l2.zero_()  # flush L2 between steps (256 MiB > 126 MB L2)
            torch.cuda.synchronize(local)
            # device time of the step: CUDA events on every worker stream (first start -> last end)
            n, dev_ms = pool.run_timed(ins * args.per_thread, args.batch, **kw)
            total += n
            ms += dev_ms
        return ms, total

    steps(max(3, args.warmup), {})
    steps(1, {"inputs_resident": False})  # every worker's inputs now resident in its arena
    launches0 = mbx.lib().mbx_kernel_launch_count()
    dev_ms, n1 = steps(args.steps, {"inputs_resident": True, "outputs_on_device": True})
    launches = mbx.lib().mbx_kernel_launch_count() - launches0
    e2e_ms, n2 = steps(args.steps, {})
    t = torch.tensor([dev_ms, e2e_ms, float(n1), float(n2)], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        import torch.distributed as dist
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        tot = t.clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        dev_ms, e2e_ms, n1, n2 = float(mx[0]), float(mx[1]), float(tot[2]), float(tot[3])
    pool.close()
    return {"value": n1 / (dev_ms / 1e3), "e2e": n2 / (e2e_ms / 1e3), "ms_per_step": dev_ms / args.steps,
            "e2e_ms_per_step": e2e_ms / args.steps, "threads": T, "cores": cores, "per_thread": args.per_thread,
            "launches": int(launches), "parity": parity}


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

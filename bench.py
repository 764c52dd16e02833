#!/usr/bin/env python
"""Benchmark of the B200 AMS-Quant fused linear (BASELINE.json).

N = 1 (default): config 2. A *step* is one pass over the Llama-3.1-8B layer linears
(qkv 6144x4096, o 4096x4096, gate_up 28672x4096, down 4096x14336) at every batch M in
{1, 4, 8, 16}: 16 fused restore+linear calls on FP5.33-e2m3 weights, captured as one CUDA
graph. ``value`` is packed-weight GB/s over the timed region (reference-stream payload
bytes, quantize.hpp:64-69, / device time), inputs resident in HBM; ``e2e`` is the same
metric through the C-ABI ``amsq_gemv_host`` (pinned host x/y, H2D + kernel + D2H per call).
Weights rotate over enough copies to stream > 2x the 126 MB L2 per rotation.

N > 1 (torchrun): config 4, the north-star multi-GPU path. Each rank holds the N-shard
[p*N/P, (p+1)*N/P) of every Llama-3.1-70B linear, and one call is the C-ABI
``amsq_linear_tp``: the rank's fused linear, ``ncclAllGather`` of the [M][N/P] outputs
over NVLink and the unshard permutation into the reference [M][N] layout. ``value`` is the
whole job's packed GB/s (all shards' bytes / max-over-ranks device time).

The headline JSON line is compact and printed last. ``--extra FILE`` adds the batch sweep
(config 3), the 32-layer stack (config 5) and the per-rank 70B shard kernels, written to
FILE (not to stdout). ``--impl reference`` times the reference's own CPU ``amsq::gemv``
(oracle/_ref, all host threads) on the same workload; it never loads this repo's library.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SHAPES_8B = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096),
             "down": (4096, 14336)}
SHAPES_70B = {"qkv": (10240, 8192), "o": (8192, 8192), "gate_up": (57344, 8192),
              "down": (8192, 28672)}
L2_BYTES = 126 * 1024 * 1024
ROTATE_BYTES = 2.1 * L2_BYTES  # a rotation over the copies streams > 2x L2

# (block, words_per_block) of the reference stream, packing.hpp:6-25 -- kept local so the
# reference arm never loads this repo's library
_BLOCK = {"fp4.25-e2m2": (4, 64, 17), "fp5.33-e2m3": (7, 3, 1)}
METRIC = ("AMS linear packed-weight HBM GB/s (Llama-3.1-8B qkv/o/gate_up/down x batch "
          "1/4/8/16; per-call us and speedup vs FP16 cuBLAS)")
METRIC_TP = ("AMS linear packed-weight HBM GB/s, Llama-3.1-70B qkv/o/gate_up/down N-sharded "
             "over the GPUs + NCCL all-gather (x batch 1/4/8/16)")


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return (float(d["hbm_gbs"]), float(d.get("bf16_tflops_sustained", 1379.1)),
                "MEASURED_PEAKS.json hbm_gbs (copy peak)")
    except Exception:
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


def _dist():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
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
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ workload data (numpy only)
def make_stream(scheme, rows, cols, seed):
    """Random valid packed stream: (padded_cols, scales u16, payload u16).

    Every u16 stream unpacks and decodes finite (packing.hpp:190-212, format.hpp:113-118);
    FP5.33 padding codes are zeroed so the padding restores to 0."""
    sid, block, wpb = _BLOCK[scheme]
    rng = np.random.default_rng(seed)
    pc = (cols + block - 1) // block * block
    wpr = pc // block * wpb
    payload = rng.integers(0, 1 << 16, size=(rows, wpr), dtype=np.uint16)
    for c in range(cols, pc):  # only FP5.33 pads (K = 4096/14336/8192/28672 are 64-aligned)
        blk, j = divmod(c, block)
        payload[:, blk] &= np.uint16(~(0x1F << (5 * j)) & 0x7FFF)
    scales = rng.uniform(0.002, 0.02, size=rows).astype(np.float16).view(np.uint16)
    return pc, scales, payload.reshape(-1)


def payload_bytes_of(scheme, rows, cols):
    """packed_payload_bytes (quantize.hpp:64-69)."""
    _, block, wpb = _BLOCK[scheme]
    return rows * ((cols + block - 1) // block) * wpb * 2


def algorithmic_bytes(pbytes, rows, cols, m):
    """payload + scales + x + y per call."""
    return pbytes + 2 * rows + 2 * m * cols + 2 * m * rows


def _qt(scheme, rows, cols, seed):
    import paper_2510_16045_b200 as amsq
    pc, scales, payload = make_stream(scheme, rows, cols, seed)
    return amsq.QuantizedTensor(amsq.scheme_by_name(scheme), rows, cols, pc, scales, payload)


def _n_copies(nbytes, minimum=2):
    return max(minimum, int(np.ceil(ROTATE_BYTES / max(1, nbytes))))


def _graph_us(fn, reps_in_graph, replays, stream, cap):
    """Device time per call of fn(r), captured reps_in_graph times in one CUDA graph."""
    import torch
    with torch.cuda.stream(cap):
        fn(0)
        cap.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            for r in range(reps_in_graph):
                fn(r)
    stream.wait_stream(cap)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(replays):
        g.replay()
    b.record(stream)
    torch.cuda.synchronize()
    del g
    return a.elapsed_time(b) * 1e3 / (replays * reps_in_graph)


def _lin(handle, x, m, y, st):
    from paper_2510_16045_b200._lib import lib
    rc = lib().amsq_linear(handle, x.data_ptr(), m, y.data_ptr(), st)
    if rc:
        raise RuntimeError(lib().amsq_last_error().decode())


# ------------------------------------------------------------------ GPU arm, N = 1: config 2
def run_config2(args, local):
    import torch
    import torch.nn.functional as F

    import paper_2510_16045_b200 as amsq

    dev = torch.device(f"cuda:{local}")
    shapes = SHAPES_8B
    batches = [int(b) for b in args.batches.split(",")]
    pbytes = {name: payload_bytes_of(args.scheme, n, k) for name, (n, k) in shapes.items()}
    copies = _n_copies(sum(pbytes.values()))
    sets = [{name: amsq.DeviceWeight(_qt(args.scheme, n, k, seed=1000 * c + i), device=local)
             for i, (name, (n, k)) in enumerate(shapes.items())} for c in range(copies)]
    xs = {(name, m): torch.randn(m, k, device=dev).half() for name, (n, k) in shapes.items()
          for m in batches}
    ys = {(name, m): torch.empty(m, n, device=dev, dtype=torch.float16)
          for name, (n, k) in shapes.items() for m in batches}
    calls = [(name, m) for m in batches for name in shapes]
    stream = torch.cuda.current_stream()
    cap = torch.cuda.Stream()
    cap.wait_stream(stream)

    # one step = the 16 calls as one CUDA graph per weight copy (PDL-chained launches)
    graphs, per_step = [], 0
    with torch.cuda.stream(cap):
        for c in range(copies):  # per-function attributes are set outside capture
            for name, m in calls:
                _lin(sets[c][name].handle, xs[(name, m)], m, ys[(name, m)], cap.cuda_stream)
        cap.synchronize()
        for c in range(copies):
            g = torch.cuda.CUDAGraph()
            l0 = amsq.kernel_launch_count()
            with torch.cuda.graph(g, stream=cap):
                for name, m in calls:
                    _lin(sets[c][name].handle, xs[(name, m)], m, ys[(name, m)], cap.cuda_stream)
            per_step = amsq.kernel_launch_count() - l0
            graphs.append(g)
    stream.wait_stream(cap)
    total_ms, clocks = _timed_replays(args, graphs, stream, local, world=1, dev=dev)
    bytes_per_step = sum(pbytes[name] for name, m in calls)
    value = bytes_per_step * args.steps / (total_ms * 1e-3) / 1e9

    # per-call device time: graph of back-to-back calls of one (shape, M), weights rotating
    # over the copies; cuBLAS FP16 (F.linear -> cublasGemmEx) rotated the same way
    R = 2 * copies
    per_call, cub = {}, {}
    for name, m in calls:
        per_call[(name, m)] = _graph_us(
            lambda r, name=name, m=m: _lin(sets[r % copies][name].handle, xs[(name, m)], m,
                                           ys[(name, m)], cap.cuda_stream),
            R, max(5, args.steps), stream, cap)
    for name, (n, k) in shapes.items():
        nd = _n_copies(2 * n * k)
        dense = [torch.randn(n, k, device=dev).half() for _ in range(nd)]
        for m in batches:
            cub[(name, m)] = _graph_us(
                lambda r, name=name, m=m: F.linear(xs[(name, m)], dense[r % nd]),
                2 * nd, max(5, args.steps), stream, cap)
        del dense
    torch.cuda.empty_cache()

    peak, _, peak_kind = _peaks()
    alg_total, t_total = 0.0, 0.0
    for name, m in calls:
        n, k = shapes[name]
        alg_total += algorithmic_bytes(pbytes[name], n, k, m)
        t_total += per_call[(name, m)] * 1e-6
    achieved = alg_total / t_total / 1e9

    e2e = run_e2e(args, sets, shapes, calls, pbytes, world=1, dev=dev)
    traffic = _ncu_traffic(args.scheme)
    names = list(shapes)
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp16",
        "data": "synthetic: random valid packed streams, random fp16 x",
        "config": {"workload": f"config 2: {args.scheme} linear, Llama-3.1-8B qkv/o/gate_up/down "
                               f"x batch {args.batches} = {len(calls)} calls/step",
                   "scheme": args.scheme,
                   "l2": f"inputs > L2: weights rotate over {copies} copies "
                         f"({copies * sum(pbytes.values()) / 1e6:.0f} MB)",
                   "parallelism": "1 GPU"},
        "e2e": e2e,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic, "kernel": "amsq_linear_kernel (K2)",
                     "peak_src": peak_kind},
        "gpu_launches": int(per_step * args.steps),
        "clocks": clocks,
        "us_per_call": {nm: [round(per_call[(nm, m)], 2) for m in batches] for nm in names},
        "cublas_fp16_us": {nm: [round(cub[(nm, m)], 2) for m in batches] for nm in names},
    }
    if not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args, shapes, batches)
    if args.extra:
        for c in sets:
            for w in c.values():
                w.free()
        torch.cuda.empty_cache()
        extra = {"detail": [
            {"layer": nm, "N": shapes[nm][0], "K": shapes[nm][1], "M": m,
             "us": round(per_call[(nm, m)], 2),
             "packed_GBps": round(pbytes[nm] / per_call[(nm, m)] / 1e3, 1),
             "frac_of_peak": round(algorithmic_bytes(pbytes[nm], *shapes[nm], m)
                                   / per_call[(nm, m)] / 1e3 / peak, 3),
             "cublas_fp16_us": round(cub[(nm, m)], 2),
             "speedup_vs_cublas": round(cub[(nm, m)] / per_call[(nm, m)], 2)}
            for nm, m in calls]}
        t = time.time()
        for key, fn in (("batch_sweep", lambda: run_batch_sweep(args, dev, stream, cap)),
                        ("stack_32L", lambda: run_stack(args, dev, stream, cap)),
                        ("tp_shards_70B", lambda: run_tp_shards(args, dev, stream, cap))):
            try:
                extra[key] = fn()
            except Exception as e:  # an extra section must not take the headline down
                torch.cuda.synchronize()
                extra[key] = {"error": f"{type(e).__name__}: {e}"[:300]}
        extra["extra_seconds"] = round(time.time() - t, 1)
        _write_extra(args.extra, line, extra)
        line["extra_file"] = os.path.relpath(os.path.abspath(args.extra), ROOT)
    return line


def _timed_replays(args, graphs, stream, local, world, dev):
    """W warm-up replays, then EXACTLY `steps` replays between barrier + synchronize, device
    time (CUDA events on the replay stream), max over ranks; clocks sampled meanwhile."""
    import torch
    n = len(graphs)
    for i in range(args.warmup):
        graphs[i % n].replay()
    torch.cuda.synchronize()

    def busy(seconds):  # back-to-back replays so the clock samples see the loaded GPU
        end, i = time.time() + seconds, 0
        while time.time() < end:
            for _ in range(10):
                graphs[i % n].replay()
                i += 1
            torch.cuda.synchronize()

    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        busy(0.6)  # nvidia-smi needs ~0.1-0.3 s to start emitting samples
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0.record(stream)
        for i in range(args.steps):
            graphs[i % n].replay()
        t1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        busy(0.4)
    total_ms = t0.elapsed_time(t1)
    if world > 1:
        tt = torch.tensor([total_ms], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(tt.item())
    return total_ms, clk.summary()


def _ncu_traffic(scheme):
    """dram__bytes_read.sum + dram__bytes_write.sum of the dominant launch from one
    `ncu --set full` capture (profiles/ncu_traffic.json), per launch; None when absent."""
    try:
        rec = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get(scheme)
        return int(rec["traffic_bytes_per_launch"]) if rec else None
    except Exception:
        return None


def _write_extra(path, line, extra):
    d = os.path.dirname(os.path.abspath(path))
    os.makedirs(d, exist_ok=True)
    with open(path, "w") as f:
        json.dump({"headline": line, **extra}, f, indent=1)


def run_e2e(args, sets, shapes, calls, pbytes, world, dev):
    """The reference call shape through the C-ABI: amsq_gemv_host with pinned host x/y --
    H2D of x, the fused linear, D2H of y, synchronise -- for every call of the step."""
    import torch

    from paper_2510_16045_b200._lib import lib

    stream = torch.cuda.current_stream()
    hx = {(name, m): torch.randn(m, shapes[name][1]).half().pin_memory() for name, m in calls}
    hy = {(name, m): torch.empty(m, shapes[name][0], dtype=torch.float16).pin_memory()
          for name, m in calls}
    h2d = sum(2 * m * shapes[name][1] for name, m in calls)
    d2h = sum(2 * m * shapes[name][0] for name, m in calls)
    steps = max(3, args.steps // 2)

    def one(i):
        ws = sets[i % len(sets)]
        for name, m in calls:
            rc = lib().amsq_gemv_host(ws[name].handle, hx[(name, m)].data_ptr(),
                                      m * shapes[name][1], m, hy[(name, m)].data_ptr(),
                                      stream.cuda_stream)
            if rc:
                raise RuntimeError(lib().amsq_last_error().decode())

    # warm-up touches every weight copy: each handle's first M > 8 call creates its per-stream
    # workspace (a cudaMalloc), which must not land in the timed region
    for i in range(max(2, len(sets))):
        one(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for i in range(steps):
        one(i)
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    val = sum(pbytes[n] for n, m in calls) * steps / (ms * 1e-3) / 1e9
    return {"value": round(val, 1), "unit": "GB/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": round(ms / steps, 4),
            "path": "amsq_gemv_host per call (pinned host x/y)"}


# ------------------------------------------------------------------ GPU arm, N > 1: config 4
def run_config4_tp(args, world, rank, local):
    """Each rank: its N-shard of every 70B linear; one call = amsq_linear_tp (fused linear on
    the shard, ncclAllGather over NVLink, unshard to [M][N]); eager launches on one stream."""
    import ctypes as C

    import torch

    import paper_2510_16045_b200 as amsq
    from paper_2510_16045_b200._lib import check, lib

    dev = torch.device(f"cuda:{local}")
    stream = torch.cuda.current_stream()
    shapes = SHAPES_70B
    batches = [int(b) for b in args.batches.split(",")]
    P = world
    # one NCCL communicator over all ranks, made through the C-ABI (ncclCommInitRank)
    uid = (C.c_uint8 * 128)()
    if rank == 0:
        check(lib().amsq_nccl_unique_id(uid, 128), "nccl_unique_id")
    obj = [bytes(uid)]
    torch.distributed.broadcast_object_list(obj, src=0)
    C.memmove(uid, obj[0], 128)
    comm = C.c_void_p()
    check(lib().amsq_nccl_comm_init_rank(uid, 128, P, rank, local, C.byref(comm)),
          "nccl_comm_init_rank")

    shard_bytes = {name: payload_bytes_of(args.scheme, n // P, k) for name, (n, k) in shapes.items()}
    copies = _n_copies(sum(shard_bytes.values()))
    sets = []
    for c in range(copies):
        ws = {}
        for i, (name, (n, k)) in enumerate(shapes.items()):
            nl = n // P  # the rank's rows [rank*nl, (rank+1)*nl): generated directly
            ws[name] = amsq.DeviceWeight(_qt(args.scheme, nl, k, seed=10000 * c + 100 * i + rank),
                                         device=local)
        sets.append(ws)
    calls = [(name, m) for m in batches for name in shapes]
    xs = {(name, m): torch.randn(m, shapes[name][1], device=dev).half() for name, m in calls}
    ys = {(name, m): torch.empty(m, shapes[name][0], device=dev, dtype=torch.float16)
          for name, m in calls}
    need = max(2 * m * (shapes[name][0] // P) * (P + 1) for name, m in calls)
    scratch = torch.empty(need, dtype=torch.uint8, device=dev)

    def step(i):
        ws = sets[i % copies]
        for name, m in calls:
            rc = lib().amsq_linear_tp(ws[name].handle, xs[(name, m)].data_ptr(), m,
                                      ys[(name, m)].data_ptr(), scratch.data_ptr(), need, comm,
                                      P, stream.cuda_stream)
            if rc:
                raise RuntimeError(lib().amsq_last_error().decode())

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    l0 = amsq.kernel_launch_count()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        time.sleep(0.3)
        torch.distributed.barrier()
        torch.cuda.synchronize()
        t0.record(stream)
        for i in range(args.steps):
            step(i)
        t1.record(stream)
        torch.cuda.synchronize()
        torch.distributed.barrier()
    launches = amsq.kernel_launch_count() - l0
    total_ms = t0.elapsed_time(t1)
    tt = torch.tensor([total_ms], device=dev)
    torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
    total_ms = float(tt.item())
    full_bytes = sum(payload_bytes_of(args.scheme, *shapes[name]) for name, m in calls)
    value = full_bytes * args.steps / (total_ms * 1e-3) / 1e9

    # e2e: pinned host x -> H2D, amsq_linear_tp, D2H of the gathered [M][N] y, per call
    hx = {(name, m): torch.randn(m, shapes[name][1]).half().pin_memory() for name, m in calls}
    hy = {(name, m): torch.empty(m, shapes[name][0], dtype=torch.float16).pin_memory()
          for name, m in calls}

    def e2e_step(i):
        ws = sets[i % copies]
        for name, m in calls:
            xs[(name, m)].copy_(hx[(name, m)], non_blocking=True)
            rc = lib().amsq_linear_tp(ws[name].handle, xs[(name, m)].data_ptr(), m,
                                      ys[(name, m)].data_ptr(), scratch.data_ptr(), need, comm,
                                      P, stream.cuda_stream)
            if rc:
                raise RuntimeError(lib().amsq_last_error().decode())
            hy[(name, m)].copy_(ys[(name, m)], non_blocking=True)
            stream.synchronize()

    for i in range(copies):  # every weight copy once before the timed region
        e2e_step(i)
    torch.distributed.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    es = max(3, args.steps // 2)
    a.record(stream)
    for i in range(es):
        e2e_step(i)
    b.record(stream)
    torch.cuda.synchronize()
    ems = torch.tensor([a.elapsed_time(b)], device=dev)
    torch.distributed.all_reduce(ems, op=torch.distributed.ReduceOp.MAX)
    e2e_val = full_bytes * es / (float(ems.item()) * 1e-3) / 1e9
    fused = _tp_fused_variant(args, sets, calls, xs, shapes, P, rank, local, stream, copies,
                              full_bytes)
    peak, _, peak_kind = _peaks()
    per_rank_bytes = sum(shard_bytes[name] for name, m in calls)
    line = {
        "metric": METRIC_TP, "value": round(value, 1), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "fp16",
        "data": "synthetic: random valid packed streams, random fp16 x",
        "config": {"workload": f"config 4: {args.scheme} Llama-3.1-70B qkv/o/gate_up/down, "
                               f"N-sharded over {P} GPUs + ncclAllGather, x batch "
                               f"{args.batches} = {len(calls)} calls/step",
                   "scheme": args.scheme, "parallelism": f"tp{P} (column-parallel N-shards)",
                   "l2": f"inputs > L2: per-rank weights rotate over {copies} copies"},
        "e2e": {"value": round(e2e_val, 1), "unit": "GB/s",
                "h2d_bytes_per_step": sum(2 * m * shapes[nm][1] for nm, m in calls),
                "d2h_bytes_per_step": sum(2 * m * shapes[nm][0] for nm, m in calls),
                "path": "pinned H2D x, amsq_linear_tp, D2H y, sync per call"},
        "roofline": {"bound": "hbm", "achieved": round(per_rank_bytes * args.steps
                                                        / (total_ms * 1e-3) / 1e9, 1),
                     "peak": peak, "unit": "GB/s",
                     "frac": round(per_rank_bytes * args.steps / (total_ms * 1e-3) / 1e9 / peak, 4),
                     "traffic": None, "kernel": "per-rank shard bytes / step time (incl. all-gather)",
                     "peak_src": peak_kind},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "fused_tp": fused,
    }
    lib().amsq_nccl_comm_destroy(comm)
    return line


def _tp_fused_variant(args, sets, calls, xs, shapes, P, rank, local, stream, copies, full_bytes):
    """The same step through amsq_linear_tp_fused (K2 epilogue stores into every rank's arena
    over NVLink + device flag barrier; CUDA-IPC segments exchanged with all_gather_object).
    Reported beside the NCCL line; any failure is recorded, never fatal."""
    import ctypes as C

    import torch

    from paper_2510_16045_b200._lib import check, lib
    try:
        per_call = [2 * m * shapes[name][0] for name, m in calls]  # one arena region per call
        offs = np.concatenate([[0], np.cumsum(per_call)]).astype(np.int64)
        arena = int(offs[-1])
        h = (C.c_uint8 * 64)()
        tp = C.c_void_p()
        check(lib().amsq_tp_segment_create(P, rank, local, arena, h, C.byref(tp)), "tp_segment")
        allh = [None] * P
        torch.distributed.all_gather_object(allh, bytes(h))
        blob = (C.c_uint8 * (64 * P)).from_buffer_copy(b"".join(allh))
        check(lib().amsq_tp_attach(tp, blob), "tp_attach")

        def step(i):
            ws = sets[i % copies]
            for c, (name, m) in enumerate(calls):
                rc = lib().amsq_linear_tp_fused(ws[name].handle, tp, xs[(name, m)].data_ptr(), m,
                                                int(offs[c]), stream.cuda_stream)
                if rc:
                    raise RuntimeError(lib().amsq_last_error().decode())

        for i in range(args.warmup):
            step(i)
        torch.cuda.synchronize()
        torch.distributed.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for i in range(args.steps):
            step(i)
        b.record(stream)
        torch.cuda.synchronize()
        err = C.c_int(0)
        check(lib().amsq_tp_error(tp, C.byref(err)), "tp_error")
        ms = torch.tensor([a.elapsed_time(b)], device=f"cuda:{local}")
        torch.distributed.all_reduce(ms, op=torch.distributed.ReduceOp.MAX)
        lib().amsq_tp_destroy(tp)
        t = float(ms.item())
        return {"value": round(full_bytes * args.steps / (t * 1e-3) / 1e9, 1), "unit": "GB/s",
                "ms_per_step": round(t / args.steps, 4), "barrier_error": int(err.value)}
    except Exception as e:  # noqa: BLE001 -- reported, the NCCL line stands
        return {"error": f"{type(e).__name__}: {e}"[:200]}


# ------------------------------------------------------------------ extras (--extra FILE)
def _rotation(w, min_bytes=ROTATE_BYTES):
    n = max(2, int(np.ceil(min_bytes / w.payload_bytes)))
    return [w] + [w.clone() for _ in range(n - 1)]


def run_batch_sweep(args, dev, stream, cap):
    """Config 3: both schemes x 8B shapes x M in 1..256 (memory-bound -> tcgen05 crossover)."""
    import torch
    import torch.nn.functional as F

    import paper_2510_16045_b200 as amsq
    from paper_2510_16045_b200._lib import lib
    shapes = SHAPES_8B
    batches = [int(b) for b in args.sweep_batches.split(",")]
    peak, tpeak, _ = _peaks()
    out, cub = [], {}
    for name, (n, k) in shapes.items():
        nd = _n_copies(2 * n * k)
        dense = [torch.randn(n, k, device=dev).half() for _ in range(nd)]
        for m in batches:
            x = torch.randn(m, k, device=dev).half()
            cub[(name, m)] = _graph_us(lambda r, x=x: F.linear(x, dense[r % nd]), 2 * nd, 5,
                                       stream, cap)
        del dense
    torch.cuda.empty_cache()
    for scheme in ("fp5.33-e2m3", "fp4.25-e2m2"):
        for i, (name, (n, k)) in enumerate(shapes.items()):
            ws = _rotation(amsq.DeviceWeight(_qt(scheme, n, k, seed=500 + i), device=dev.index))
            pb = ws[0].payload_bytes
            for m in batches:
                x = torch.randn(m, k, device=dev).half()
                y = torch.empty(m, n, device=dev, dtype=torch.float16)
                us = _graph_us(lambda r, x=x, y=y, m=m: _lin(ws[r % len(ws)].handle, x, m, y,
                                                             cap.cuda_stream),
                               2 * len(ws), 5, stream, cap)
                flops = 2.0 * m * n * k
                out.append({"scheme": scheme, "layer": name, "M": m,
                            "kernel": "K3" if lib().amsq_linear_uses_tc(ws[0].scheme.id, m) else "K2",
                            "us": round(us, 2), "packed_GBps": round(pb / us / 1e3, 1),
                            "hbm_frac": round(algorithmic_bytes(pb, n, k, m) / us / 1e3 / peak, 3),
                            "TFLOPs": round(flops / us / 1e6, 1),
                            "tensor_frac": round(flops / us / 1e6 / tpeak, 3),
                            "cublas_fp16_us": round(cub[(name, m)], 2),
                            "speedup_vs_cublas": round(cub[(name, m)] / us, 2)})
            for w in ws:
                w.free()
    return out


def run_stack(args, dev, stream, cap):
    """Config 5: the 32-layer Llama-3.1-8B decode-step linear stack (128 linears, distinct
    weights in HBM) as ONE CUDA graph, FP5.33 vs FP4.25 vs FP16 cuBLAS, per batch."""
    import torch
    import torch.nn.functional as F

    import paper_2510_16045_b200 as amsq
    shapes = SHAPES_8B
    batches = [int(b) for b in args.stack_batches.split(",")]
    L = args.stack_layers
    res = {"layers": L, "linears": 4 * L}
    xs = {m: {name: torch.randn(m, k, device=dev).half() for name, (n, k) in shapes.items()}
          for m in batches}
    ys = {m: {name: torch.empty(m, n, device=dev, dtype=torch.float16)
              for name, (n, k) in shapes.items()} for m in batches}
    for scheme in ("fp5.33-e2m3", "fp4.25-e2m2"):
        base = {name: amsq.DeviceWeight(_qt(scheme, n, k, seed=900 + i), device=dev.index)
                for i, (name, (n, k)) in enumerate(shapes.items())}
        layers = [base] + [{name: w.clone() for name, w in base.items()} for _ in range(L - 1)]
        total = sum(w.payload_bytes for lay in layers for w in lay.values())
        per = {}
        for m in batches:
            def step(r, m=m):
                for lay in layers:
                    for name in shapes:
                        _lin(lay[name].handle, xs[m][name], m, ys[m][name], cap.cuda_stream)
            us = _graph_us(step, 1, 5, stream, cap)
            per[str(m)] = {"us": round(us, 1), "packed_GBps": round(total / us / 1e3, 1)}
        res[scheme] = {"weight_bytes": total, "per_batch": per}
        for lay in layers:
            for w in lay.values():
                w.free()
        torch.cuda.empty_cache()
    dense = [{name: torch.randn(n, k, device=dev).half() for name, (n, k) in shapes.items()}
             for _ in range(L)]
    per = {}
    for m in batches:
        def step16(r, m=m):
            for lay in dense:
                for name in shapes:
                    F.linear(xs[m][name], lay[name])
        per[str(m)] = {"us": round(_graph_us(step16, 1, 5, stream, cap), 1)}
    res["fp16-cublas"] = {"weight_bytes": sum(2 * n * k for n, k in shapes.values()) * L,
                          "per_batch": per}
    for scheme in ("fp5.33-e2m3", "fp4.25-e2m2"):
        for m in batches:
            res[scheme]["per_batch"][str(m)]["speedup_vs_cublas"] = round(
                per[str(m)]["us"] / res[scheme]["per_batch"][str(m)]["us"], 2)
    del dense
    torch.cuda.empty_cache()
    return res


def run_tp_shards(args, dev, stream, cap):
    """Config 4's per-rank kernels on one GPU: rows N/P of each 70B linear, P = 2/4/8."""
    import torch

    import paper_2510_16045_b200 as amsq
    out = []
    for scheme in ("fp5.33-e2m3", "fp4.25-e2m2"):
        for i, (name, (n, k)) in enumerate(SHAPES_70B.items()):
            for P in (2, 4, 8):
                rows = n // P
                ws = _rotation(amsq.DeviceWeight(_qt(scheme, rows, k, seed=700 + i), device=dev.index))
                pb = ws[0].payload_bytes
                for m in (1, 16):
                    x = torch.randn(m, k, device=dev).half()
                    y = torch.empty(m, rows, device=dev, dtype=torch.float16)
                    us = _graph_us(lambda r, x=x, y=y, m=m: _lin(ws[r % len(ws)].handle, x, m, y,
                                                                 cap.cuda_stream),
                                   2 * len(ws), 5, stream, cap)
                    out.append({"scheme": scheme, "layer": name, "P": P, "rows": rows, "M": m,
                                "us": round(us, 2), "packed_GBps": round(pb / us / 1e3, 1),
                                "allgather_bytes_per_rank": 2 * m * n * (P - 1) // P})
                for w in ws:
                    w.free()
    return out


# ------------------------------------------------------------------ CPU reference
def _ref_timings(scheme, shapes, batches, passes, warmup, per_call_median):
    """The reference's own amsq::gemv (oracle/_ref, -O2 -ffp-contract=off, all host threads)
    over every (shape, M) call of the step. Returns (payload bytes per pass, seconds per pass
    list or per-call medians, threads, kind)."""
    from oracle import COracle, load_ref

    ref = load_ref()
    sid = _BLOCK[scheme][0]
    calls = [(name, m) for m in batches for name in shapes]
    tensors = {name: make_stream(scheme, n, k, seed=17 + i)
               for i, (name, (n, k)) in enumerate(shapes.items())}
    xs = {(name, m): np.random.default_rng(m).standard_normal(m * shapes[name][1])
          .astype(np.float16).view(np.uint16) for name, m in calls}
    ys = {(name, m): np.zeros(m * shapes[name][0], np.uint16) for name, m in calls}
    if ref is not None:
        handles = {}
        for name, (pc, sc, pl) in tensors.items():
            n, k = shapes[name]
            handles[name] = ref.lib.ref_tensor_new(sid, n, k, pc, sc, pl, pl.size)
        threads = ref.lib.ref_resolve_threads(0)

        def call(name, m):
            rc = ref.lib.ref_tensor_gemv(handles[name], xs[(name, m)].ctypes.data, m, threads,
                                         ys[(name, m)].ctypes.data)
            if rc:
                raise RuntimeError("reference gemv failed")
        kind, cores = "reference", threads
        desc = f"reference amsq::gemv (oracle/_ref), threads={threads}"
    else:  # the plain-C restatement, one thread: bounded to the two small shapes
        orc = COracle()
        calls = [c for c in calls if c[0] in ("o", "qkv") and c[1] == 1]

        def call(name, m):
            n, k = shapes[name]
            pc, sc, pl = tensors[name]
            orc.gemv(sid, n, k, pc, sc, pl, xs[(name, m)], m)
        kind, cores, handles = "port", 1, {}
        desc = "C oracle port (amsq_oracle.c), 1 thread"
    pass_bytes = sum(payload_bytes_of(scheme, *shapes[name]) for name, m in calls)
    for _ in range(warmup):
        for c in calls:
            call(*c)
    if per_call_median:  # median_ns semantics per call (kernels.hpp:312-325)
        med = []
        for c in calls:
            ts = []
            for _ in range(passes):
                t = time.perf_counter()
                call(*c)
                ts.append(time.perf_counter() - t)
            med.append(statistics.median(ts))
        out = [sum(med)]
    else:
        out = []
        for _ in range(passes):
            t = time.perf_counter()
            for c in calls:
                call(*c)
            out.append(time.perf_counter() - t)
    if ref is not None:
        for h in handles.values():
            ref.lib.ref_tensor_free(h)
    return pass_bytes, out, cores, kind, desc, len(calls)


def cpu_baseline(args, shapes, batches):
    """Reported baseline on the box's host cores: 1 warm-up + median of 5 per call."""
    pb, t, cores, kind, desc, ncalls = _ref_timings(args.scheme, shapes, batches, passes=5,
                                                    warmup=1, per_call_median=True)
    return {"value": round(pb / t[0] / 1e9, 4), "unit": "GB/s", "cores": int(cores),
            "kind": kind, "host_cores": os.cpu_count(), "cpu": _cpu_model()[:60],
            "sample": f"{desc}: the step's {ncalls} calls, 1 warm-up + median of 5 each"}


def run_reference_arm(args, world, rank):
    """The reference's CPU amsq::gemv on the same workload, steps x warm-up as asked (rank 0
    only). Never imports paper_2510_16045_b200."""
    if rank != 0:
        return None
    shapes = SHAPES_8B if world == 1 else SHAPES_70B
    batches = [int(b) for b in args.batches.split(",")]
    pb, ts, cores, kind, desc, ncalls = _ref_timings(args.scheme, shapes, batches,
                                                     passes=args.steps, warmup=args.warmup,
                                                     per_call_median=False)
    total = sum(ts)
    value = pb * args.steps / total / 1e9
    wl = ("config 2: {s} linear, Llama-3.1-8B qkv/o/gate_up/down x batch {b} = {n} calls/step"
          if world == 1 else
          "config 4: {s} Llama-3.1-70B qkv/o/gate_up/down (full N: the CPU reference does not "
          "shard) x batch {b} = {n} calls/step")
    return {
        "impl": "reference", "metric": METRIC if world == 1 else METRIC_TP,
        "value": round(value, 4), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total / args.steps * 1e3, 2),
        "higher_is_better": True, "scaling": "weak" if world == 1 else "strong",
        "vs_baseline": None, "dtype": "fp16",
        "data": "synthetic: random valid packed streams, random fp16 x",
        "config": {"workload": wl.format(s=args.scheme, b=args.batches, n=ncalls),
                   "scheme": args.scheme, "parallelism": "host threads"},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": int(cores),
                         "kind": kind, "cpu": _cpu_model()[:60],
                         "sample": f"{desc}: every step = the workload's {ncalls} calls"},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def _emit(line):
    s = json.dumps(line, separators=(",", ":"))
    if len(s) > 1900:  # keep the headline parseable from a short stdout tail
        for k in ("cublas_fp16_us", "us_per_call"):
            line.pop(k, None)
        s = json.dumps(line, separators=(",", ":"))
    print(s, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scheme", default="fp5.33-e2m3", choices=sorted(_BLOCK))
    ap.add_argument("--batches", default="1,4,8,16")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--extra", default=None, metavar="FILE",
                    help="also run the batch sweep (config 3), the 32-layer stack (config 5) "
                         "and the per-rank 70B shard kernels; write them to FILE")
    ap.add_argument("--sweep-batches", default="1,2,4,8,16,32,64,128,256")
    ap.add_argument("--stack-batches", default="1,4,8,16")
    ap.add_argument("--stack-layers", type=int, default=32)
    args = ap.parse_args()
    world, rank, local = _dist()
    if args.impl == "reference":
        line = run_reference_arm(args, world, rank)
        if line is not None:
            _emit(line)
        return
    args.warmup = max(args.warmup, 3)
    import torch
    torch.cuda.set_device(local)
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        line = run_config4_tp(args, world, rank, local)
    else:
        line = run_config2(args, local)
    if rank == 0:
        _emit(line)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()

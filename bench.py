#!/usr/bin/env python
"""Benchmark of the B200 AMS-Quant fused linear (BASELINE.json config 2 by default).

A *step* is one pass over the Llama-3.1-8B layer linears (qkv 6144x4096, o 4096x4096,
gate_up 28672x4096, down 4096x14336) at every batch M in {1, 4, 8, 16}: 16 fused
restore+linear calls on FP5.33-e2m3 weights. ``value`` is packed-weight GB/s over the
timed region (sum of reference-stream payload bytes / device time), inputs resident in
HBM; ``e2e`` is the same metric through the C-ABI ``amsq_gemv_host`` with pinned host
buffers (H2D x and D2H y inside the timed region). Weights rotate across two copies
(>2x the 126 MB L2) so every call streams from HBM.

``--impl reference`` times the reference's own CPU ``amsq::gemv`` (oracle/_ref, all host
threads) on the same workload. Multi-GPU (torchrun): every rank runs the same workload on
its own GPU (replicas, weak scaling; the TP all-gather path is ``--tp``).
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
BATCHES = [1, 4, 8, 16]
L2_BYTES = 126 * 1024 * 1024


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops_sustained", 1375.8)), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
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
                "samples": len(sm), "window": "1 s of back-to-back step replays bracketing "
                                              "the timed region"}


# ------------------------------------------------------------------ workload data
def make_payload(sid, rows, cols, seed):
    """Random valid packed stream; FP5.33 padding codes zeroed."""
    import paper_2510_16045_b200 as amsq
    s = amsq.scheme_by_id(sid)
    rng = np.random.default_rng(seed)
    pc = amsq.round_up(cols, s.block)
    wpr = pc // s.block * s.words_per_block
    payload = rng.integers(0, 1 << 16, size=(rows, wpr), dtype=np.uint16)
    if pc > cols:  # padding columns restore to 0: clear their code segments (keep shared = 0)
        for c in range(cols, pc):
            blk, j = divmod(c, s.block)
            if sid == 7:
                payload[:, blk] &= np.uint16(~(0x1F << (5 * j)) & 0x7FFF)
            else:
                raise NotImplementedError
    scales = rng.uniform(0.002, 0.02, size=rows).astype(np.float16).view(np.uint16)
    return amsq.QuantizedTensor(s, rows, cols, pc, scales, payload.reshape(-1))


def algorithmic_bytes(payload_bytes, rows, cols, m):
    return payload_bytes + 2 * rows + 2 * m * cols + 2 * m * rows


# ------------------------------------------------------------------ GPU arm
def run_ours(args, world, rank, local):
    import torch
    import torch.nn.functional as F

    import paper_2510_16045_b200 as amsq
    from paper_2510_16045_b200._lib import lib

    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    sid = amsq.scheme_by_name(args.scheme).id
    shapes = SHAPES_8B if args.model == "8b" else SHAPES_70B
    batches = [int(b) for b in args.batches.split(",")]
    copies = args.copies
    # weights: `copies` independent sets so consecutive calls never hit L2
    sets = []
    for c in range(copies):
        ws = {}
        for i, (name, (n, k)) in enumerate(shapes.items()):
            qt = make_payload(sid, n, k, seed=1000 * c + i + 17 * rank)
            ws[name] = amsq.DeviceWeight(qt, device=local)
        sets.append(ws)
    payload_bytes = {name: sets[0][name].payload_bytes for name in shapes}
    xs = {(name, m): torch.randn(m, k, device=dev).half() for name, (n, k) in shapes.items()
          for m in batches}
    ys = {(name, m): torch.empty(m, n, device=dev, dtype=torch.float16)
          for name, (n, k) in shapes.items() for m in batches}
    calls = [(name, m) for m in batches for name in shapes]
    stream = torch.cuda.current_stream()

    def launch(ws, name, m, st):
        rc = lib().amsq_linear(ws[name].handle, xs[(name, m)].data_ptr(), m,
                               ys[(name, m)].data_ptr(), st)
        if rc:
            raise RuntimeError(lib().amsq_last_error().decode())

    # One step = the 16 calls, captured once per weight copy as a CUDA graph (the decode
    # step of a serving stack is graph-launched; launches are PDL-chained inside).
    cap = torch.cuda.Stream()
    cap.wait_stream(stream)
    graphs = []
    with torch.cuda.stream(cap):
        for c in range(copies):  # warm the per-function attributes outside capture
            for name, m in calls:
                launch(sets[c], name, m, cap.cuda_stream)
        cap.synchronize()
        per_step = None
        for c in range(copies):
            g = torch.cuda.CUDAGraph()
            l0 = amsq.kernel_launch_count()
            with torch.cuda.graph(g, stream=cap):
                for name, m in calls:
                    launch(sets[c], name, m, cap.cuda_stream)
            per_step = amsq.kernel_launch_count() - l0
            graphs.append(g)
    stream.wait_stream(cap)

    for i in range(args.warmup):
        graphs[i % copies].replay()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def busy(seconds):  # back-to-back replays so the clock samples see the loaded GPU
        end = time.time() + seconds
        i = 0
        while time.time() < end:
            for _ in range(20):
                graphs[i % copies].replay()
                i += 1
            torch.cuda.synchronize()

    with ClockSampler(local) as clk:
        busy(0.6)  # nvidia-smi needs ~0.1-0.3 s to start emitting samples
        torch.cuda.synchronize()
        t0.record(stream)
        for i in range(args.steps):
            graphs[i % copies].replay()
        t1.record(stream)
        busy(0.4)
        torch.cuda.synchronize()
    launches = per_step * args.steps
    total_ms = t0.elapsed_time(t1)
    if world > 1:
        tt = torch.tensor([total_ms], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(tt.item())
    bytes_per_step = sum(payload_bytes[name] for name, m in calls)
    value = world * bytes_per_step * args.steps / (total_ms * 1e-3) / 1e9

    # Per-call device time: a graph of R back-to-back calls of one (shape, M), weights
    # rotating over the copies, replayed; same for cuBLAS FP16 (F.linear -> cublasGemmEx).
    R = 4 * copies
    dense = [{name: torch.randn(n, k, device=dev).half() for name, (n, k) in shapes.items()}
             for _ in range(copies)]

    def graph_time(fn):
        with torch.cuda.stream(cap):
            fn(0)
            cap.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cap):
                for r in range(R):
                    fn(r)
        stream.wait_stream(cap)
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(3, args.steps)
        a.record(stream)
        for _ in range(reps):
            g.replay()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) * 1e3 / (reps * R)

    per_call, cub = {}, {}
    for name, m in calls:
        per_call[(name, m)] = graph_time(
            lambda r, name=name, m=m: launch(sets[r % copies], name, m, cap.cuda_stream))
        cub[(name, m)] = graph_time(
            lambda r, name=name, m=m: F.linear(xs[(name, m)], dense[r % copies][name]))
    del dense
    torch.cuda.empty_cache()

    peak, tpeak, peak_kind = _peaks()
    detail = []
    alg_total, t_total = 0.0, 0.0
    for name, m in calls:
        n, k = shapes[name]
        us = per_call[(name, m)]
        cub_us = cub[(name, m)]
        alg = algorithmic_bytes(payload_bytes[name], n, k, m)
        alg_total += alg
        t_total += us * 1e-6
        detail.append({"layer": name, "N": n, "K": k, "M": m, "us": round(us, 2),
                       "packed_GBps": round(payload_bytes[name] / us / 1e3, 1),
                       "alg_GBps": round(alg / us / 1e3, 1),
                       "frac_of_peak": round(alg / us / 1e3 / peak, 3),
                       "cublas_fp16_us": round(cub_us, 2),
                       "speedup_vs_cublas": round(cub_us / us, 2)})
    achieved = alg_total / t_total / 1e9

    # --- end to end through the C-ABI with pinned host buffers
    e2e = run_e2e(args, sets, shapes, calls, payload_bytes, dev, world)
    extra = {}
    if not args.no_extra and rank == 0:
        for c in sets:
            for w in c.values():
                w.free()
        torch.cuda.empty_cache()
        t = time.time()
        for key, fn in (("batch_sweep", lambda: run_batch_sweep(args, shapes, dev, stream, cap)),
                        ("stack_32L", lambda: run_stack(args, shapes, dev, stream, cap)),
                        ("tp_shards_70B", lambda: run_tp_shards(args, dev, stream, cap))):
            try:
                extra[key] = fn()
            except Exception as e:  # an extra section must not take the headline line down
                torch.cuda.synchronize()
                extra[key] = {"error": f"{type(e).__name__}: {e}"[:300]}
        extra["extra_seconds"] = round(time.time() - t, 1)

    # dram__bytes_read.sum + dram__bytes_write.sum of one ncu --set full capture of the
    # dominant launch (profiles/ncu_traffic.json), per launch, beside its algorithmic bytes
    traffic, traffic_note = None, None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        try:
            rec = json.load(open(tfile)).get(args.scheme)
            if rec:
                traffic = rec["traffic_bytes_per_launch"]
                traffic_note = (f"{rec['launch']}: dram {rec['traffic_bytes_per_launch']} B vs "
                                f"algorithmic {rec['algorithmic_bytes_per_launch']} B "
                                f"(ratio {rec['ratio']})")
        except Exception:
            traffic = None

    line = {
        "metric": "AMS linear packed-weight HBM GB/s (Llama-3.1-8B qkv/o/gate_up/down, "
                  "batch 1/4/8/16; per-call us and speedup vs FP16 cuBLAS in detail)",
        "value": round(value, 1), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp16",
        "data": "synthetic: random valid packed streams (FP5.33 padding zeroed), random fp16 x",
        "config": {"workload": f"{args.scheme} linear, Llama-3.1-{args.model.upper()} layer "
                               f"shapes x batch {args.batches}, 1 step = {len(calls)} calls",
                   "scheme": args.scheme, "shapes": {k: list(v) for k, v in shapes.items()},
                   "batches": batches,
                   "l2": f"weights rotated over {copies} copies "
                         f"({copies * sum(payload_bytes.values()) / 1e6:.0f} MB > 126 MB L2)",
                   "parallelism": f"replicas x{world}"},
        "e2e": e2e,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "traffic_note": traffic_note,
                     "kernel": "amsq_linear_kernel", "peak_kind": peak_kind,
                     "bytes": "algorithmic = packed_payload_bytes + 2N + 2MK + 2MN per call"},
        "gpu_launches": int(launches),
        "timing": "device time of CUDA-graph replays (16 PDL-chained calls per step); per-call "
                  "detail from graphs of back-to-back calls of one shape",
        "clocks": clk.summary(),
        "detail": detail,
    }
    line.update(extra)
    if rank == 0 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args, shapes, batches, sid, sample_only=True)
    return line


def _graph_us(fn, reps_in_graph, replays, stream, cap):
    """Device time per call of `fn(r)` captured reps_in_graph times in one CUDA graph."""
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


def _rotation(w, min_bytes=260e6):
    """w plus device clones so a rotation over them streams > 2x the 126 MB L2."""
    n = max(2, int(np.ceil(min_bytes / w.payload_bytes)))
    return [w] + [w.clone() for _ in range(n - 1)]


def run_batch_sweep(args, shapes, dev, stream, cap):
    """Config 3: both schemes x 8B shapes x M in 1..256 (memory-bound -> tcgen05 crossover)."""
    import torch
    import torch.nn.functional as F

    import paper_2510_16045_b200 as amsq
    from paper_2510_16045_b200._lib import lib
    batches = [int(b) for b in args.sweep_batches.split(",")]
    peak, tpeak, _ = _peaks()
    out = []
    dense = {name: [torch.randn(n, k, device=dev).half() for _ in range(2)]
             for name, (n, k) in shapes.items()}
    cub = {}
    for name, (n, k) in shapes.items():
        for m in batches:
            x = torch.randn(m, k, device=dev).half()
            cub[(name, m)] = _graph_us(lambda r, x=x, name=name: F.linear(x, dense[name][r % 2]),
                                       8, 5, stream, cap)
    del dense
    torch.cuda.empty_cache()
    k3_min = lib().amsq_debug_set_k3_min_batch(0)  # the library's K2 / K3 dispatch threshold
    for scheme in ("fp5.33-e2m3", "fp4.25-e2m2"):
        sid = amsq.scheme_by_name(scheme).id
        for i, (name, (n, k)) in enumerate(shapes.items()):
            ws = _rotation(amsq.DeviceWeight(make_payload(sid, n, k, seed=500 + i), device=dev.index))
            pb = ws[0].payload_bytes
            for m in batches:
                x = torch.randn(m, k, device=dev).half()
                y = torch.empty(m, n, device=dev, dtype=torch.float16)

                def call(r, x=x, y=y, m=m):
                    rc = lib().amsq_linear(ws[r % len(ws)].handle, x.data_ptr(), m, y.data_ptr(),
                                           cap.cuda_stream)
                    if rc:
                        raise RuntimeError(lib().amsq_last_error().decode())
                us = _graph_us(call, 2 * len(ws), 5, stream, cap)
                flops = 2.0 * m * n * k
                out.append({"scheme": scheme, "layer": name, "N": n, "K": k, "M": m,
                            "kernel": ("K3 tcgen05" if m >= k3_min else
                                       "K2 mma.sync" if m <= 32 else "K2 mma.sync x%d" % -(-m // 32)),
                            "us": round(us, 2), "packed_GBps": round(pb / us / 1e3, 1),
                            "hbm_frac": round(algorithmic_bytes(pb, n, k, m) / us / 1e3 / peak, 3),
                            "TFLOPs": round(flops / us / 1e6, 1),
                            "tensor_frac": round(flops / us / 1e6 / tpeak, 3),
                            "cublas_fp16_us": round(cub[(name, m)], 2),
                            "speedup_vs_cublas": round(cub[(name, m)] / us, 2)})
            for w in ws:
                w.free()
    return out


def run_stack(args, shapes, dev, stream, cap):
    """Config 5: the 32-layer Llama-3.1-8B decode-step linear stack (qkv, o, gate_up, down per
    layer = 128 linears, distinct weights in HBM) as ONE CUDA graph, FP5.33 vs FP4.25 vs FP16
    cuBLAS, per batch."""
    import torch
    import torch.nn.functional as F

    import paper_2510_16045_b200 as amsq
    from paper_2510_16045_b200._lib import lib
    batches = [int(b) for b in args.stack_batches.split(",")]
    L = args.stack_layers
    res = {"layers": L, "linears": 4 * L, "batches": batches}
    xs = {m: {name: torch.randn(m, k, device=dev).half() for name, (n, k) in shapes.items()}
          for m in batches}
    ys = {m: {name: torch.empty(m, n, device=dev, dtype=torch.float16)
              for name, (n, k) in shapes.items()} for m in batches}
    for scheme in ("fp5.33-e2m3", "fp4.25-e2m2"):
        sid = amsq.scheme_by_name(scheme).id
        base = {name: amsq.DeviceWeight(make_payload(sid, n, k, seed=900 + i), device=dev.index)
                for i, (name, (n, k)) in enumerate(shapes.items())}
        layers = [base] + [{name: w.clone() for name, w in base.items()} for _ in range(L - 1)]
        total_bytes = sum(w.payload_bytes for lay in layers for w in lay.values())
        per = {}
        for m in batches:
            def step(r, m=m):
                for lay in layers:
                    for name in shapes:
                        rc = lib().amsq_linear(lay[name].handle, xs[m][name].data_ptr(), m,
                                               ys[m][name].data_ptr(), cap.cuda_stream)
                        if rc:
                            raise RuntimeError(lib().amsq_last_error().decode())
            us = _graph_us(step, 1, 5, stream, cap)
            per[str(m)] = {"us": round(us, 1), "packed_GBps": round(total_bytes / us / 1e3, 1)}
        res[scheme] = {"weight_bytes": total_bytes, "per_batch": per}
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
                    F.linear(xs[m][name], lay[name], out=None)
        us = _graph_us(step16, 1, 5, stream, cap)
        per[str(m)] = {"us": round(us, 1)}
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
    """Config 4 on one GPU: the per-rank share of the N-sharded Llama-3.1-70B linears at
    P = 2/4/8 (rows N/P, full K). The NCCL all-gather itself needs P GPUs (not timed here)."""
    import torch

    import paper_2510_16045_b200 as amsq
    from paper_2510_16045_b200._lib import lib
    out = []
    for scheme in ("fp5.33-e2m3", "fp4.25-e2m2"):
        sid = amsq.scheme_by_name(scheme).id
        for i, (name, (n, k)) in enumerate(SHAPES_70B.items()):
            for P in (2, 4, 8):
                rows = n // P
                ws = _rotation(amsq.DeviceWeight(make_payload(sid, rows, k, seed=700 + i), device=dev.index))
                pb = ws[0].payload_bytes
                for m in (1, 16):
                    x = torch.randn(m, k, device=dev).half()
                    y = torch.empty(m, rows, device=dev, dtype=torch.float16)

                    def call(r, x=x, y=y, m=m):
                        rc = lib().amsq_linear(ws[r % len(ws)].handle, x.data_ptr(), m,
                                               y.data_ptr(), cap.cuda_stream)
                        if rc:
                            raise RuntimeError(lib().amsq_last_error().decode())
                    us = _graph_us(call, 2 * len(ws), 5, stream, cap)
                    out.append({"scheme": scheme, "layer": name, "P": P, "rows_per_rank": rows,
                                "K": k, "M": m, "us": round(us, 2),
                                "packed_GBps_per_rank": round(pb / us / 1e3, 1),
                                "allgather_bytes_per_rank": 2 * m * n * (P - 1) // P})
                for w in ws:
                    w.free()
    return out


def run_e2e(args, sets, shapes, calls, payload_bytes, dev, world):
    import torch

    from paper_2510_16045_b200._lib import lib

    stream = torch.cuda.current_stream()
    hx = {(name, m): torch.randn(m, shapes[name][1]).half().pin_memory() for name, m in calls}
    hy = {(name, m): torch.empty(m, shapes[name][0], dtype=torch.float16).pin_memory()
          for name, m in calls}
    h2d = sum(2 * m * shapes[name][1] for name, m in calls)
    d2h = sum(2 * m * shapes[name][0] for name, m in calls)
    steps = max(2, args.steps // 2)

    def one(i):
        ws = sets[i % len(sets)]
        for name, m in calls:
            rc = lib().amsq_gemv_host(ws[name].handle, hx[(name, m)].data_ptr(),
                                      m * shapes[name][1], m, hy[(name, m)].data_ptr(),
                                      stream.cuda_stream)
            if rc:
                raise RuntimeError(lib().amsq_last_error().decode())

    for i in range(2):
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
    val = world * sum(payload_bytes[n] for n, m in calls) * steps / (ms * 1e-3) / 1e9
    return {"value": round(val, 1), "unit": "GB/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": round(ms / steps, 4),
            "path": "amsq_gemv_host (pinned host x/y, H2D + kernel + D2H per call)"}


# ------------------------------------------------------------------ CPU reference arm
def cpu_baseline(args, shapes, batches, sid, sample_only=True, steps=1, warmup=0):
    """The reference's own amsq::gemv (oracle/_ref) on all host threads; falls back to the
    plain-C oracle port (1 thread) when the reference was never compiled."""
    from oracle import COracle, load_ref

    ref = load_ref()
    cores = os.cpu_count() or 1
    kind = "reference" if ref is not None else "port"
    calls = [(name, m) for m in batches for name in shapes]
    if kind == "port":  # single-threaded C port: keep the sample bounded
        calls = [("o", 1), ("qkv", 1)]
    tensors = {}
    for i, name in enumerate(shapes):
        if any(c[0] == name for c in calls):
            n, k = shapes[name]
            tensors[name] = make_payload(sid, n, k, seed=i + 17)
    total_bytes, total_s = 0, 0.0
    if kind == "reference":
        import ctypes as C
        handles = {}
        for name, qt in tensors.items():
            handles[name] = ref.lib.ref_tensor_new(sid, qt.rows, qt.cols, qt.padded_cols,
                                                   qt.scales, qt.payload, qt.payload.size)
        threads = ref.lib.ref_resolve_threads(0)
        for it in range(warmup + steps):
            for name, m in calls:
                n, k = shapes[name]
                x = np.random.default_rng(m).standard_normal(m * k).astype(np.float16).view(np.uint16)
                y = np.zeros(m * n, np.uint16)
                t = time.perf_counter()
                rc = ref.lib.ref_tensor_gemv(handles[name], x.ctypes.data, m, threads, y.ctypes.data)
                dt = time.perf_counter() - t
                if rc:
                    raise RuntimeError("reference gemv failed")
                if it >= warmup:
                    total_bytes += tensors[name].payload.size * 2
                    total_s += dt
        for h in handles.values():
            ref.lib.ref_tensor_free(h)
        cores_used = threads
        sample = (f"reference amsq::gemv (oracle/_ref, -O2 -ffp-contract=off), {len(calls)} calls "
                  f"x {steps} pass(es): all layer shapes x batch {batches}, threads={threads}")
    else:
        orc = COracle()
        for it in range(warmup + steps):
            for name, m in calls:
                qt = tensors[name]
                x = np.random.default_rng(m).standard_normal(m * qt.cols).astype(np.float16).view(np.uint16)
                t = time.perf_counter()
                orc.gemv(sid, qt.rows, qt.cols, qt.padded_cols, qt.scales, qt.payload, x, m)
                dt = time.perf_counter() - t
                if it >= warmup:
                    total_bytes += qt.payload.size * 2
                    total_s += dt
        cores_used = 1
        sample = f"C oracle port, 1 thread, calls {calls}"
    value = total_bytes / total_s / 1e9
    return {"value": round(value, 4), "unit": "GB/s", "cores": int(cores_used),
            "host_cores": cores, "kind": kind, "sample": sample,
            "seconds": round(total_s, 2)}


def run_reference_arm(args, world, rank):
    import paper_2510_16045_b200 as amsq  # scheme table only (host)

    if rank != 0:
        return None
    sid = amsq.scheme_by_name(args.scheme).id
    shapes = SHAPES_8B if args.model == "8b" else SHAPES_70B
    batches = [int(b) for b in args.batches.split(",")]
    steps = max(1, min(args.steps, 3))
    warm = 1 if args.warmup > 0 else 0
    cb = cpu_baseline(args, shapes, batches, sid, steps=steps, warmup=warm)
    n_calls = len(batches) * len(shapes)
    return {
        "impl": "reference",
        "metric": "AMS linear packed-weight HBM GB/s (Llama-3.1-8B qkv/o/gate_up/down, "
                  "batch 1/4/8/16; per-call us and speedup vs FP16 cuBLAS in detail)",
        "value": cb["value"], "unit": "GB/s", "n_gpus": world, "steps": steps,
        "warmup": warm, "ms_per_step": round(cb["seconds"] / steps * 1e3, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp16",
        "data": "synthetic: random valid packed streams, random fp16 x",
        "config": {"workload": f"{args.scheme} linear, Llama-3.1-{args.model.upper()} layer "
                               f"shapes x batch {args.batches}, 1 step = {n_calls} calls",
                   "scheme": args.scheme, "batches": batches},
        "cpu_baseline": cb,
        "e2e": {"value": cb["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scheme", default="fp5.33-e2m3")
    ap.add_argument("--model", default="8b", choices=["8b", "70b"])
    ap.add_argument("--batches", default="1,4,8,16")
    ap.add_argument("--copies", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the batch sweep (config 3), 32-layer stack (config 5), TP shards")
    ap.add_argument("--sweep-batches", default="1,2,4,8,16,32,64,128,256")
    ap.add_argument("--stack-batches", default="1,4,8,16")
    ap.add_argument("--stack-layers", type=int, default=32)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    world, rank, local = _dist()
    if args.impl == "reference":
        line = run_reference_arm(args, world, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    if world > 1:
        import torch
        torch.distributed.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    line = run_ours(args, world, rank, local)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()

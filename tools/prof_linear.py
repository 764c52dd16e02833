#!/usr/bin/env python
"""Profiling driver: run the fused linear (and optionally cuBLAS FP16) on one shape.

Used under ncu on the GPU box, e.g.
  ncu --set full -k regex:amsq_linear -s 4 -c 2 -o gpurun_out/prof python tools/prof_linear.py \
      --scheme fp5.33-e2m3 --n 28672 --k 4096 --m 1
Also prints CUDA-graph timings (no CPU launch gaps) when run without ncu.
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2510_16045_b200 as amsq  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scheme", default="fp5.33-e2m3")
    ap.add_argument("--n", type=int, default=28672)
    ap.add_argument("--k", type=int, default=4096)
    ap.add_argument("--m", type=int, default=1)
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--cublas", action="store_true")
    ap.add_argument("--graph", action="store_true")
    ap.add_argument("--empty", action="store_true", help="time an empty kernel per call")
    ap.add_argument("--k3min", type=int, default=0, help="K3 dispatch threshold (0: default)")
    args = ap.parse_args()
    if args.k3min > 0:
        from paper_2510_16045_b200._lib import lib
        lib().amsq_debug_set_k3_min_batch(args.k3min)
    sid = amsq.scheme_by_name(args.scheme).id
    copies = max(2, int(np.ceil(260e6 / amsq.packed_payload_bytes(sid, args.n, args.k))))
    ws = [amsq.DeviceWeight(bench._qt(args.scheme, args.n, args.k, seed=c)) for c in range(copies)]
    x = torch.randn(args.m, args.k, device="cuda").half()
    y = torch.empty(args.m, args.n, device="cuda", dtype=torch.float16)
    for i in range(args.iters):
        ws[i % copies].linear(x, out=y)
    if args.cublas:
        dense = [torch.randn(args.n, args.k, device="cuda").half() for _ in range(2)]
        for i in range(args.iters):
            torch.nn.functional.linear(x, dense[i % 2])
    torch.cuda.synchronize()
    if args.graph:
        reps = 4 * copies
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(reps):
                ws[i % copies].linear(x, out=y)
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with bench.ClockSampler(0) as clk:
            a.record()
            for _ in range(200):
                g.replay()
            b.record()
            torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / (200 * reps)
        pb = ws[0].payload_bytes
        print(f"graph: {args.scheme} N={args.n} K={args.k} M={args.m}: {us:.2f} us/call, "
              f"{pb / us / 1e3:.0f} GB/s packed  clocks={clk.summary()}")


if __name__ == "__main__":
    main()

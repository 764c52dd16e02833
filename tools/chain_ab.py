#!/usr/bin/env python
"""A/B of amsq_linear vs amsq_linear_chain (successor L2 prefetch) on the config-2 step
(16 calls as one CUDA graph, weights rotating > 2x L2) and the 32-layer stack."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2510_16045_b200 as amsq  # noqa: E402
from paper_2510_16045_b200._lib import lib  # noqa: E402


def graph_ms(fn, reps=30):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn(s)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn(s)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main(scheme="fp5.33-e2m3", layers=32):
    shapes = bench.SHAPES_8B
    for pf in (65536, 32768, 131072):
        lib().amsq_debug_set_chain_prefetch(pf)
        for M in (1, 8, 16):
            ws = [{n: amsq.DeviceWeight(bench._qt(scheme, r, c, seed=100 * l + i))
                   for i, (n, (r, c)) in enumerate(shapes.items())} for l in range(4)]
            seq = [(l, n) for l in range(4) for n in shapes]  # 16 calls, distinct weights
            xs = {n: torch.randn(M, c, device="cuda").half() for n, (r, c) in shapes.items()}
            ys = {n: torch.empty(M, r, device="cuda", dtype=torch.float16) for n, (r, c) in shapes.items()}

            def run(s, chain):
                for i, (l, n) in enumerate(seq):
                    nl, nn = seq[(i + 1) % len(seq)]
                    nxt = ws[nl][nn].handle if chain else None
                    rc = lib().amsq_linear_chain(ws[l][n].handle, xs[n].data_ptr(), M,
                                                 ys[n].data_ptr(), nxt, s.cuda_stream)
                    assert rc == 0, lib().amsq_last_error()
            t0 = min(graph_ms(lambda s: run(s, False)) for _ in range(3))
            t1 = min(graph_ms(lambda s: run(s, True)) for _ in range(3))
            tot = sum(ws[l][n].payload_bytes for l, n in seq)
            print(f"{scheme} pf={pf} M={M}: plain {t0*1e3:.1f} us ({tot/t0/1e6:.0f} GB/s)  chain "
                  f"{t1*1e3:.1f} us ({tot/t1/1e6:.0f} GB/s)  ratio {t1/t0:.3f}", flush=True)
            for d in ws:
                for w in d.values():
                    w.free()


if __name__ == "__main__":
    main(*(sys.argv[1:2] or []))

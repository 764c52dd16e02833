#!/usr/bin/env python
"""Per-CTA timeline of one K3 (tcgen05) launch: start, per-stage A ready (decode warp 0) and
MMA commits, epilogue start/end (globaltimer, us from the first CTA start)."""
import argparse, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa
import paper_2510_16045_b200 as amsq  # noqa
from paper_2510_16045_b200._lib import lib  # noqa
ap = argparse.ArgumentParser()
ap.add_argument("--scheme", default="fp5.33-e2m3"); ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--k", type=int, default=4096); ap.add_argument("--m", type=int, default=32)
a = ap.parse_args()
sid = amsq.scheme_by_name(a.scheme).id
ws = [amsq.DeviceWeight(bench._qt(a.scheme, a.n, a.k, seed=c)) for c in range(3)]
x = torch.randn(a.m, a.k, device="cuda").half(); y = torch.empty(a.m, a.n, device="cuda", dtype=torch.float16)
tr = torch.zeros(1024 * 64, dtype=torch.int64, device="cuda")
for i in range(6): ws[i % 3].linear(x, out=y)
torch.cuda.synchronize()
lib().amsq_debug_set_trace(tr.data_ptr()); ws[0].linear(x, out=y); torch.cuda.synchronize()
lib().amsq_debug_set_trace(None)
t = tr.view(1024, 64).cpu().numpy().astype(np.float64)
n = int((t[:, 0] > 0).sum()); t = t[:n]; t0 = t[:, 0].min()
r = lambda v: (v - t0) / 1e3
print(f"{a.scheme} N={a.n} K={a.k} M={a.m}: ctas={n}")
for name, i in (("start", 0), ("epilogue", 2), ("end", 3)):
    v = r(t[:, i]); print(f"  {name:9s} min {v.min():6.2f} med {np.median(v):6.2f} max {v.max():6.2f}")
us = lambda c, v: (v - t[c, 1]) / 1965.0  # clock64 cycles -> us at the max SM clock
rows = (("producer loop top", 8), ("producer issued", 16), ("w0 landed", 24), ("w0 A ready", 32),
        ("w15 A ready", 56), ("MMA ready", 40), ("MMA issued", 48))
for c in (0, n // 2):
    print(f"  CTA {c} (us from CTA start, clock64):")
    for name, base in rows:
        v = [us(c, t[c, base + s]) for s in range(8) if t[c, base + s] > 0]
        print(f"    {name:18s}", " ".join(f"{x:6.2f}" for x in v))

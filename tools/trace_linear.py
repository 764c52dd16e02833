#!/usr/bin/env python
"""Per-CTA timeline of one fused-linear launch (globaltimer stamps via amsq_debug_set_trace)."""
import argparse, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa
import paper_2510_16045_b200 as amsq  # noqa
from paper_2510_16045_b200._lib import lib  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--scheme", default="fp5.33-e2m3"); ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--k", type=int, default=4096); ap.add_argument("--m", type=int, default=1)
a = ap.parse_args()
sid = amsq.scheme_by_name(a.scheme).id
ws = [amsq.DeviceWeight(bench._qt(a.scheme, a.n, a.k, seed=c)) for c in range(3)]
x = torch.randn(a.m, a.k, device="cuda").half(); y = torch.empty(a.m, a.n, device="cuda", dtype=torch.float16)
tr = torch.zeros(1024 * 64, dtype=torch.int64, device="cuda")
for i in range(6): ws[i % 3].linear(x, out=y)
torch.cuda.synchronize()
lib().amsq_debug_set_trace(tr.data_ptr())
ws[0].linear(x, out=y); torch.cuda.synchronize()
lib().amsq_debug_set_trace(None)
info = ws[0].info()
t = tr.view(1024, 64).cpu().numpy().astype(np.float64)
nct = int((t[:, 0] > 0).sum())
t = t[:nct]
t0 = t[:, 0].min()
rel = lambda v: (v - t0) / 1e3
st, first, loop, end = [rel(t[:, i]) for i in range(4)]
def q(v): return f"min {v.min():6.2f} med {np.median(v):6.2f} max {v.max():6.2f}"
print(f"{a.scheme} N={a.n} K={a.k} M={a.m} ctas={len(t)} plan=(groups {info.n_groups}, G {info.g_big}, "
      f"big {info.n_big}, csplit {info.csplit}) (us from first CTA start)")
print("  start      ", q(st)); print("  first stage", q(first)); print("  stream done", q(loop)); print("  end        ", q(end))
print("  first-stage latency per CTA", q(first - st), " epilogue per CTA", q(end - loop))
GHZ = 1.9  # SM clock under this load (clocks.sm ~1965 MHz); stamps 4.. are clock64
clk = lambda c, v: st[c] + (v - t[c, 63]) / GHZ / 1e3
print("  producer: after pdl_wait (CTA 0):", f"{clk(0, t[0, 4]):.2f}")
for c in (0, len(t) // 2):
    land = [clk(c, t[c, 8 + s]) for s in range(24) if t[c, 8 + s] > 0]
    iss = [clk(c, t[c, 32 + s]) for s in range(24) if t[c, 32 + s] > 0]
    last = [clk(c, t[c, 56 + s]) for s in range(7) if t[c, 56 + s] > 0]
    print(f"  CTA {c}: start {st[c]:.2f}")
    print("    x issued :", " ".join(f"{v:.2f}" for v in iss))
    print("    landed   :", " ".join(f"{v:.2f}" for v in land))
    print("    last warp done:", " ".join(f"{v:.2f}" for v in last))

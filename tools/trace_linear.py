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
ap.add_argument("--dry", action="store_true")
a = ap.parse_args()
sid = amsq.scheme_by_name(a.scheme).id
lib().amsq_debug_set_dry_run(1 if a.dry else 0)
ws = [amsq.DeviceWeight(bench.make_payload(sid, a.n, a.k, seed=c)) for c in range(3)]
x = torch.randn(a.m, a.k, device="cuda").half(); y = torch.empty(a.m, a.n, device="cuda", dtype=torch.float16)
tr = torch.zeros(1024 * 8, dtype=torch.int64, device="cuda")
for i in range(6): ws[i % 3].linear(x, out=y)
torch.cuda.synchronize()
lib().amsq_debug_set_trace(tr.data_ptr())
ws[0].linear(x, out=y); torch.cuda.synchronize()
lib().amsq_debug_set_trace(None)
t = tr.view(1024, 8).cpu().numpy().astype(np.float64)
nct = int((t[:, 0] > 0).sum())
t = t[:nct]
t0 = t[:, 0].min()
st, first, loop, end = [(t[:, i] - t0) / 1e3 for i in range(4)]
def q(v): return f"min {v.min():6.2f} med {np.median(v):6.2f} max {v.max():6.2f}"
print(f"{a.scheme} N={a.n} K={a.k} M={a.m} dry={a.dry} ctas={len(t)} (us from first CTA start)")
print("  start      ", q(st)); print("  first stage", q(first)); print("  stream done", q(loop)); print("  end        ", q(end))
print("  first-stage latency per CTA", q(first - st), " fixup per CTA", q(end - loop))

slots = np.arange(len(t)) // 148
for sl in range(slots.max() + 1):
    sel = slots == sl
    print(f"  CTA slot {sl} (blockIdx {sl*148}..): stream done", q(loop[sel]), " end", q(end[sel]))

"""compute-sanitizer driver (racecheck / synccheck / memcheck): one launch of each K2/K3
synchronisation class -- C=1, C=2 and C=8 cluster reductions, the M<=16 xprep path, the
M<=32 NB=4 path and a K3 (tcgen05) launch with a 2-CTA split -- each checked against the
oracle so a silent corruption under the tool also fails.

  compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import paper_2510_16045_b200 as amsq  # noqa: E402
from helpers import check_linear, gaussian_x, random_payload  # noqa: E402
from oracle import COracle  # noqa: E402
from paper_2510_16045_b200._lib import lib  # noqa: E402

CASES = [  # (scheme, rows, cols, batch, k3)
    (7, 512, 1000, 1, False),      # C=1, natural-row activations
    (4, 4096, 14336, 4, False),    # C=2 cluster reduction
    (4, 1280, 8192, 1, False),     # C=8 cluster reduction
    (7, 2560, 8192, 12, False),    # C=4, xprep (M <= 16)
    (7, 1024, 2049, 32, False),    # NB=4 (M <= 32)
    (4, 512, 2048, 48, True),      # K3 tcgen05, 2-CTA split-K
    (7, 1024, 4096, 5, True),      # K3 with one 16-column N chunk (A in TMEM, M < 16)
    (7, 2048, 2048, 128, True),    # K3 C=1, 8 N chunks
    (7, 4096, 4096, 64, "pair"),   # K3 CTA pair (cta_group::2, M = 256), forced
]


def main():
    only = [int(a) for a in sys.argv[1:]] or range(len(CASES))
    orc = COracle()
    for i in only:
        sid, rows, cols, batch, k3 = CASES[i]
        prev = lib().amsq_debug_set_k3_min_batch(1 if k3 else 100000)
        prev_pair = lib().amsq_debug_set_k3_pair(1 if k3 == "pair" else -1)
        qt = random_payload(sid, rows, cols, seed=i)
        dw = amsq.DeviceWeight(qt)
        x = gaussian_x(batch, cols, seed=i)
        xt = torch.from_numpy(x.view(np.float16).reshape(batch, cols)).cuda()
        y = dw.linear(xt).cpu().numpy().view(np.uint16).reshape(batch, rows)
        yref = orc.gemv(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
        _, yabs = orc.gemv_f64(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
        rel = check_linear(y, yref, yabs)
        lib().amsq_debug_set_k3_min_batch(prev)
        lib().amsq_debug_set_k3_pair(prev_pair)
        info = dw.info()
        print(f"case {i}: scheme {sid} {rows}x{cols} M={batch} {'K3 pair' if k3 == 'pair' else 'K3' if k3 else 'K2'} "
              f"plan G={info.g_big} C={info.csplit}: rel {rel:.2e} OK", flush=True)
        dw.free()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Summarise tools/gpu_ab.sh output: per case, the min over repeats of each library's us/call."""
import collections, sys
rows = collections.defaultdict(dict)
libs = []
for line in open(sys.argv[1]):
    p = line.split()
    if len(p) < 6:
        continue
    key = " ".join(p[1:4])
    lib = p[4]
    if lib not in libs:
        libs.append(lib)
    try:
        v = float(p[5])
    except ValueError:
        continue
    rows[key][lib] = min(v, rows[key].get(lib, 1e9))
print("case".ljust(36) + "".join(l[8:-3].rjust(12) for l in libs) + "   new/base")
tb = tn = 0.0
for key, d in rows.items():
    vals = [d.get(l, float("nan")) for l in libs]
    r = vals[1] / vals[0] if len(vals) > 1 and vals[0] else float("nan")
    tb += vals[0]; tn += vals[1] if len(vals) > 1 else 0
    print(key.ljust(36) + "".join(f"{v:12.2f}" for v in vals) + f"   {r:6.3f}")
print(f"sum base {tb:.1f} us, new {tn:.1f} us, ratio {tn / tb:.3f}")

#!/usr/bin/env python
"""Summarise an ncu source page (--page source --csv --print-source sass): executed warp
instructions and stall samples per opcode, and per address range (hot regions)."""
import collections
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    col = {h: i for i, h in enumerate(hdr)}
    data = []
    for r in rows[hdr_i + 1:]:
        if len(r) < len(hdr) or not r[0].startswith("0x"):
            continue
        data.append(r)
    base = int(data[0][0], 16)
    ops = collections.Counter()
    samp = collections.Counter()
    tot_i = tot_s = 0
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    stalls = collections.Counter()
    regions = []
    for r in data:
        addr = int(r[0], 16) - base
        src = r[col["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        n = int(r[col["Instructions Executed"]] or 0)
        s = int(r[col["Warp Stall Sampling (All Samples)"]] or 0)
        ops[op] += n
        samp[op] += s
        tot_i += n
        tot_s += s
        for h in stall_cols:
            stalls[h] += int(r[col[h]] or 0)
        regions.append((addr, n, s, src))
    print(f"total warp instructions {tot_i}, stall samples {tot_s}")
    print(f"{'opcode':12s} {'instr':>12s} {'%':>6s} {'samples':>8s} {'%':>6s}")
    for op, n in ops.most_common(top):
        print(f"{op:12s} {n:12d} {100*n/tot_i:6.2f} {samp[op]:8d} {100*samp[op]/max(1,tot_s):6.2f}")
    print("stall reasons:")
    for h, v in stalls.most_common(15):
        print(f"  {h:28s} {v:8d} {100*v/max(1,tot_s):6.2f}")
    # contiguous hot regions: windows of 64 instructions
    print("by 0x400-byte window (instr, samples):")
    win = collections.defaultdict(lambda: [0, 0])
    for addr, n, s, _ in regions:
        win[addr // 0x400][0] += n
        win[addr // 0x400][1] += s
    for w in sorted(win):
        n, s = win[w]
        if n > 0.005 * tot_i or s > 0.005 * tot_s:
            print(f"  0x{w*0x400:05x}: {n:10d} ({100*n/tot_i:5.1f}%)  {s:6d} ({100*s/max(1,tot_s):5.1f}%)")


if __name__ == "__main__":
    main(sys.argv[1])

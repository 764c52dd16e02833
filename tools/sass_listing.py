#!/usr/bin/env python
"""Dump the SASS of the product kernels (cuobjdump -sass) into profiles/<round>/sass/ with an
opcode histogram per kernel: the evidence that K2 issues HMMA + TMA bulk (UBLKCP) and K3
issues tcgen05 (UTCHMMA / STTM = tcgen05.st of the decoded A operand / LDTM / UTCBAR / UTCATOMSWS)
and cluster DSMEM traffic."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2510_16045_b200", "libamsq_b200.so")
OUT = os.path.join(ROOT, "profiles", sys.argv[1] if len(sys.argv) > 1 else "r01", "sass")
KEEP = ["amsq_linear_kernelILi7ELi1ELi1E", "amsq_linear_kernelILi7ELi1ELi2E",
        "amsq_linear_kernelILi4ELi1ELi2E", "amsq_linear_kernelILi7ELi2ELi2E",
        "amsq_linear_kernelILi7ELi4ELi1E",
        "amsq_linear_tc_kernelILi7ELi4E", "amsq_linear_tc_kernelILi7ELi0E", "amsq_linear_tc_kernelILi7ELi1E",
        "amsq_linear_tc_kernelILi4ELi1E", "amsq_restore_kernelILi7E", "amsq_xprep_tc_kernelILi7E",
        "amsq_quantize_kernel"]


def main():
    os.makedirs(OUT, exist_ok=True)
    text = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", text)
    summary = []
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        if not any(k in name for k in KEEP):
            continue
        body = f
        ops = collections.Counter()
        for line in body.splitlines():
            m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
            if m:
                ops[m.group(2)] += 1
        short = re.sub(r"^_ZN5amsqb3dev", "", name)[:60]
        lines = [re.sub(r"\s*/\* 0x[0-9a-f]+ \*/\s*$", "", ln) for ln in body.splitlines()]
        lines = [ln for ln in lines if ln.strip()]
        with open(os.path.join(OUT, short + ".sass"), "w") as fh:
            fh.write("Function : " + "\n".join(lines) + "\n")
        key = {k: ops.get(k, 0) for k in ("HMMA", "UTCHMMA", "UBLKCP", "LDTM", "UTCBAR",
                                          "UTCATOMSWS", "STTM", "LDGSTS", "SYNCS", "LOP3", "IMAD", "PRMT")}
        summary.append(f"{short}: {sum(ops.values())} instructions; " +
                       ", ".join(f"{k} {v}" for k, v in key.items() if v))
    with open(os.path.join(OUT, "SUMMARY.txt"), "w") as fh:
        fh.write("cuobjdump -sass paper_2510_16045_b200/libamsq_b200.so (static instruction counts)\n")
        fh.write("\n".join(summary) + "\n")
    print("\n".join(summary))


if __name__ == "__main__":
    main()

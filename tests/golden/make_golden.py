#!/usr/bin/env python
"""Generate the golden fixtures of tests/golden/ from the UNMODIFIED reference.

Run in the container that has /root/reference (the GPU box does not): it loads
oracle/_ref/libamsq_ref.so -- the reference headers compiled in place by
oracle/Makefile with the pinned flags (-O2 -ffp-contract=off) -- and records its
outputs, so the tests can pin the C oracle and the device kernels to the reference
on machines where the reference is absent.

  golden_small.npz   per scheme (all 8) x shape: weights from the reference's own RNG
                     (amsq_test-style gaussian_matrix, mt19937_64 + normal_distribution,
                     kernels.hpp:294-301), quantize_tensor's scales + payload
                     (quantize.hpp:188-216), restore_block grid bits (kernels.hpp:55-63),
                     restore_matrix fp32 (100-124), restore_matrix_half (127-133) and
                     gemv outputs (151-187) for several batches with gaussian_half
                     activations (the reference's generator, seed ^ batch as in bench,
                     kernels.hpp:352).
  golden_large.json  size-independent checks at the BASELINE.json config shapes:
                     SHA-256 of the reference's payload / scales / grid / gemv outputs for
                     numpy-seeded weights (np.random.default_rng(seed).standard_normal,
                     float32) so a machine without the reference can regenerate the
                     inputs and compare hashes.

Usage:  python tests/golden/make_golden.py            (rewrites both files)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import SCHEMES, load_ref  # noqa: E402

SMALL_SHAPES = [(32, 96), (33, 200), (4, 4096)]
SMALL_BATCHES = [1, 3, 8, 16]
# (scheme id, rows, cols, numpy seed, batches): config 1 (FP4.25 4096x4096, M=1) and the
# FP5.33 4096x4096 / K=14336 cases of config 2 at rows cut to keep the CPU time bounded.
LARGE = [
    (4, 4096, 4096, 1, [1]),
    (7, 4096, 4096, 1, [1, 4, 8, 16]),
    (4, 512, 14336, 2, [1, 8]),
    (7, 512, 14336, 2, [1, 8]),
]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def numpy_weights(rows, cols, seed):
    return np.random.default_rng(seed).standard_normal((rows, cols), dtype=np.float32)


def numpy_x(batch, cols, seed):
    return (np.random.default_rng(seed ^ batch).standard_normal(batch * cols)
            .astype(np.float16).view(np.uint16))


def grid_of(ref, sid, rows, pc, payload):
    """restore_block over every block (kernels.hpp:55-63: unpack_block, then table[code])."""
    if rows * pc > 1 << 16:  # large: the same route through the reference, vectorised
        return ref.restore_table(sid)[ref.unpack_row(sid, payload)].reshape(rows, pc)
    blk, wpb = SCHEMES[sid][1], SCHEMES[sid][2]
    wpr = pc // blk * wpb
    out = np.zeros((rows, pc), np.uint16)
    for r in range(rows):
        row = payload[r * wpr:(r + 1) * wpr]
        for b in range(pc // blk):
            out[r, b * blk:(b + 1) * blk] = ref.restore_block(sid, row[b * wpb:(b + 1) * wpb])
    return out


def main():
    ref = load_ref()
    if ref is None:
        sys.exit("oracle/_ref/libamsq_ref.so missing: run `make -C oracle` where /root/reference exists")
    small = {}
    for sid in SCHEMES:
        for rows, cols in SMALL_SHAPES:
            key = f"s{sid}_{rows}x{cols}"
            w = ref.gaussian_matrix(rows, cols, rows * 1000 + cols)
            scales, payload, pc = ref.quantize_tensor(sid, w)
            small[key + "_w"] = w
            small[key + "_scales"] = scales
            small[key + "_payload"] = payload
            small[key + "_pc"] = np.array([pc])
            small[key + "_grid"] = grid_of(ref, sid, rows, pc, payload)
            if sid in (4, 7):  # the device schemes: fp32 w*s too
                small[key + "_f32"] = ref.restore_matrix(sid, rows, cols, pc, scales, payload)
            small[key + "_f16"] = ref.restore_matrix_half(sid, rows, cols, pc, scales, payload)
            for m in SMALL_BATCHES:
                x = ref.gaussian_half(m * cols, (rows + cols) ^ m)
                small[f"x_{rows}x{cols}_{m}"] = x  # scheme-independent
                small[f"{key}_y{m}"] = ref.gemv(sid, rows, cols, pc, scales, payload, x, m)
    np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **small)

    large = []
    for sid, rows, cols, seed, batches in LARGE:
        w = numpy_weights(rows, cols, seed)
        scales, payload, pc = ref.quantize_tensor(sid, w, threads=0)
        rec = {"scheme": sid, "rows": rows, "cols": cols, "seed": seed, "padded_cols": pc,
               "weights": "np.random.default_rng(seed).standard_normal((rows, cols), float32)",
               "x": "np.random.default_rng(seed ^ M).standard_normal(M*cols) -> fp16",
               "payload_sha256": sha(payload), "scales_sha256": sha(scales),
               "grid_sha256": sha(grid_of(ref, sid, rows, pc, payload)), "gemv": {}}
        for m in batches:
            y = ref.gemv(sid, rows, cols, pc, scales, payload, numpy_x(m, cols, seed), m, threads=0)
            rec["gemv"][str(m)] = sha(y)
        large.append(rec)
        print(f"large scheme {sid} {rows}x{cols}: done", flush=True)
    with open(os.path.join(HERE, "golden_large.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py via oracle/_ref (reference "
                                "headers, g++ -std=c++20 -O2 -ffp-contract=off)",
                   "cases": large}, f, indent=1)


if __name__ == "__main__":
    main()

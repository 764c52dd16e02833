"""Shared test helpers: synthetic tensors and the linear tolerance bar."""
from __future__ import annotations

import numpy as np

import paper_2510_16045_b200 as amsq


def quantized_gaussian(scheme, rows, cols, seed=1, sigma=1.0) -> amsq.QuantizedTensor:
    rng = np.random.default_rng(seed)
    w = (rng.standard_normal((rows, cols)) * sigma).astype(np.float32)
    return amsq.quantize_tensor(w, scheme)


def random_payload(scheme, rows, cols, seed=1) -> amsq.QuantizedTensor:
    """Uniform random words: every u16 stream is a valid packed stream.
    Scales are positive finite fp16 around 0.5."""
    s = amsq.scheme_by_id(scheme) if isinstance(scheme, int) else scheme
    rng = np.random.default_rng(seed)
    pc = amsq.round_up(cols, s.block)
    wpr = pc // s.block * s.words_per_block
    payload = rng.integers(0, 1 << 16, size=rows * wpr, dtype=np.uint16)
    scales = np.array([amsq.float_to_half(v) for v in rng.uniform(0.25, 1.0, size=min(rows, 4096))],
                      np.uint16)
    scales = np.resize(scales, rows)
    return amsq.QuantizedTensor(s, rows, cols, pc, scales, payload)


def gaussian_x(batch, cols, seed=3) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.standard_normal(batch * cols).astype(np.float16).view(np.uint16)


def fp16_ulp(v: np.ndarray) -> np.ndarray:
    a = np.abs(v.astype(np.float16))
    nxt = np.nextafter(a, np.float16(np.inf), dtype=np.float16)
    return (nxt.astype(np.float64) - a.astype(np.float64))


def check_linear(y_bits, yref_bits, yabs, tol=1e-3):
    """SURVEY.md §8(d) bar: norm-wise rel err <= tol against the reference fp16 output,
    and per element |y - y_ref| <= tol * sum_i |w_i s x_i| + ulp_fp16(y_ref)."""
    y = np.asarray(y_bits, np.uint16).view(np.float16).astype(np.float64).reshape(yabs.shape)
    yr16 = np.asarray(yref_bits, np.uint16).view(np.float16).reshape(yabs.shape)
    yr = yr16.astype(np.float64)
    assert np.all(np.isfinite(y)), "non-finite output"
    den = np.linalg.norm(yr)
    rel = np.linalg.norm(y - yr) / den if den > 0 else np.linalg.norm(y - yr)
    assert rel <= tol, f"norm-wise rel err {rel:.3e} > {tol}"
    bound = tol * yabs + fp16_ulp(yr16)
    bad = np.abs(y - yr) > bound
    assert not bad.any(), (f"{bad.sum()} elements outside per-element bound; worst excess "
                           f"{(np.abs(y - yr) - bound).max():.3e}")
    return rel

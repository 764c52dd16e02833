"""Device-side quantize (csrc/quantize.cu) against the oracle's
quantize_tensor (quantize.hpp:188-216): scales and payload bit-exact for all 8 schemes, padding,
all-zero and tiny rows, exact rounding midpoints and the shared-bit ties; the reference's error
cases; the config-1 tensor's pinned SHA-256; and the device-quantized weight through the fused
linear."""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

import paper_2510_16045_b200 as amsq
from helpers import check_linear, gaussian_x

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SHAPES = [(1, 3), (16, 48), (33, 200), (64, 64), (300, 4098), (17, 14336)]


def _weights(sid, rows, cols, seed):
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((rows, cols), dtype=np.float32) * np.float32(rng.uniform(0.01, 4.0))
    if rows >= 4:
        w[1] = 0.0                                    # all-zero row: scale 1
        w[2] *= np.float32(1e-9)                      # tiny row: subnormal / clamped scale
        # exact rounding midpoints of the row's grid (ties to the even code)
        s = amsq.scheme_by_id(sid)
        table = amsq.restore_table(s).view(np.float16).astype(np.float32)
        vals = np.unique(np.abs(table[np.isfinite(table)]))
        mids = (vals[:-1] + vals[1:]) / 2
        row = np.resize(np.concatenate([mids, -mids]), cols).astype(np.float32)
        row[0] = vals[-1]                              # max |w| / M == 1: scale 1.0
        w[3] = row
    return w


@pytest.mark.parametrize("sid", range(8))
@pytest.mark.parametrize("shape", SHAPES)
def test_device_quantize_is_bit_exact(cuda, orc, sid, shape):
    rows, cols = shape
    w = _weights(sid, rows, cols, seed=rows * 7 + cols + sid)
    scales, payload, pc = orc.quantize_tensor(sid, w)
    qt = amsq.quantize_tensor_device(torch.from_numpy(w).to(cuda), sid)
    assert qt.padded_cols == pc
    assert np.array_equal(qt.scales, scales)
    assert np.array_equal(qt.payload, payload)


def test_device_quantize_matches_host_library_at_scale(cuda):
    """A 2048 x 4096 Gaussian through both of the library's quantizers (8 host threads)."""
    w = np.random.default_rng(5).standard_normal((2048, 4096), dtype=np.float32)
    for sid in (4, 7):
        host = amsq.quantize_tensor(w, sid, threads=8)
        dev = amsq.quantize_tensor_device(torch.from_numpy(w).to(cuda), sid)
        assert np.array_equal(host.scales, dev.scales)
        assert np.array_equal(host.payload, dev.payload)


def test_device_quantize_config1_sha(cuda):
    """Config 1: the reference's quantized Gaussian, pinned by golden_large.json."""
    rec = json.load(open(os.path.join(GOLDEN, "golden_large.json")))["cases"][0]
    sid, rows, cols, seed = rec["scheme"], rec["rows"], rec["cols"], rec["seed"]
    w = np.random.default_rng(seed).standard_normal((rows, cols), dtype=np.float32)
    qt = amsq.quantize_tensor_device(torch.from_numpy(w).to(cuda), sid)
    assert hashlib.sha256(qt.payload.tobytes()).hexdigest() == rec["payload_sha256"]


def test_device_quantize_errors(cuda):
    w = np.ones((4, 64), np.float32)
    w[2, 5] = np.nan
    with pytest.raises(amsq.CorruptError, match="non-finite"):
        amsq.quantize_tensor_device(torch.from_numpy(w).to(cuda), 4)
    w = np.ones((4, 64), np.float32)
    w[1, 0] = 3.0e38  # max|w| / M overflows binary16
    with pytest.raises(amsq.CorruptError, match="overflows"):
        amsq.quantize_tensor_device(torch.from_numpy(w).to(cuda), 7)
    with pytest.raises(ValueError):
        amsq.quantize_tensor_device(torch.zeros((0, 8), device=cuda), 7)


@pytest.mark.parametrize("sid", [4, 7])
def test_device_quantized_weight_runs_the_linear(cuda, orc, sid):
    rows, cols, m = 512, 4096, 4
    w = np.random.default_rng(9).standard_normal((rows, cols), dtype=np.float32)
    qt = amsq.quantize_tensor_device(torch.from_numpy(w).to(cuda), sid)
    dw = amsq.DeviceWeight(qt)
    x = gaussian_x(m, cols, seed=2)
    y = dw.linear(torch.from_numpy(x.view(np.float16).reshape(m, cols)).to(cuda))
    yref = orc.gemv(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, m).reshape(m, rows)
    wr = orc.restore_matrix(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload).astype(np.float64)
    yabs = np.abs(x.view(np.float16).astype(np.float64).reshape(m, cols)) @ np.abs(wr).T
    check_linear(y.cpu().numpy().view(np.uint16).reshape(m, rows), yref, yabs)
    dw.free()

"""bf16 activations (north star: "fp16/bf16 activations").

The reference is fp16-only (half.hpp), so bf16 is checked against the exact product in
float64: y64 = sum_i (w_i s)_fp32 * x_i with (w s) from the ORACLE's restore_matrix (bit-exact
to the reference's) and x the bf16 inputs. The device output is bf16, so it is compared with
y64 rounded to bf16: norm-wise ||y - bf16(y64)|| / ||y64|| <= 1e-3, and per element
|y - y64| <= 1e-3 * sum|w s x| + ulp_bf16(y64) (one output rounding).
"""
import numpy as np
import pytest
import torch

import paper_2510_16045_b200 as amsq
from helpers import quantized_gaussian, random_payload

pytestmark = pytest.mark.gpu


def _ref64(orc, sid, qt, x):
    w = orc.restore_matrix(sid, qt.rows, qt.cols, qt.padded_cols, qt.scales, qt.payload)
    wt = torch.from_numpy(w.astype(np.float64)).cuda()
    xt = x.double().cuda()
    return (xt @ wt.T).cpu(), (xt.abs() @ wt.abs().T).cpu()


def _check_bf16(y, y64, yabs, tol=1e-3):
    y = y.double().cpu()
    y64r = y64.to(torch.bfloat16).double()
    assert torch.isfinite(y).all()
    den = y64.norm().item()
    rel = (y - y64r).norm().item() / den if den > 0 else (y - y64r).norm().item()
    assert rel <= tol, f"norm-wise rel err {rel:.3e}"
    a = y64.abs().to(torch.bfloat16)
    ulp = (torch.nextafter(a, torch.tensor(float("inf"), dtype=torch.bfloat16)).double()
           - a.double())
    bad = (y - y64).abs() > tol * yabs + ulp
    assert not bad.any(), f"{int(bad.sum())} elements outside the per-element bound"
    return rel


@pytest.mark.parametrize("sid", [4, 7])
@pytest.mark.parametrize("shape", [(300, 1000), (4096, 4096), (1024, 14336)])
@pytest.mark.parametrize("batch", [1, 5, 8, 16, 32, 100])
def test_linear_bf16_activations(cuda, orc, sid, shape, batch):
    rows, cols = shape
    qt = random_payload(sid, rows, cols, seed=batch + rows) if rows > 300 else \
        quantized_gaussian(sid, rows, cols, seed=batch)
    g = torch.Generator().manual_seed(batch)
    x = torch.randn(batch, cols, generator=g).to(torch.bfloat16)
    y = amsq.DeviceWeight(qt).linear(x.to(cuda))
    assert y.dtype == torch.bfloat16 and y.shape == (batch, rows)
    y64, yabs = _ref64(orc, sid, qt, x)
    _check_bf16(y, y64, yabs)


@pytest.mark.parametrize("sid", [4, 7])
def test_bf16_range_extremes(cuda, orc, sid):
    """Rows far outside fp16's range (1e30, 1e-30), an outlier row, a zero row: the per-row
    power-of-two staging keeps them exact where fp16 itself would overflow or flush."""
    rows, cols = 256, 2048
    qt = random_payload(sid, rows, cols, seed=3)
    g = torch.Generator().manual_seed(0)
    x = torch.randn(5, cols, generator=g)
    x[0] *= 1e30
    x[1] *= 1e-30
    x[2, 7] = 3e4  # one outlier among N(0,1) values
    x[3] = 0
    x = x.to(torch.bfloat16)
    y = amsq.DeviceWeight(qt).linear(x.to(cuda))
    y64, yabs = _ref64(orc, sid, qt, x)
    assert torch.all(y[3].float() == 0)
    for r in (0, 1, 2, 4):
        _check_bf16(y[r:r + 1], y64[r:r + 1], yabs[r:r + 1])


def test_bf16_dtype_errors(cuda):
    qt = random_payload(7, 64, 96, seed=1)
    dw = amsq.DeviceWeight(qt)
    x = torch.randn(2, 96, device=cuda).to(torch.bfloat16)
    with pytest.raises(ValueError):
        dw.linear(x, out=torch.empty(2, 64, dtype=torch.float16, device=cuda))
    with pytest.raises(ValueError):
        dw.linear(x.float())
    from paper_2510_16045_b200._lib import lib
    assert lib().amsq_linear_ex(dw.handle, x.data_ptr(), 1, 2, x.data_ptr(), 0, 0, None) == 1


@pytest.mark.parametrize("sid", [0, 1, 2, 3, 5, 6])
@pytest.mark.parametrize("batch", [1, 16])
def test_linear_bf16_other_schemes(cuda, orc, sid, batch):
    rows, cols = 512, 3072
    qt = random_payload(sid, rows, cols, seed=sid * 7 + batch)
    g = torch.Generator().manual_seed(sid + batch)
    x = torch.randn(batch, cols, generator=g).to(torch.bfloat16)
    y = amsq.DeviceWeight(qt).linear(x.to(cuda))
    y64, yabs = _ref64(orc, sid, qt, x)
    _check_bf16(y, y64, yabs)

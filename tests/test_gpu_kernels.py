"""GPU parity tests of the sm_100a kernels against the oracle (run on the B200).

Bars: restore is bit-exact (grid bits vs restore_block, fp32 w*s vs
restore_matrix, fp16 vs restore_matrix_half); the fused linear is within
norm-wise 1e-3 and per-element 1e-3*sum|w s x| + 1 ulp of the reference gemv.
"""
import numpy as np
import pytest
import torch

import paper_2510_16045_b200 as amsq
from helpers import check_linear, gaussian_x, quantized_gaussian, random_payload

pytestmark = pytest.mark.gpu

SCHEMES = list(range(8))  # every scheme of scheme.hpp:59-74 has sm_100a kernels
AMS = [4, 7]              # the paper's two schemes (K3 tcgen05 path)
SHAPES = [(1, 64), (33, 200), (40, 100), (16, 48), (300, 1000), (257, 4096), (512, 4098)]


def _grid(dw):
    return dw.restore_grid().cpu().view(torch.int16).numpy().view(np.uint16)


@pytest.mark.parametrize("sid", SCHEMES)
@pytest.mark.parametrize("shape", SHAPES)
def test_restore_grid_bit_exact(cuda, orc, sid, shape):
    rows, cols = shape
    for qt in (quantized_gaussian(sid, rows, cols, seed=rows + cols),
               random_payload(sid, rows, cols, seed=rows * 7 + cols)):
        dw = amsq.DeviceWeight(qt)
        got = _grid(dw)
        want = orc.restore_grid(sid, rows, qt.padded_cols, qt.payload)
        assert np.array_equal(got, want), f"{(got != want).sum()} mismatching grid elements"


@pytest.mark.parametrize("sid", SCHEMES)
def test_restore_every_code_exhaustively(cuda, orc, sid):
    """kernels_test.cc:69-87 on the device: a block repeating one code, for every code."""
    s = amsq.scheme_by_id(sid)
    codes = np.repeat(np.arange(s.code_count, dtype=np.uint8), s.block)
    # consistent shared bits per group are guaranteed by repeating one code per block
    words = np.concatenate([amsq.pack_row(codes[i * s.block:(i + 1) * s.block], s)
                            for i in range(s.code_count)])
    rows = 16
    cols = s.code_count * s.block
    payload = np.tile(words, rows)
    qt = amsq.QuantizedTensor(s, rows, cols, cols, np.full(rows, 0x3C00, np.uint16), payload)
    got = _grid(amsq.DeviceWeight(qt))
    table = amsq.restore_table(s)
    want = np.tile(table[codes], (rows, 1))
    assert np.array_equal(got, want)
    assert np.array_equal(table, orc.restore_table(sid))


@pytest.mark.parametrize("sid", SCHEMES)
@pytest.mark.parametrize("shape", [(33, 200), (300, 1000), (64, 4096)])
def test_restore_matrix_f32_f16_bit_exact(cuda, orc, ref, sid, shape):
    rows, cols = shape
    qt = quantized_gaussian(sid, rows, cols, seed=11)
    dw = amsq.DeviceWeight(qt)
    f32 = dw.restore_f32().cpu().numpy()
    want = orc.restore_matrix(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload)
    assert np.array_equal(f32.view(np.uint32), want.view(np.uint32))
    f16 = dw.restore_f16().cpu().view(torch.int16).numpy().view(np.uint16)
    want16 = ref.restore_matrix_half(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload)
    assert np.array_equal(f16, want16)


@pytest.mark.parametrize("sid", SCHEMES)
@pytest.mark.parametrize("shape", [(33, 200), (256, 256), (300, 1000), (1000, 4098)])
@pytest.mark.parametrize("batch", [1, 2, 3, 5, 8, 9, 16, 17, 33])
def test_linear_matches_reference_gemv(cuda, orc, sid, shape, batch):
    rows, cols = shape
    qt = quantized_gaussian(sid, rows, cols, seed=batch + rows)
    x = gaussian_x(batch, cols, seed=batch)
    dw = amsq.DeviceWeight(qt)
    xt = torch.from_numpy(x.view(np.float16).reshape(batch, cols)).to(cuda)
    y = dw.linear(xt).cpu().numpy().view(np.uint16).reshape(batch, rows)
    yref = orc.gemv(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    _, yabs = orc.gemv_f64(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    check_linear(y, yref, yabs)


@pytest.mark.parametrize("sid", SCHEMES)
def test_linear_random_payload_large_k(cuda, orc, sid):
    """Random valid payload (every code incl. -0 and subnormals) at K = 14336 (8B down)."""
    rows, cols, batch = 256, 14336, 4
    qt = random_payload(sid, rows, cols, seed=5)
    x = gaussian_x(batch, cols, seed=9)
    dw = amsq.DeviceWeight(qt)
    y = dw.gemv_host(x, batch).reshape(batch, rows)
    yref = orc.gemv(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    _, yabs = orc.gemv_f64(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    check_linear(y, yref, yabs)


@pytest.mark.parametrize("batch", [1, 16, 40, 128])
@pytest.mark.parametrize("sid", SCHEMES)
def test_gemv_host_pinned_y_direct(cuda, orc, sid, batch):
    """amsq_gemv_host into page-locked host y: the epilogue (K2 or K3) stores y over the host
    link instead of a D2H copy. Bit-identical to the pageable-y path, within the bar."""
    import torch

    from paper_2510_16045_b200._lib import check, lib
    rows, cols = 1024, 4096
    qt = random_payload(sid, rows, cols, seed=batch)
    x = gaussian_x(batch, cols, seed=batch + 1)
    dw = amsq.DeviceWeight(qt)
    y_pageable = dw.gemv_host(x, batch)
    hy = torch.full((batch * rows,), -1, dtype=torch.int16).pin_memory()
    hx = torch.from_numpy(x.view(np.int16).copy()).pin_memory()
    st = torch.cuda.current_stream().cuda_stream
    check(lib().amsq_gemv_host(dw._h, hx.data_ptr(), x.size, batch, hy.data_ptr(), st), "gemv")
    y_direct = hy.numpy().view(np.uint16)
    assert np.array_equal(y_direct, y_pageable)
    prev = lib().amsq_debug_set_host_direct(0)
    try:
        hy.fill_(-1)
        check(lib().amsq_gemv_host(dw._h, hx.data_ptr(), x.size, batch, hy.data_ptr(), st), "gemv")
    finally:
        lib().amsq_debug_set_host_direct(prev)
    assert np.array_equal(hy.numpy().view(np.uint16), y_pageable)
    yref = orc.gemv(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    _, yabs = orc.gemv_f64(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    check_linear(y_direct.reshape(batch, rows), yref, yabs)


@pytest.mark.parametrize("sid", SCHEMES)
def test_subnormal_codes_survive_the_tensor_cores(cuda, orc, sid):
    """Placed subnormal-source codes are binary16 subnormals; the MMA must not flush them."""
    s = amsq.scheme_by_id(sid)
    sub = [c for c in range(1, s.code_count // 2) if (c >> s.man_bits) == 0]  # exp field 0
    rows, cols = 16, s.block * 64
    codes = np.zeros(cols, np.uint8)
    for i in range(0, cols, s.k):
        codes[i:i + s.k] = sub[(i // s.k) % len(sub)] & ~1 | ((i // s.k) & 1)
    codes = np.array([c if c != s.sign_mask else 0 for c in codes], np.uint8)
    words = amsq.pack_row(codes, s)
    qt = amsq.QuantizedTensor(s, rows, cols, cols, np.full(rows, 0x3C00, np.uint16),
                              np.tile(words, rows))
    x = np.full(cols, 0x3C00, np.uint16)  # ones
    y = amsq.DeviceWeight(qt).gemv_host(x, 1)
    want = sum(orc.decode(int(c), sid) for c in codes)
    got = y.view(np.float16).astype(np.float64)
    assert np.all(np.abs(got - want) <= 1e-3 * abs(want) + 1e-3), (got[:4], want)


@pytest.mark.parametrize("sid", SCHEMES)
def test_linear_deterministic_and_graph_replayable(cuda, sid):
    rows, cols, batch = 4096, 4096, 8
    qt = random_payload(sid, rows, cols, seed=1)
    dw = amsq.DeviceWeight(qt)
    x = torch.from_numpy(gaussian_x(batch, cols).view(np.float16).reshape(batch, cols)).to(cuda)
    y0 = dw.linear(x).clone()
    for _ in range(3):
        assert torch.equal(dw.linear(x), y0)
    out = torch.empty_like(y0)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        dw.linear(x, out=out, stream=s)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        dw.linear(x, out=out)
    for _ in range(3):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, y0)


@pytest.mark.parametrize("sid", SCHEMES)
def test_upload_download_round_trip(cuda, sid):
    for rows, cols in [(33, 200), (300, 4098), (1, 3)]:
        qt = random_payload(sid, rows, cols, seed=rows)
        back = amsq.DeviceWeight(qt).download()
        assert np.array_equal(back.payload, qt.payload)
        assert np.array_equal(back.scales, qt.scales)


def test_shape_errors(cuda):
    qt = quantized_gaussian(7, 4, 9)
    dw = amsq.DeviceWeight(qt)
    with pytest.raises(ValueError):
        dw.gemv_host(np.zeros(7, np.uint16), 1)
    with pytest.raises(ValueError):
        dw.gemv_host(np.zeros(9, np.uint16), 0)
    with pytest.raises(ValueError):
        amsq.gemv(qt, np.zeros(8, np.uint16), 1)


def test_reference_call_shapes(cuda, orc):
    """amsq.gemv / restore_matrix with the reference signatures (host in, host out)."""
    qt = quantized_gaussian(4, 70, 130, seed=2)
    x = gaussian_x(3, 130)
    y = amsq.gemv(qt, x, 3).reshape(3, 70)
    yref = orc.gemv(4, 70, 130, qt.padded_cols, qt.scales, qt.payload, x, 3)
    _, yabs = orc.gemv_f64(4, 70, 130, qt.padded_cols, qt.scales, qt.payload, x, 3)
    check_linear(y, yref, yabs)
    m = amsq.restore_matrix(qt)
    want = orc.restore_matrix(4, 70, 130, qt.padded_cols, qt.scales, qt.payload)
    assert np.array_equal(m.view(np.uint32), want.view(np.uint32))


def test_cpp_dropin_against_reference(cuda):
    """The reference's own QuantizedTensor / gemv / restore_matrix(_half) next to
    include/amsq_b200.hpp (tests/cpp/dropin_test.cpp, prebuilt into oracle/_ref)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle",
                       "_ref", "dropin_test")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/dropin_test was not built where /root/reference exists")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failure(s)" in r.stdout


@pytest.fixture
def force_k3():
    """Route every batch > 16 to K3 (default: K2 in 32-row chunks below the per-scheme crossover)."""
    from paper_2510_16045_b200._lib import lib
    prev = lib().amsq_debug_set_k3_min_batch(17)
    yield
    lib().amsq_debug_set_k3_min_batch(prev)


@pytest.fixture
def force_k3_all():
    from paper_2510_16045_b200._lib import lib
    prev = lib().amsq_debug_set_k3_min_batch(1)
    yield
    lib().amsq_debug_set_k3_min_batch(prev)


@pytest.fixture
def force_k2():
    from paper_2510_16045_b200._lib import lib
    prev = lib().amsq_debug_set_k3_min_batch(100000)
    yield
    lib().amsq_debug_set_k3_min_batch(prev)


@pytest.mark.parametrize("sid", SCHEMES)
@pytest.mark.parametrize("shape", [(33, 200), (300, 1000), (1000, 4098), (80000, 64)])
@pytest.mark.parametrize("batch", [17, 24, 31, 32, 40, 64])
def test_linear_k2_batch_chunks(cuda, orc, sid, shape, batch, force_k2):
    """17 <= M < 65 runs K2 in 32-row chunks (M <= 32: the NB = 4 kernel; groups taller than
    32 row tiles fall back to two M <= 16 launches)."""
    rows, cols = shape
    qt = quantized_gaussian(sid, rows, cols, seed=batch * 5 + rows)
    x = gaussian_x(batch, cols, seed=batch + 13)
    xt = torch.from_numpy(x.view(np.float16).reshape(batch, cols)).to(cuda)
    y = amsq.DeviceWeight(qt).linear(xt).cpu().numpy().view(np.uint16).reshape(batch, rows)
    yref = orc.gemv(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    _, yabs = orc.gemv_f64(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    check_linear(y, yref, yabs)


@pytest.mark.parametrize("sid", AMS)
@pytest.mark.parametrize("shape", [(128, 64), (300, 1000), (1000, 4098)])
@pytest.mark.parametrize("batch", [24, 32, 64, 100, 256, 300])
def test_linear_large_batch_tcgen05(cuda, orc, sid, shape, batch, force_k3):
    """K3 (tcgen05.mma + TMEM, up to 256 batch rows per launch), forced for every M > 16."""
    rows, cols = shape
    qt = quantized_gaussian(sid, rows, cols, seed=batch * 3 + rows)
    x = gaussian_x(batch, cols, seed=batch + 11)
    dw = amsq.DeviceWeight(qt)
    xt = torch.from_numpy(x.view(np.float16).reshape(batch, cols)).to(cuda)
    y = dw.linear(xt).cpu().numpy().view(np.uint16).reshape(batch, rows)
    yref = orc.gemv(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    _, yabs = orc.gemv_f64(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    check_linear(y, yref, yabs)


@pytest.mark.parametrize("sid", AMS)
@pytest.mark.parametrize("shape", [(128, 64), (300, 1000), (4096, 4098)])
@pytest.mark.parametrize("batch", [1, 5, 16])
def test_linear_tcgen05_small_batch(cuda, orc, sid, shape, batch, force_k3_all):
    """K3 below 16 rows (one 16-column N chunk, zero-padded batch rows): the A-in-TMEM MMA path
    at the smallest N the kind::f16 instruction takes."""
    rows, cols = shape
    qt = quantized_gaussian(sid, rows, cols, seed=batch * 7 + rows)
    x = gaussian_x(batch, cols, seed=batch + 3)
    xt = torch.from_numpy(x.view(np.float16).reshape(batch, cols)).to(cuda)
    y = amsq.DeviceWeight(qt).linear(xt).cpu().numpy().view(np.uint16).reshape(batch, rows)
    yref = orc.gemv(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    _, yabs = orc.gemv_f64(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    check_linear(y, yref, yabs)


@pytest.fixture
def force_pairs():
    from paper_2510_16045_b200._lib import lib
    prev = lib().amsq_debug_set_k3_pair(1)
    yield
    lib().amsq_debug_set_k3_pair(prev)


@pytest.mark.parametrize("sid", AMS)
@pytest.mark.parametrize("rows", [19032, 19200])
@pytest.mark.parametrize("batch", [17, 64, 128, 200])
def test_linear_tcgen05_cta_pairs(cuda, orc, sid, rows, batch, force_k3, force_pairs):
    """K3 in CTA-pair mode (cta_group::2, M = 256 MMAs over two CTAs' 128-row blocks, the
    activation image split by N across the pair), forced at every batch: 149 row blocks (an odd
    count: the last pair's follower has no rows) and 150."""
    cols = 256
    qt = quantized_gaussian(sid, rows, cols, seed=rows + batch)
    x = gaussian_x(batch, cols, seed=batch + 5)
    xt = torch.from_numpy(x.view(np.float16).reshape(batch, cols)).to(cuda)
    y = amsq.DeviceWeight(qt).linear(xt).cpu().numpy().view(np.uint16).reshape(batch, rows)
    yref = orc.gemv(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    _, yabs = orc.gemv_f64(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    check_linear(y, yref, yabs)


@pytest.mark.parametrize("sid", AMS)
@pytest.mark.parametrize("batch", [17, 48, 112, 144, 200])
def test_linear_tcgen05_cluster_split_odd_chunks(cuda, orc, sid, batch, force_k3):
    """K3 with a 2/4-CTA K split and a batch whose 16-column chunk count is odd."""
    rows, cols = 512, 2048 if sid == 4 else 2049
    qt = quantized_gaussian(sid, rows, cols, seed=batch)
    x = gaussian_x(batch, cols, seed=batch + 1)
    xt = torch.from_numpy(x.view(np.float16).reshape(batch, cols)).to(cuda)
    y = amsq.DeviceWeight(qt).linear(xt).cpu().numpy().view(np.uint16).reshape(batch, rows)
    yref = orc.gemv(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    _, yabs = orc.gemv_f64(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    check_linear(y, yref, yabs)


@pytest.mark.parametrize("sid", [0, 1, 2, 3, 5, 6])
@pytest.mark.parametrize("batch", [65, 100, 256])
def test_other_schemes_large_batch_run_k2_chunks(cuda, orc, sid, batch):
    """The six non-AMS schemes have no K3 instance: every batch runs K2 in 32-row chunks."""
    rows, cols = 600, 2048
    qt = random_payload(sid, rows, cols, seed=batch + sid)
    x = gaussian_x(batch, cols, seed=batch)
    xt = torch.from_numpy(x.view(np.float16).reshape(batch, cols)).to(cuda)
    y = amsq.DeviceWeight(qt).linear(xt).cpu().numpy().view(np.uint16).reshape(batch, rows)
    yref = orc.gemv(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    _, yabs = orc.gemv_f64(sid, rows, cols, qt.padded_cols, qt.scales, qt.payload, x, batch)
    check_linear(y, yref, yabs)

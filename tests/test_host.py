"""CPU tests of the product's host side (libamsq_b200.so C++ core through the C-ABI).

* the library loads and exports every symbol include/amsq_b200.h declares;
* the host quantizer, pack/unpack, restore table and container are bit-identical to the
  oracle and to the reference fixtures (the host drop-in half of SURVEY.md §8(b));
* the device tile layout is an exact bit permutation of the reference stream
  (repack -> unrepack round trip) and -- through a numpy emulation of the kernel's
  register decode (tests/emulate.py) -- restores to the reference grid bit for bit;
* device entry points fail loudly (NoDeviceError) without a GPU: no CPU fallback.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2510_16045_b200 as amsq
from paper_2510_16045_b200._lib import LIB_PATH, SIGNATURES, lib

import emulate
from helpers import random_payload

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def _header_symbols():
    text = open(os.path.join(ROOT, "include", "amsq_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(amsq_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    syms = _header_symbols()
    assert len(syms) >= 30
    L = C.CDLL(LIB_PATH)
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert set(syms) == set(SIGNATURES), set(syms) ^ set(SIGNATURES)


def test_library_is_sm100a_only():
    """The fatbin holds sm_100a SASS and nothing else (no PTX JIT / other arch)."""
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_schemes_match_reference_table(orc):
    from oracle import SCHEMES
    for s in amsq.all_schemes():
        name, blk, wpb, k, e, m, bias = SCHEMES[s.id]
        assert (s.name, s.block, s.words_per_block, s.k, s.exp_bits, s.man_bits, s.bias) == \
            (name, blk, wpb, k, e, m, bias)
        assert s.device_supported  # every scheme has sm_100a kernels
    assert amsq.scheme_by_name("fp5.33-e2m3").id == 7
    assert amsq.all_schemes()[4].effective_bits() == 4.25
    with pytest.raises(ValueError):
        amsq.scheme_by_name("fp3")


def test_half_and_table_vs_oracle(orc):
    for h in range(0, 0x10000, 3):
        f = amsq.half_to_float(h)
        if np.isnan(f):
            continue
        assert f == orc.half_to_float(h)
    rng = np.random.default_rng(0)
    for f in np.concatenate([rng.standard_normal(2000) * 10.0 ** rng.integers(-9, 6, 2000),
                             [65519.99, 65520.0, 2.0 ** -25, 3 * 2.0 ** -25, -0.0]]):
        assert amsq.float_to_half(float(f)) == orc.float_to_half(float(f))
    for sid in range(8):
        assert np.array_equal(amsq.restore_table(sid), orc.restore_table(sid))


@pytest.fixture(scope="module")
def small():
    return np.load(os.path.join(GOLDEN, "golden_small.npz"))


def test_host_quantizer_matches_reference_fixtures(small):
    """quantize_tensor (RTN + Adaptive Searching + pack) bit-identical to the reference."""
    keys = sorted({k.rsplit("_", 1)[0] for k in small.files if k.endswith("_payload")})
    for key in keys:
        sid = int(key[1:key.index("_")])
        for threads in (1, 3):
            qt = amsq.quantize_tensor(small[key + "_w"], sid, threads=threads)
            assert qt.padded_cols == int(small[key + "_pc"][0])
            assert np.array_equal(qt.scales, small[key + "_scales"]), key
            assert np.array_equal(qt.payload, small[key + "_payload"]), key


@pytest.mark.parametrize("sid", range(8))
def test_host_quantizer_matches_oracle_random(orc, sid):
    rng = np.random.default_rng(sid)
    w = (rng.standard_normal((37, 301)) * rng.uniform(0.01, 3, (37, 1))).astype(np.float32)
    w[3, :7] = 0.0
    w[5] = 0.0
    qt = amsq.quantize_tensor(w, sid, threads=0)
    scales, payload, pc = orc.quantize_tensor(sid, w)
    assert qt.padded_cols == pc
    assert np.array_equal(qt.scales, scales) and np.array_equal(qt.payload, payload)


def test_quantizer_errors():
    """quantize_test.cc:328-338: empty -> invalid_argument; non-finite -> runtime_error,
    also from worker threads."""
    with pytest.raises(ValueError):
        amsq.quantize_tensor(np.zeros((0, 4), np.float32), 7)
    bad = np.zeros((1, 2), np.float32)
    bad[0, 1] = np.inf
    with pytest.raises(RuntimeError):
        amsq.quantize_tensor(bad, 2)
    wide = np.zeros((8, 4), np.float32)
    wide[7, 3] = np.nan
    with pytest.raises(RuntimeError):
        amsq.quantize_tensor(wide, 2, threads=4)


@pytest.mark.parametrize("sid", range(8))
def test_host_pack_unpack_vs_oracle(orc, sid):
    s = amsq.scheme_by_id(sid)
    rng = np.random.default_rng(50 + sid)
    words = rng.integers(0, 1 << 16, size=s.words_per_block * 7, dtype=np.uint16)
    codes = amsq.unpack_row(words, s)
    assert np.array_equal(codes, orc.unpack_row(sid, words))
    assert np.array_equal(amsq.pack_row(codes, s), orc.pack_row(sid, codes))


def test_pack_errors_map_to_reference_exceptions():
    s7 = amsq.scheme_by_id(7)
    with pytest.raises(amsq.CorruptError):  # std::runtime_error (packing.hpp:176-179)
        amsq.pack_row(np.array([1, 0, 1], np.uint8), s7)
    with pytest.raises(ValueError):  # std::invalid_argument (packing.hpp:220)
        amsq.pack_row(np.zeros(10, np.uint8), amsq.scheme_by_id(2))
    with pytest.raises(ValueError):
        amsq.unpack_row(np.zeros(7, np.uint16), amsq.scheme_by_id(2))


def test_byte_formula():
    """kernels_test.cc:186-218, quantize.hpp:64-69."""
    assert amsq.packed_payload_bytes(4, 1, 64) == 34
    fp16 = 2.0 * 5120 * 25600
    assert fp16 / amsq.packed_payload_bytes(4, 5120, 25600) == 16.0 / 4.25
    assert abs(fp16 / amsq.packed_payload_bytes(7, 5120, 25600) - 3.0) <= 1e-3
    for sid, (n, k, want) in {7: (4096, 4096, 11190272), 4: (28672, 4096, 62390272)}.items():
        assert amsq.packed_payload_bytes(sid, n, k) == want  # SURVEY.md §8(a) probe table


# ------------------------------------------------------------------ container
def test_container_round_trip_and_header(small):
    qt = amsq.quantize_tensor(small["s7_33x200_w"], 7)
    blob = amsq.write_amsq(qt)
    # container.hpp:4-9: "AMSQ" | u16 version 1 | u8 scheme | u8 k | u32 rows | u32 cols | u32 padded
    assert blob[:4] == b"AMSQ" and blob[4:6] == b"\x01\x00" and blob[6] == 7 and blob[7] == 3
    assert int.from_bytes(blob[8:12], "little") == 33
    assert int.from_bytes(blob[12:16], "little") == 200
    assert int.from_bytes(blob[16:20], "little") == 201
    back = amsq.read_amsq(blob)
    assert np.array_equal(back.payload, qt.payload) and np.array_equal(back.scales, qt.scales)
    assert amsq.write_amsq(back) == blob  # byte-stable on rewrite (io_test.cc:133-153)


def test_container_golden_header_bytes():
    """io_test.cc:155-171."""
    blob = amsq.write_amsq(amsq.quantize_tensor(np.zeros((1, 2), np.float32), 0))
    assert list(blob[:22]) == [ord("A"), ord("M"), ord("S"), ord("Q"), 1, 0, 0, 1, 1, 0, 0, 0,
                               2, 0, 0, 0, 16, 0, 0, 0, 0, 0x3C]
    assert len(blob) == 20 + 2 + 8 + 8


def test_container_rejects_corruption():
    """io_test.cc:173-213, same exception types (std::runtime_error / invalid_argument)."""
    qt = amsq.quantize_tensor(np.random.default_rng(1).standard_normal((2, 3)).astype(np.float32), 7)
    good = amsq.write_amsq(qt)

    def mutated(pos, val):
        b = bytearray(good)
        b[pos] = val
        return bytes(b)

    for pos, val in [(0, ord("X")), (4, 2), (7, 2)]:
        with pytest.raises(amsq.CorruptError):
            amsq.read_amsq(mutated(pos, val))
    with pytest.raises(ValueError):  # scheme id out of range -> invalid_argument
        amsq.read_amsq(mutated(6, 9))
    with pytest.raises(amsq.CorruptError):  # truncated
        amsq.read_amsq(good[:-1])
    pos = 20 + 2 * qt.rows  # payload_len disagrees with the layout formula
    with pytest.raises(amsq.CorruptError):
        amsq.read_amsq(mutated(pos, (good[pos] + 2) & 0xFF))


# ------------------------------------------------------------------ device layout
def _repack(qt):
    n = lib().amsq_device_layout_bytes(qt.scheme.id, qt.rows, qt.cols)
    tiles = np.zeros(n, np.uint8)
    from paper_2510_16045_b200._lib import check
    check(lib().amsq_repack(qt.scheme.id, qt.rows, qt.cols, qt.padded_cols, qt.payload.ctypes.data,
                            qt.payload.size, tiles.ctypes.data, tiles.size), "repack")
    back = np.zeros_like(qt.payload)
    check(lib().amsq_unrepack(qt.scheme.id, qt.rows, qt.cols, qt.padded_cols, tiles.ctypes.data,
                              tiles.size, back.ctypes.data, back.size), "unrepack")
    return tiles, back


def _plan(sid, rows, cols):
    plan = (C.c_int * 4)()
    from paper_2510_16045_b200._lib import check
    check(lib().amsq_device_layout_plan(sid, rows, cols, plan), "plan")
    return tuple(plan)


@pytest.mark.parametrize("sid", range(8))
def test_work_plans_at_config_shapes(sid):
    """Every Llama-3.1-8B/70B (and TP-shard) shape gets a plan that covers its row tiles
    exactly, fits 148 SMs, keeps <= 64 row tiles per CTA and balances within 16 %."""
    shapes = [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336), (10240, 8192),
              (8192, 8192), (57344, 8192), (8192, 28672), (1280, 8192), (1024, 8192),
              (7168, 8192), (1024, 28672), (33, 200), (1, 3)]
    tk = emulate.TRAITS[sid]["tk"]
    for rows, cols in shapes:
        n_groups, g_big, n_big, cs = _plan(sid, rows, cols)
        rt = -(-rows // 16)
        kt = -(-amsq.round_up(cols, amsq.scheme_by_id(sid).block) // tk)
        assert n_big * g_big + (n_groups - n_big) * (g_big - 1) == rt
        assert 1 <= n_big <= n_groups and n_groups * cs <= 148 and 1 <= g_big <= 64
        assert cs in (1, 2, 4, 8)
        if rt * kt >= 148 * 32:  # big enough to fill the GPU: per-CTA work near the ideal
            ideal = rt * kt / 148
            assert g_big * -(-kt // cs) <= 1.16 * ideal + g_big, (rows, cols, n_groups, g_big, cs)


LAYOUT_SHAPES = [(1, 3), (1, 64), (16, 48), (33, 200), (40, 100), (257, 4096), (300, 4098),
                 (17, 14336)]


@pytest.mark.parametrize("sid", range(8))
@pytest.mark.parametrize("shape", LAYOUT_SHAPES)
def test_repack_is_exact_bit_permutation(sid, shape):
    rows, cols = shape
    qt = random_payload(sid, rows, cols, seed=rows * 31 + cols)
    if sid == 7 and qt.padded_cols > cols:  # padding codes are zero in real streams
        qt.payload.reshape(rows, -1)[:, -1] &= np.uint16(0x7FFF >> (5 * (3 - (qt.padded_cols - cols))))
    tiles, back = _repack(qt)
    assert np.array_equal(back, qt.payload)
    # a permutation preserves the number of set bits (padding adds only zeros)
    assert int(np.unpackbits(tiles).sum()) == int(np.unpackbits(qt.payload.view(np.uint8)).sum())


@pytest.mark.parametrize("sid", range(8))
@pytest.mark.parametrize("shape", [(16, 48), (33, 200), (300, 1000), (40, 4098)])
def test_emulated_kernel_decode_restores_reference_grid(orc, sid, shape):
    """The tile bytes, decoded exactly as the sm_100a registers do (decode_s4/decode_s7 +
    the A/B fragment column map), give the reference restore grid (x 2^14)."""
    rows, cols = shape
    qt = random_payload(sid, rows, cols, seed=rows + 7 * cols)
    if qt.padded_cols > cols:
        qt = amsq.quantize_tensor(np.random.default_rng(1).standard_normal((rows, cols)).astype(np.float32), sid)
    tiles, _ = _repack(qt)
    tk = emulate.TRAITS[sid]["tk"]
    row_tiles = -(-rows // 16)
    k_tiles = -(-qt.padded_cols // tk)
    placed = emulate.placed_matrix(sid, tiles, row_tiles, k_tiles, _plan(sid, rows, cols))
    grid = emulate.placed_to_grid(placed, sid)[:rows, :qt.padded_cols]
    want = orc.restore_grid(sid, rows, qt.padded_cols, qt.payload)
    # -0 codes place to 0x8000 and stay -0 after the exact rescale
    assert np.array_equal(grid, want)
    assert not grid[:, qt.padded_cols:].any() if grid.shape[1] > qt.padded_cols else True


# ------------------------------------------------------------------ no CPU fallback
def test_device_entry_points_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    qt = random_payload(7, 16, 48)
    with pytest.raises(amsq.NoDeviceError):
        amsq.DeviceWeight(qt)
    with pytest.raises(amsq.NoDeviceError):
        amsq.gemv(qt, np.zeros(48, np.uint16), 1)
    h = C.c_void_p(None)
    rc = lib().amsq_linear(h, None, 1, None, None)
    assert rc != 0
    # the device quantizer: valid arguments, no device -> AMSQ_ENODEV (never the host path)
    fake = C.c_void_p(256)
    from paper_2510_16045_b200._lib import AMSQ_ENODEV
    assert lib().amsq_quantize_device(7, fake, 4, 6, 6, fake, fake, 8, 0, None) == AMSQ_ENODEV


def test_container_file_upload_validates_before_the_device(tmp_path):
    """amsq_weight_upload_file: mmap + container.hpp:79-115 validation. Missing or corrupt
    files are data errors (CorruptError = std::runtime_error) on any machine; a valid file
    without a GPU fails loudly with NoDeviceError (no CPU fallback)."""
    import torch
    qt = random_payload(4, 20, 128)
    good = tmp_path / "w.amsq"
    good.write_bytes(amsq.write_amsq(qt))
    with pytest.raises(amsq.CorruptError):
        amsq.DeviceWeight.from_file(str(tmp_path / "missing.amsq"))
    bad = tmp_path / "bad.amsq"
    bad.write_bytes(b"AMSX" + good.read_bytes()[4:])
    with pytest.raises(amsq.CorruptError):
        amsq.DeviceWeight.from_file(str(bad))
    trunc = tmp_path / "trunc.amsq"
    trunc.write_bytes(good.read_bytes()[:-2])
    with pytest.raises(amsq.CorruptError):
        amsq.DeviceWeight.from_file(str(trunc))
    if not torch.cuda.is_available():
        with pytest.raises(amsq.NoDeviceError):
            amsq.DeviceWeight.from_file(str(good))


def test_cpp_dropin_without_gpu():
    """tests/cpp/dropin_test.cpp (reference headers + include/amsq_b200.hpp): without a
    GPU every device call raises std::runtime_error and shape errors invalid_argument."""
    import subprocess
    import torch
    exe = os.path.join(ROOT, "oracle", "_ref", "dropin_test")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/dropin_test not built (no /root/reference here)")
    if torch.cuda.is_available():
        pytest.skip("GPU present: the GPU suite runs this binary")
    r = subprocess.run([exe, "--no-gpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


def test_k2_k3_dispatch_crossover():
    """amsq_linear_uses_tc: the measured per-scheme crossover (FP5.33 K3 from 33 rows, FP4.25
    from 40, the other schemes always K2), the override knob and its restore."""
    L = lib()
    assert L.amsq_debug_set_k3_min_batch(0) == -1  # defaults in force
    assert [L.amsq_linear_uses_tc(7, m) for m in (1, 16, 32, 33, 256)] == [0, 0, 0, 1, 1]
    assert [L.amsq_linear_uses_tc(4, m) for m in (16, 32, 39, 40, 300)] == [0, 0, 0, 1, 1]
    assert L.amsq_linear_uses_tc(2, 1000) == 0
    prev = L.amsq_debug_set_k3_min_batch(17)
    assert prev == -1 and L.amsq_linear_uses_tc(4, 17) == 1 and L.amsq_linear_uses_tc(7, 16) == 0
    assert L.amsq_debug_set_k3_min_batch(prev) == 17
    assert L.amsq_linear_uses_tc(7, 32) == 0 and L.amsq_linear_uses_tc(4, 39) == 0


def test_quantize_device_host_query_and_errors():
    """amsq_quantize_device_host: the size query works without a device (as amsq_quantize_tensor's
    does); argument errors are EINVAL; a real call without a GPU is ENODEV (no host fallback)."""
    from paper_2510_16045_b200._lib import AMSQ_EINVAL, AMSQ_ENODEV
    import torch
    pc, nw = C.c_size_t(0), C.c_size_t(0)
    assert lib().amsq_quantize_device_host(7, 5, 10, None, 0, C.byref(pc), C.byref(nw), None, None) == 0
    assert (pc.value, nw.value) == (12, 5 * 4)
    assert lib().amsq_quantize_device_host(7, 0, 10, None, 0, C.byref(pc), C.byref(nw), None, None) == AMSQ_EINVAL
    if not torch.cuda.is_available():
        w = np.ones((5, 10), np.float32)
        sc = np.zeros(5, np.uint16)
        pl = np.zeros(20, np.uint16)
        assert lib().amsq_quantize_device_host(7, 5, 10, w.ctypes.data, 0, C.byref(pc), C.byref(nw),
                                               sc.ctypes.data, pl.ctypes.data) == AMSQ_ENODEV

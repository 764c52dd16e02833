"""Pin the C oracle (oracle/amsq_oracle.c) before trusting it (CPU only).

(a) the golden vectors of the reference's own unit tests, restated
    (packing_test.cc, kernels_test.cc, half_test.cc, format_test.cc, quantize_test.cc);
(b) the fixtures tests/golden/make_golden.py generated from the unmodified reference
    (oracle/_ref): small tensors bit for bit, config-size tensors by SHA-256;
(c) live comparison against oracle/_ref when it is built on this machine.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import SCHEMES, padded_cols

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def small():
    return np.load(os.path.join(GOLDEN, "golden_small.npz"))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---------------------------------------------------------------- (a) golden vectors
def test_half_known_patterns(orc):
    """half_test.cc:16-60."""
    f2h = orc.float_to_half
    assert f2h(0.0) == 0x0000 and f2h(-0.0) == 0x8000
    assert f2h(1.0) == 0x3C00 and f2h(-2.0) == 0xC000 and f2h(0.5) == 0x3800
    assert f2h(65504.0) == 0x7BFF and f2h(7.5) == 0x4780
    assert f2h(2.0 ** -24) == 0x0001 and f2h(2.0 ** -14) == 0x0400
    assert f2h(1.0 + 2.0 ** -11) == 0x3C00 and f2h(1.0 + 3 * 2.0 ** -11) == 0x3C02
    assert f2h(2.0 ** -25) == 0x0000 and f2h(3 * 2.0 ** -25) == 0x0002
    assert f2h(65520.0) == 0x7C00 and f2h(-65520.0) == 0xFC00 and f2h(1e20) == 0x7C00
    assert f2h(float("inf")) == 0x7C00
    assert np.isnan(orc.half_to_float(0x7C01))
    assert orc.half_to_float(0x03FF) == 1023 * 2.0 ** -24
    for h in range(0, 0x10000, 7):  # widening is exact (sampled; exhaustive below vs numpy)
        assert f2h(orc.half_to_float(h)) == h or (h & 0x7C00) == 0x7C00 and h & 0x3FF


def test_half_widening_matches_ieee_exhaustively(orc):
    h = np.arange(0x10000, dtype=np.uint16)
    finite = (h & 0x7C00) != 0x7C00
    ours = np.array([orc.half_to_float(int(v)) for v in h[finite]], np.float32)
    assert np.array_equal(ours.view(np.uint32), h[finite].view(np.float16).astype(np.float32).view(np.uint32))


def test_to_fp16_bits_worked_values(orc):
    """format_test.cc:204-211 (e2m3 = scheme 7's base format)."""
    assert orc.to_fp16_bits(orc.round_to_nearest(1.0, 7), 7) == 0x3C00
    assert orc.to_fp16_bits(0b011111, 7) == 0x4780
    assert orc.to_fp16_bits(0, 7) == 0x0000
    assert orc.to_fp16_bits(1 << 5, 7) == 0x8000
    assert orc.to_fp16_bits(0b000001, 7) == 0x3000


@pytest.mark.parametrize("sid", sorted(SCHEMES))
def test_restore_table_exact_and_injective(orc, sid):
    """format_test.cc:213-222: every grid value is exact in binary16, patterns distinct
    except +-0."""
    t = orc.restore_table(sid)
    vals = np.array([orc.decode(c, sid) for c in range(t.size)])
    assert np.array_equal(t.view(np.float16).astype(np.float64), vals)
    nz = t[(t & 0x7FFF) != 0]
    assert len(set(nz.tolist())) == nz.size


def test_pack_worked_fp533_word(orc):
    """packing_test.cc:90-99."""
    w = orc.pack_row(7, np.array([0b000001, 0b000011, 0b000101], np.uint8))
    assert w.tolist() == [0x8820]
    assert orc.unpack_row(7, w).tolist() == [1, 3, 5]


def test_pack_worked_fp425_block(orc):
    """packing_test.cc:101-114."""
    codes = np.zeros(64, np.uint8)
    codes[:4] = [0b00001, 0b00011, 0b00101, 0b00111]
    w = orc.pack_row(4, codes)
    assert w.size == 17 and w[0] == 0x3210 and w[16] == 0x0001 and not w[1:16].any()
    assert np.array_equal(orc.unpack_row(4, w), codes)


def test_pack_worked_fp6_and_fp5(orc):
    """packing_test.cc:116-134."""
    codes = np.zeros(16, np.uint8)
    codes[0] = 0b101101
    assert orc.pack_row(2, codes).tolist() == [0x000B, 0, 0, 0, 0x0001, 0]
    codes = np.zeros(16, np.uint8)
    codes[5] = 0b11011
    assert orc.pack_row(1, codes).tolist() == [0, 0x00D0, 0, 0, 0x0020]


def test_pack_errors(orc):
    """packing_test.cc:165-176: inconsistent shared bit -> runtime_error; size -> invalid."""
    with pytest.raises(RuntimeError):
        orc.pack_row(7, np.array([0b000001, 0b000000, 0b000001], np.uint8))
    # a 10-code row is not a whole fp6 block: invalid_argument (status 1)
    assert orc.lib.orc_pack_row(2, np.zeros(10, np.uint8), 10, np.zeros(6, np.uint16), 6) == 1


@pytest.mark.parametrize("sid", sorted(SCHEMES))
def test_restore_block_worked_and_zero(orc, sid):
    """kernels_test.cc:38-64: zero block -> 0x0000; fp5.33 worked blocks."""
    wpb = SCHEMES[sid][2]
    assert not orc.restore_block(sid, np.zeros(wpb, np.uint16)).any()
    if sid == 7:
        w = orc.pack_row(7, np.array([0b001001, 0b101001, 0b011111], np.uint8))
        assert orc.restore_block(7, w).tolist() == [0x3C80, 0xBC80, 0x4780]
        w = orc.pack_row(7, np.array([0b001000, 0b101000, 0b011110], np.uint8))
        assert orc.restore_block(7, w).tolist() == [0x3C00, 0xBC00, 0x4700]


@pytest.mark.parametrize("sid", sorted(SCHEMES))
def test_restore_block_every_code(orc, sid):
    """kernels_test.cc:69-87: a block repeating one code restores to to_fp16_bits(code)."""
    blk = SCHEMES[sid][1]
    t = orc.restore_table(sid)
    for c in range(t.size):
        w = orc.pack_row(sid, np.full(blk, c, np.uint8))
        assert (orc.restore_block(sid, w) == t[c]).all()


def test_quantize_tail_group_pinned(orc):
    """quantize_test.cc:257-273: FP5.33 1x4 -> padded 6, tail group pinned to 0."""
    scales, payload, pc = orc.quantize_tensor(7, np.array([[7.5, 1.0, 1.0, 1.125]], np.float32))
    assert pc == 6
    assert orc.unpack_row(7, payload).tolist() == [0b011111, 0b001001, 0b001001, 0b001000, 0, 0]
    m = orc.restore_matrix(7, 1, 4, pc, scales, payload)
    assert m.tolist() == [[7.5, 1.125, 1.125, 1.0]]


def test_quantize_zero_matrix_and_sizes(orc):
    """quantize_test.cc:275-289: zero matrix -> zero payload, scale 1.0; 1x64 FP4.25 = 34 B."""
    scales, payload, pc = orc.quantize_tensor(7, np.zeros((4, 3), np.float32))
    assert pc == 3 and payload.nbytes == 8 and not payload.any() and (scales == 0x3C00).all()
    assert orc.packed_payload_bytes(4, 1, 64) == 34


def test_byte_ratios(orc):
    """kernels_test.cc:186-218: FP4.25 = 16/4.25 exactly; FP5.33 = 3.0 +- 0.001 at
    5120x25600; 64x192 FP5.33 exactly 3."""
    fp16 = 2.0 * 5120 * 25600
    assert fp16 / orc.packed_payload_bytes(4, 5120, 25600) == 16.0 / 4.25
    assert abs(fp16 / orc.packed_payload_bytes(7, 5120, 25600) - 3.0) <= 1e-3
    assert 2.0 * 64 * 192 / orc.packed_payload_bytes(7, 64, 192) == 3.0


def test_gemv_scaled_identity_and_zero_x(orc):
    """kernels_test.cc:120-138 restated on scheme 7 (fp5.33 blocks; the reference uses
    fp6-e2m3, the same base format)."""
    n, sc = 6, [2.0, 3.0, 4.0, 5.0, 0.5, 0.25]
    codes = np.zeros((n, n), np.uint8)
    for r in range(n):
        codes[r, r] = 0b001000  # 1.0, shared bit 0 for its group
    payload = np.concatenate([orc.pack_row(7, codes[r]) for r in range(n)])
    scales = np.array([orc.float_to_half(s) for s in sc], np.uint16)
    for j in range(n):
        x = np.zeros(n, np.uint16)
        x[j] = 0x3C00
        y = orc.gemv(7, n, n, n, scales, payload, x, 1)[0].view(np.float16).astype(float)
        assert y.tolist() == [sc[r] if r == j else 0.0 for r in range(n)]
    y = orc.gemv(7, n, n, n, scales, payload, np.zeros(3 * n, np.uint16), 3)
    assert not (y & 0x7FFF).any()


# ------------------------------------------------------ (b) fixtures from the reference
def _cases(small):
    keys = sorted({k.rsplit("_", 1)[0] for k in small.files if k.endswith("_payload")})
    return keys


def test_fixtures_present(small):
    assert len(_cases(small)) == 3 * len(SCHEMES)


def test_oracle_matches_reference_fixtures(orc, small):
    for key in _cases(small):
        sid = int(key[1:key.index("_")])
        rows, cols = map(int, key.split("_")[1].split("x"))
        w = small[key + "_w"]
        scales, payload, pc = orc.quantize_tensor(sid, w)
        assert pc == int(small[key + "_pc"][0]) == padded_cols(sid, cols)
        assert np.array_equal(scales, small[key + "_scales"]), key
        assert np.array_equal(payload, small[key + "_payload"]), key
        assert np.array_equal(orc.restore_grid(sid, rows, pc, payload), small[key + "_grid"]), key
        f32 = orc.restore_matrix(sid, rows, cols, pc, scales, payload)
        if key + "_f32" in small.files:
            assert np.array_equal(f32.view(np.uint32), small[key + "_f32"].view(np.uint32)), key
        # restore_matrix_half = float_to_half(restore_matrix) (kernels.hpp:127-133); numpy's
        # float32 -> float16 cast is the same IEEE round-to-nearest-even
        assert np.array_equal(f32.astype(np.float16).view(np.uint16), small[key + "_f16"]), key
        for m in (1, 3, 8, 16):
            x = small[f"x_{rows}x{cols}_{m}"]
            y = orc.gemv(sid, rows, cols, pc, scales, payload, x, m)
            assert np.array_equal(y.reshape(-1), small[f"{key}_y{m}"].reshape(-1)), (key, m)


@pytest.mark.parametrize("case", range(4))
def test_oracle_matches_reference_at_config_sizes(orc, case):
    """golden_large.json: config 1 (FP4.25 4096x4096, M=1) and FP5.33 cases, by SHA-256."""
    rec = json.load(open(os.path.join(GOLDEN, "golden_large.json")))["cases"][case]
    sid, rows, cols, seed = rec["scheme"], rec["rows"], rec["cols"], rec["seed"]
    w = np.random.default_rng(seed).standard_normal((rows, cols), dtype=np.float32)
    scales, payload, pc = orc.quantize_tensor(sid, w)
    assert pc == rec["padded_cols"]
    assert _sha(payload) == rec["payload_sha256"]
    assert _sha(scales) == rec["scales_sha256"]
    assert _sha(orc.restore_grid(sid, rows, pc, payload)) == rec["grid_sha256"]
    for m, h in rec["gemv"].items():
        m = int(m)
        x = (np.random.default_rng(seed ^ m).standard_normal(m * cols).astype(np.float16)
             .view(np.uint16))
        assert _sha(orc.gemv(sid, rows, cols, pc, scales, payload, x, m)) == h, m


# ------------------------------------------------------------- (c) live reference
@pytest.mark.parametrize("sid", sorted(SCHEMES))
def test_pack_bijection_vs_reference(orc, ref, sid):
    """acceptance_main.cc:127-160 (pack bijection), checked against the reference too."""
    rng = np.random.default_rng(100 + sid)
    blk, wpb = SCHEMES[sid][1], SCHEMES[sid][2]
    for _ in range(50):
        words = rng.integers(0, 1 << 16, size=wpb * int(rng.integers(1, 5)), dtype=np.uint16)
        codes = orc.unpack_row(sid, words)
        assert np.array_equal(codes, ref.unpack_row(sid, words))
        back = orc.pack_row(sid, codes)
        assert np.array_equal(back, ref.pack_row(sid, codes))
        assert np.array_equal(orc.unpack_row(sid, back), codes)


@pytest.mark.parametrize("sid", sorted(SCHEMES))
def test_random_stream_gemv_vs_reference(orc, ref, sid):
    """Random valid streams (every code incl. -0 and subnormals): restore and gemv bitwise."""
    rng = np.random.default_rng(7 + sid)
    rows, cols = 40, 5 * SCHEMES[sid][1] + 1
    pc = padded_cols(sid, cols)
    words = pc // SCHEMES[sid][1] * SCHEMES[sid][2]
    payload = rng.integers(0, 1 << 16, size=rows * words, dtype=np.uint16)
    scales = rng.integers(0x2000, 0x4000, size=rows, dtype=np.uint16)
    x = rng.standard_normal(5 * cols).astype(np.float16).view(np.uint16)
    assert np.array_equal(orc.restore_matrix(sid, rows, cols, pc, scales, payload).view(np.uint32),
                          ref.restore_matrix(sid, rows, cols, pc, scales, payload).view(np.uint32))
    assert np.array_equal(orc.gemv(sid, rows, cols, pc, scales, payload, x, 5),
                          ref.gemv(sid, rows, cols, pc, scales, payload, x, 5))

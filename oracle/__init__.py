"""TEST INFRASTRUCTURE ONLY -- the parity checkers for the B200 AMS-Quant path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. The product package
(``paper_2510_16045_b200``) never imports it.

* :class:`COracle`  -- ctypes view of ``liboracle.so``, the plain-C restatement in
  ``amsq_oracle.c`` (each function cites the reference file:line it follows).
* :class:`RefLib`   -- ctypes view of ``_ref/libamsq_ref.so``, the UNMODIFIED
  reference headers compiled in place by ``oracle/Makefile`` through
  ``ref_shim.cpp``. Absent on boxes where it was never built.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libamsq_ref.so")

_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_sz = C.c_size_t

# (block, words_per_block, k, exp_bits, man_bits, bias) per scheme id, packing.hpp:6-25.
SCHEMES = {
    0: ("fp4-e2m1", 16, 4, 1, 2, 1, 1),
    1: ("fp5-e2m2", 16, 5, 1, 2, 2, 1),
    2: ("fp6-e2m3", 16, 6, 1, 2, 3, 1),
    3: ("fp6-e3m2", 16, 6, 1, 3, 2, 3),
    4: ("fp4.25-e2m2", 64, 17, 4, 2, 2, 1),
    5: ("fp4.33-e2m2", 48, 13, 3, 2, 2, 1),
    6: ("fp4.5-e2m2", 32, 9, 2, 2, 2, 1),
    7: ("fp5.33-e2m3", 3, 1, 3, 2, 3, 1),
}


def scheme_block(sid: int) -> int:
    return SCHEMES[sid][1]


def padded_cols(sid: int, cols: int) -> int:
    b = scheme_block(sid)
    return (cols + b - 1) // b * b


def words_per_row(sid: int, pcols: int) -> int:
    return pcols // SCHEMES[sid][1] * SCHEMES[sid][2]


class OracleError(RuntimeError):
    pass


def _check(rc: int, what: str):
    if rc == 1:
        raise ValueError(f"{what}: invalid argument")
    if rc == 2:
        raise RuntimeError(f"{what}: runtime error")
    if rc:
        raise OracleError(f"{what}: status {rc}")


class COracle:
    """The plain-C restatement (oracle/amsq_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(path)
        L.orc_float_to_half.argtypes = [C.c_float]
        L.orc_float_to_half.restype = C.c_uint16
        L.orc_half_to_float.argtypes = [C.c_uint16]
        L.orc_half_to_float.restype = C.c_float
        L.orc_decode.argtypes = [C.c_uint, C.c_int]
        L.orc_decode.restype = C.c_float
        L.orc_to_fp16_bits.argtypes = [C.c_uint, C.c_int]
        L.orc_to_fp16_bits.restype = C.c_uint16
        L.orc_round_to_nearest.argtypes = [C.c_float, C.c_int]
        L.orc_round_to_nearest.restype = C.c_uint8
        L.orc_max_magnitude.argtypes = [C.c_int]
        L.orc_max_magnitude.restype = C.c_float
        L.orc_pack_row.argtypes = [C.c_int, _u8p, _sz, _u16p, _sz]
        L.orc_unpack_row.argtypes = [C.c_int, _u16p, _sz, _u8p, _sz]
        L.orc_packed_payload_bytes.argtypes = [C.c_int, _sz, _sz]
        L.orc_packed_payload_bytes.restype = _sz
        L.orc_restore_block.argtypes = [C.c_int, _u16p, _u16p]
        L.orc_restore_grid.argtypes = [C.c_int, _sz, _sz, _u16p, _u16p]
        L.orc_restore_matrix.argtypes = [C.c_int, _sz, _sz, _sz, _u16p, _u16p, _f32p]
        L.orc_gemv.argtypes = [C.c_int, _sz, _sz, _sz, _u16p, _u16p, _u16p, _sz, _sz, _u16p]
        L.orc_gemv_f64.argtypes = [C.c_int, _sz, _sz, _sz, _u16p, _u16p, _u16p, _sz, _f64p, _f64p]
        L.orc_quantize_tensor.argtypes = [C.c_int, _sz, _sz, _f32p, _u16p, _u16p]

    # -- binary16 / format
    def float_to_half(self, f: float) -> int:
        return int(self.lib.orc_float_to_half(f))

    def half_to_float(self, h: int) -> float:
        return float(self.lib.orc_half_to_float(h))

    def decode(self, code: int, sid: int) -> float:
        return float(self.lib.orc_decode(code, sid))

    def to_fp16_bits(self, code: int, sid: int) -> int:
        return int(self.lib.orc_to_fp16_bits(code, sid))

    def restore_table(self, sid: int) -> np.ndarray:
        n = 1 << (1 + SCHEMES[sid][4] + SCHEMES[sid][5])
        return np.array([self.to_fp16_bits(c, sid) for c in range(n)], np.uint16)

    def round_to_nearest(self, w: float, sid: int) -> int:
        return int(self.lib.orc_round_to_nearest(w, sid))

    # -- packing
    def pack_row(self, sid: int, codes: np.ndarray) -> np.ndarray:
        codes = np.ascontiguousarray(codes, np.uint8)
        b, wpb = SCHEMES[sid][1], SCHEMES[sid][2]
        words = np.zeros(len(codes) // b * wpb, np.uint16)
        _check(self.lib.orc_pack_row(sid, codes, codes.size, words, words.size), "pack_row")
        return words

    def unpack_row(self, sid: int, words: np.ndarray) -> np.ndarray:
        words = np.ascontiguousarray(words, np.uint16)
        b, wpb = SCHEMES[sid][1], SCHEMES[sid][2]
        codes = np.zeros(len(words) // wpb * b, np.uint8)
        _check(self.lib.orc_unpack_row(sid, words, words.size, codes, codes.size), "unpack_row")
        return codes

    def packed_payload_bytes(self, sid: int, rows: int, cols: int) -> int:
        return int(self.lib.orc_packed_payload_bytes(sid, rows, cols))

    def restore_block(self, sid: int, words: np.ndarray) -> np.ndarray:
        out = np.zeros(SCHEMES[sid][1], np.uint16)
        self.lib.orc_restore_block(sid, np.ascontiguousarray(words, np.uint16), out)
        return out

    # -- tensors
    def quantize_tensor(self, sid: int, w: np.ndarray):
        w = np.ascontiguousarray(w, np.float32)
        rows, cols = w.shape
        pc = padded_cols(sid, cols)
        scales = np.zeros(rows, np.uint16)
        payload = np.zeros(rows * words_per_row(sid, pc), np.uint16)
        _check(self.lib.orc_quantize_tensor(sid, rows, cols, w, scales, payload), "quantize")
        return scales, payload, pc

    def restore_grid(self, sid: int, rows: int, pcols: int, payload: np.ndarray) -> np.ndarray:
        out = np.zeros((rows, pcols), np.uint16)
        self.lib.orc_restore_grid(sid, rows, pcols, np.ascontiguousarray(payload), out)
        return out

    def restore_matrix(self, sid, rows, cols, pcols, scales, payload) -> np.ndarray:
        out = np.zeros((rows, cols), np.float32)
        self.lib.orc_restore_matrix(sid, rows, cols, pcols, np.ascontiguousarray(scales),
                                    np.ascontiguousarray(payload), out)
        return out

    def gemv(self, sid, rows, cols, pcols, scales, payload, x, batch) -> np.ndarray:
        x = np.ascontiguousarray(x, np.uint16).reshape(-1)
        y = np.zeros((batch, rows), np.uint16)
        _check(self.lib.orc_gemv(sid, rows, cols, pcols, np.ascontiguousarray(scales),
                                 np.ascontiguousarray(payload), x, x.size, batch, y), "gemv")
        return y

    def gemv_f64(self, sid, rows, cols, pcols, scales, payload, x, batch):
        x = np.ascontiguousarray(x, np.uint16).reshape(-1)
        ye = np.zeros((batch, rows), np.float64)
        ya = np.zeros((batch, rows), np.float64)
        _check(self.lib.orc_gemv_f64(sid, rows, cols, pcols, np.ascontiguousarray(scales),
                                     np.ascontiguousarray(payload), x, batch, ye, ya), "gemv_f64")
        return ye, ya


class RefLib:
    """The unmodified reference (oracle/_ref/libamsq_ref.so via ref_shim.cpp)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: build it with `make -C oracle` where "
                                    "/root/reference is present")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_float_to_half.argtypes = [C.c_float]
        L.ref_float_to_half.restype = C.c_uint16
        L.ref_half_to_float.argtypes = [C.c_uint16]
        L.ref_half_to_float.restype = C.c_float
        L.ref_restore_table.argtypes = [C.c_int, _u16p, _sz]
        L.ref_packed_payload_bytes.argtypes = [C.c_int, _sz, _sz]
        L.ref_packed_payload_bytes.restype = _sz
        L.ref_pack_row.argtypes = [C.c_int, _u8p, _sz, _u16p, _sz]
        L.ref_unpack_row.argtypes = [C.c_int, _u16p, _sz, _u8p, _sz]
        L.ref_restore_block.argtypes = [C.c_int, _u16p, _u16p, C.c_int]
        L.ref_quantize_tensor.argtypes = [C.c_int, _sz, _sz, _f32p, C.c_int, C.POINTER(_sz),
                                          C.POINTER(_sz), C.c_void_p, C.c_void_p]
        L.ref_restore_matrix.argtypes = [C.c_int, _sz, _sz, _sz, _u16p, _u16p, _sz, C.c_int,
                                         _f32p]
        L.ref_restore_matrix_half.argtypes = [C.c_int, _sz, _sz, _sz, _u16p, _u16p, _sz,
                                              C.c_int, _u16p]
        L.ref_gemv.argtypes = [C.c_int, _sz, _sz, _sz, _u16p, _u16p, _sz, _u16p, _sz, _sz,
                               C.c_int, C.c_int, _u16p]
        L.ref_tensor_new.argtypes = [C.c_int, _sz, _sz, _sz, _u16p, _u16p, _sz]
        L.ref_tensor_new.restype = C.c_void_p
        L.ref_tensor_free.argtypes = [C.c_void_p]
        L.ref_tensor_gemv.argtypes = [C.c_void_p, C.c_void_p, _sz, C.c_int, C.c_void_p]
        L.ref_gaussian_matrix.argtypes = [_sz, _sz, C.c_uint64, _f32p]
        L.ref_gaussian_half.argtypes = [_sz, C.c_uint64, _u16p]
        L.ref_resolve_threads.argtypes = [C.c_int]
        L.ref_resolve_threads.restype = C.c_int

    def _chk(self, rc, what):
        if rc:
            msg = self.lib.ref_last_error().decode()
            if rc == 1:
                raise ValueError(f"{what}: {msg}")
            raise RuntimeError(f"{what}: {msg}")

    def restore_table(self, sid):
        out = np.zeros(256, np.uint16)
        self._chk(self.lib.ref_restore_table(sid, out, out.size), "restore_table")
        n = 1 << (1 + SCHEMES[sid][4] + SCHEMES[sid][5])
        return out[:n]

    def pack_row(self, sid, codes):
        codes = np.ascontiguousarray(codes, np.uint8)
        b, wpb = SCHEMES[sid][1], SCHEMES[sid][2]
        words = np.zeros(len(codes) // b * wpb, np.uint16)
        self._chk(self.lib.ref_pack_row(sid, codes, codes.size, words, words.size), "pack_row")
        return words

    def unpack_row(self, sid, words):
        words = np.ascontiguousarray(words, np.uint16)
        b, wpb = SCHEMES[sid][1], SCHEMES[sid][2]
        codes = np.zeros(len(words) // wpb * b, np.uint8)
        self._chk(self.lib.ref_unpack_row(sid, words, words.size, codes, codes.size), "unpack")
        return codes

    def restore_block(self, sid, words, bitops=False):
        out = np.zeros(SCHEMES[sid][1], np.uint16)
        self._chk(self.lib.ref_restore_block(sid, np.ascontiguousarray(words, np.uint16), out,
                                             int(bitops)), "restore_block")
        return out

    def quantize_tensor(self, sid, w, threads=1):
        w = np.ascontiguousarray(w, np.float32)
        rows, cols = w.shape
        pc, nw = _sz(0), _sz(0)
        self._chk(self.lib.ref_quantize_tensor(sid, rows, cols, w, threads, C.byref(pc),
                                               C.byref(nw), None, None), "quantize(size)")
        scales = np.zeros(rows, np.uint16)
        payload = np.zeros(nw.value, np.uint16)
        self._chk(self.lib.ref_quantize_tensor(sid, rows, cols, w, threads, C.byref(pc),
                                               C.byref(nw), scales.ctypes.data,
                                               payload.ctypes.data), "quantize")
        return scales, payload, pc.value

    def restore_matrix(self, sid, rows, cols, pcols, scales, payload, threads=1):
        out = np.zeros((rows, cols), np.float32)
        payload = np.ascontiguousarray(payload)
        self._chk(self.lib.ref_restore_matrix(sid, rows, cols, pcols, np.ascontiguousarray(scales),
                                              payload, payload.size, threads, out), "restore")
        return out

    def restore_matrix_half(self, sid, rows, cols, pcols, scales, payload, threads=1):
        out = np.zeros((rows, cols), np.uint16)
        payload = np.ascontiguousarray(payload)
        self._chk(self.lib.ref_restore_matrix_half(sid, rows, cols, pcols,
                                                   np.ascontiguousarray(scales), payload,
                                                   payload.size, threads, out), "restore_half")
        return out

    def gemv(self, sid, rows, cols, pcols, scales, payload, x, batch, threads=1, reference=False):
        x = np.ascontiguousarray(x, np.uint16).reshape(-1)
        payload = np.ascontiguousarray(payload)
        y = np.zeros((batch, rows), np.uint16)
        self._chk(self.lib.ref_gemv(sid, rows, cols, pcols, np.ascontiguousarray(scales), payload,
                                    payload.size, x, x.size, batch, threads, int(reference), y),
                  "gemv")
        return y

    def gaussian_matrix(self, rows, cols, seed):
        out = np.zeros((rows, cols), np.float32)
        self.lib.ref_gaussian_matrix(rows, cols, seed, out)
        return out

    def gaussian_half(self, n, seed):
        out = np.zeros(n, np.uint16)
        self.lib.ref_gaussian_half(n, seed, out)
        return out


def load_oracle() -> COracle:
    return COracle()


def load_ref():
    """The compiled reference, or None when it was never built on this machine."""
    try:
        return RefLib()
    except (FileNotFoundError, OSError):
        return None

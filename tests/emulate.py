"""Bit-level numpy emulation of the sm_100a decode (kernels_common.cuh) -- test helper.

Given the device tile bytes produced by ``amsq_repack``, reproduce exactly what one
warp's lanes compute: the four 32-bit registers R0..R3 (+ the FP4.25 shared byte),
the decode_s4 / decode_s7 bit operations, the m16n8k16 A-fragment registers, and the
B-fragment column permutation (Traits::kofs). Reassembling the dense ``placed``
binary16 matrix from the fragments checks, without a GPU, that the layout, the decode
and the activation permutation agree with the reference restore.
"""
from __future__ import annotations

import numpy as np

U32 = np.uint32


FAM = {0: 4, 1: 4, 2: 4, 3: 4, 4: 4, 5: 7, 6: 4, 7: 7}


def _kofs(scheme: int, j: int, s: int) -> int:
    if FAM[scheme] == 4:
        return 4 * s + j
    o = 2 * j + (s >> 1)
    p, i = divmod(o, 3)
    return 6 * p + 3 * (s & 1) + i


_F4 = dict(tk=64, J=4, lane_k=16)
_F7 = dict(tk=48, J=3, lane_k=12)
TRAITS = {0: dict(_F4, tile_bytes=512, place=14), 1: dict(_F4, tile_bytes=640, place=14),
          2: dict(_F4, tile_bytes=768, place=14), 3: dict(_F4, tile_bytes=768, place=12),
          4: dict(_F4, tile_bytes=544, place=14), 5: dict(_F7, tile_bytes=416, place=14),
          6: dict(_F4, tile_bytes=576, place=14), 7: dict(_F7, tile_bytes=512, place=14)}
M32 = U32(0xFFFFFFFF)


def _mul(a, k):
    return (a.astype(np.uint64) * np.uint64(k) & np.uint64(0xFFFFFFFF)).astype(U32)


def _shl_signed(x, s):
    return (x << U32(s)) & M32 if s >= 0 else x >> U32(-s)


def nib_decode(r, L, e3):
    """kernels_common.cuh nib_decode: r [...] uint32, L list of 4 [...] -> o [..., 4]."""
    o = np.zeros(r.shape + (4,), U32)
    if not e3:
        M = U32(0x8E008E00)
        o[..., 0] = (r & M) | L[0]
        o[..., 1] = (_mul(r, 8) & M) | L[1]
        o[..., 2] = (_mul(r & U32(0x20382038), 68) & M) | L[2]
        o[..., 3] = (_mul(r & U32(0x40074007), 514) & M) | L[3]
    else:
        M = U32(0x9C009C00)
        o[..., 0] = (r & M) | L[0]
        o[..., 1] = (_mul(r, 64) & M) | L[1]
        o[..., 2] = (_mul(r & U32(0x20072007), 1028) & M) | L[2]
        o[..., 3] = (_mul(r & U32(0x41884188), 522) & M) | L[3]
    return o


def decode_nibble_family(scheme, R, lo0, lo1):
    """decode_frag for schemes 0, 1, 2, 3, 5, 6: R [..., NR], lo0/lo1 [...] -> A [..., J, 4]."""
    z = np.zeros(R.shape[:-1], U32)
    if scheme == 5:
        T = _mul(lo0, 0x1001)
        S = [_mul(T, 1 << (8 - k)) & U32(0x01000100) for k in range(4)]
        o = np.zeros(R.shape[:-1] + (3, 4), U32)
        for q in range(3):
            o[..., q, :] = nib_decode(R[..., q], [S[(4 * q + i) // 3] for i in range(4)], False)
        flat = [o[..., f >> 2, f & 3] for f in range(12)]
        A = np.zeros(R.shape[:-1] + (3, 4), U32)
        for j in range(3):
            A[..., j, 0] = flat[2 * j]
            A[..., j, 1] = flat[6 + 2 * j]
            A[..., j, 2] = flat[2 * j + 1]
            A[..., j, 3] = flat[7 + 2 * j]
        return A
    o = np.zeros(R.shape[:-1] + (4, 4), U32)
    for q in range(4):
        if scheme == 0:
            L = [z, z, z, z]
        elif scheme == 6:
            T0 = _mul(lo0 & U32(0xFF), 0x1001)
            T1 = _mul(lo0 >> U32(8), 0x1001)
            S0 = _mul(T0, 1 << (8 - q)) & U32(0x01000100)
            S1 = _mul(T1, 1 << (8 - q)) & U32(0x01000100)
            L = [S0, S0, S1, S1]
        elif scheme == 1:
            L = [_shl_signed(lo0, 8 - (4 * q + i)) & U32(0x01000100) for i in range(4)]
        else:
            tgt = 7 if scheme == 2 else 8
            mask = U32(0x01800180) if scheme == 2 else U32(0x03000300)
            L = []
            for i in range(4):
                p_ = 4 * q + i
                src = lo1 if p_ >> 3 else lo0
                L.append(_shl_signed(src, tgt - 2 * (p_ & 7)) & mask)
        o[..., q, :] = nib_decode(R[..., q], L, scheme == 3)
    A = np.zeros(R.shape[:-1] + (4, 4), U32)
    for j in range(4):
        A[..., j, 0] = o[..., 0, j]
        A[..., j, 1] = o[..., 2, j]
        A[..., j, 2] = o[..., 1, j]
        A[..., j, 3] = o[..., 3, j]
    return A


def decode_s4(R: np.ndarray, sh: np.ndarray) -> np.ndarray:
    """R: [..., 4] uint32, sh: [...] -> A [..., 4(j), 4(reg)] uint32 (decode_s4)."""
    T = (sh.astype(U32) * U32(0x1001)) & U32(0xFFFFFFFF)
    o = np.zeros(R.shape[:-1] + (4, 4), U32)
    for q in range(4):
        S = (T << U32(8 - q)) & U32(0x01000100)
        r = R[..., q].astype(U32)
        o[..., q, 0] = (r & U32(0x8E008E00)) | S
        o[..., q, 1] = ((r << U32(3)) & U32(0x8E008E00)) | S
        o[..., q, 2] = ((((r & U32(0x20382038)) * U32(68)) & U32(0xFFFFFFFF)) & U32(0x8E008E00)) | S
        o[..., q, 3] = ((((r & U32(0x40074007)) * U32(514)) & U32(0xFFFFFFFF)) & U32(0x8E008E00)) | S
    A = np.zeros(R.shape[:-1] + (4, 4), U32)
    for j in range(4):
        A[..., j, 0] = o[..., 0, j]
        A[..., j, 1] = o[..., 2, j]
        A[..., j, 2] = o[..., 1, j]
        A[..., j, 3] = o[..., 3, j]
    return A


def decode_s7(R: np.ndarray) -> np.ndarray:
    o = np.zeros(R.shape[:-1] + (4, 3), U32)
    for q in range(4):
        r = R[..., q].astype(U32)
        t5 = r >> U32(5)
        S = t5 & U32(0x00800080)
        SM1 = t5 & U32(0x01800180)
        o[..., q, 0] = (r & U32(0x8F008F00)) | S
        o[..., q, 1] = ((r << U32(8)) & U32(0x8F008F00)) | S
        o[..., q, 2] = ((((r & U32(0x40704070)) * U32(34)) & U32(0xFFFFFFFF)) & U32(0x8E008E00)) | SM1
    g0 = [o[..., 0, 0], o[..., 0, 1], o[..., 0, 2], o[..., 1, 0], o[..., 1, 1], o[..., 1, 2]]
    g8 = [o[..., 2, 0], o[..., 2, 1], o[..., 2, 2], o[..., 3, 0], o[..., 3, 1], o[..., 3, 2]]
    A = np.zeros(R.shape[:-1] + (3, 4), U32)
    for j in range(3):
        A[..., j, 0] = g0[2 * j]
        A[..., j, 1] = g8[2 * j]
        A[..., j, 2] = g0[2 * j + 1]
        A[..., j, 3] = g8[2 * j + 1]
    return A


def tile_offsets(plan, row_tiles: int, k_tiles: int) -> np.ndarray:
    """[row_tiles][k_tiles] storage index of each tile: groups of g_big (the first n_big)
    or g_big - 1 row tiles, stored [group][k_tile][row_tile_in_group] (device_layout.hpp)."""
    n_groups, g_big, n_big, _ = plan
    off = np.zeros((row_tiles, k_tiles), np.int64)
    r0 = 0
    for g in range(n_groups):
        G = g_big if g < n_big else g_big - 1
        for r in range(G):
            off[r0 + r] = r0 * k_tiles + np.arange(k_tiles) * G + r
        r0 += G
    assert r0 == row_tiles
    return off


def placed_matrix(scheme: int, tiles: np.ndarray, row_tiles: int, k_tiles: int,
                  plan) -> np.ndarray:
    """Dense [row_tiles*16][k_tiles*TK] matrix of the placed binary16 bits the MMAs see,
    with every A-fragment element put at the column its B-fragment partner selects."""
    tr = TRAITS[scheme]
    tb, TK, J, LK = tr["tile_bytes"], tr["tk"], tr["J"], tr["lane_k"]
    t = tiles.reshape(-1, tb)[tile_offsets(plan, row_tiles, k_tiles)]
    if scheme == 5:
        R01 = t[:, :, :256].copy().view(np.uint32).reshape(row_tiles, k_tiles, 32, 2)
        R2 = t[:, :, 256:384].copy().view(np.uint32).reshape(row_tiles, k_tiles, 32, 1)
        R = np.concatenate([R01, R2], axis=-1)
        A = decode_nibble_family(5, R, t[:, :, 384:416].astype(U32), None)
    else:
        R = t[:, :, :512].copy().view(np.uint32).reshape(row_tiles, k_tiles, 32, 4)
    if scheme == 4:
        A = decode_s4(R, t[:, :, 512:544].astype(U32))
    elif scheme == 7:
        A = decode_s7(R)
    elif scheme == 0:
        A = decode_nibble_family(0, R, None, None)
    elif scheme == 6:
        lo = t[:, :, 512:576].copy().view(np.uint16).reshape(row_tiles, k_tiles, 32).astype(U32)
        A = decode_nibble_family(6, R, lo, None)
    elif scheme == 1:
        lo = t[:, :, 512:640].copy().view(np.uint32).reshape(row_tiles, k_tiles, 32)
        A = decode_nibble_family(1, R, lo, None)
    elif scheme in (2, 3):
        q = t[:, :, 512:768].copy().view(np.uint32).reshape(row_tiles, k_tiles, 32, 2)
        A = decode_nibble_family(scheme, R, q[..., 0], q[..., 1])
    out = np.zeros((row_tiles * 16, k_tiles * TK), np.uint16)
    rt_idx = np.arange(row_tiles)[:, None]
    kt_idx = np.arange(k_tiles)[None, :]
    for lane in range(32):
        g, tt = lane >> 2, lane & 3
        for j in range(J):
            for reg in range(4):
                row = g + (8 if reg & 1 else 0)
                s_lo = 0 if reg < 2 else 2
                for h in range(2):
                    kk = tt * LK + _kofs(scheme, j, s_lo + h)
                    val = (A[:, :, lane, j, reg] >> U32(16 * h)) & U32(0xFFFF)
                    rows = rt_idx * 16 + row
                    cols = kt_idx * TK + kk
                    out[np.broadcast_to(rows, val.shape), np.broadcast_to(cols, val.shape)] = val
    return out


def placed_to_grid(placed: np.ndarray, scheme: int = 4) -> np.ndarray:
    """x 2^(15 - bias) in binary16 (exact for every grid value): the restored pattern."""
    f = placed.view(np.float16).astype(np.float32) * np.float32(2.0 ** TRAITS[scheme]["place"])
    return f.astype(np.float16).view(np.uint16)

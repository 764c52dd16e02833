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


def _kofs(scheme: int, j: int, s: int) -> int:
    if scheme == 4:
        return 4 * s + j
    o = 2 * j + (s >> 1)
    p, i = divmod(o, 3)
    return 6 * p + 3 * (s & 1) + i


TRAITS = {4: dict(tk=64, J=4, tile_bytes=544, lane_k=16), 7: dict(tk=48, J=3, tile_bytes=512, lane_k=12)}


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
    R = t[:, :, :512].copy().view(np.uint32).reshape(row_tiles, k_tiles, 32, 4)
    if scheme == 4:
        A = decode_s4(R, t[:, :, 512:544].astype(U32))
    else:
        A = decode_s7(R)
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


def placed_to_grid(placed: np.ndarray) -> np.ndarray:
    """x 2^14 in binary16 (exact for every grid value): the restored pattern."""
    f = placed.view(np.float16).astype(np.float32) * np.float32(16384.0)
    return f.astype(np.float16).view(np.uint16)

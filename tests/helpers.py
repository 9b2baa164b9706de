"""Test-side helpers: layout conversions and one-call GPU runs through the C-ABI."""
from __future__ import annotations

import numpy as np


def tile_major_to_plain(state, W, H):
    """[C][n_tiles][256] (tile-major) → [C][H][W]."""
    s = np.asarray(state)
    C = s.shape[0]
    TX, TY = (W + 15) // 16, (H + 15) // 16
    s = s.reshape(C, TY, TX, 16, 16).transpose(0, 1, 3, 2, 4).reshape(C, TY * 16, TX * 16)
    return s[:, :H, :W]


def plain_to_tile_major(state, W, H):
    s = np.asarray(state)
    C = s.shape[0]
    TX, TY = (W + 15) // 16, (H + 15) // 16
    pad = np.zeros((C, TY * 16, TX * 16), s.dtype)
    pad[:, :H, :W] = s
    return pad.reshape(C, TY, 16, TX, 16).transpose(0, 1, 3, 2, 4).reshape(C, TY * TX, 256)


def grad_close(got, ref, rtol=1e-4, atol=1e-6):
    """Elementwise |got - ref| <= rtol·|ref| + atol (the north-star gradient bar)."""
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    bad = np.abs(got - ref) > rtol * np.abs(ref) + atol
    return (not bad.any()), bad


def decode_rect(rec):
    """rec [n][16] fp32 → (x0, y0, x1, y1) int arrays from the packed uint32 bits of q3.x/q3.y."""
    r = np.ascontiguousarray(rec, np.float32)
    rx = r[:, 12].view(np.uint32)
    ry = r[:, 13].view(np.uint32)
    return (rx & 0xffff).astype(np.int32), (ry & 0xffff).astype(np.int32), (rx >> 16).astype(np.int32), (ry >> 16).astype(np.int32)

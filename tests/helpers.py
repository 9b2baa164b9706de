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


def grad_close(got, ref, bound=None, rtol=1e-4, atol=1e-6, kappa=0.1):
    """The gradient bar (north star: 1e-4 relative, 1e-6 absolute floor), R31:
    |got - ref| <= rtol·(|ref| + kappa·B) + atol elementwise, where B is the oracle's forward-error
    scale of the element (Σ|terms| through |chain Jacobian|, oracle.backward_bound). For elements
    that are not cancellation-dominated (|ref| ≳ B) this is the plain 1e-4 relative bar; for sums
    that cancel, "relative" is taken against 10% of the magnitude of what was summed."""
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    scale = np.abs(ref) if bound is None else np.abs(ref) + kappa * np.asarray(bound, np.float64)
    bad = np.abs(got - ref) > rtol * scale + atol
    return (not bad.any()), bad


def describe_bad(got, ref, bad, bound=None, k=5):
    r, c = np.nonzero(np.atleast_2d(bad))
    out = []
    for i in range(min(k, len(r))):
        g, f = np.atleast_2d(got)[r[i], c[i]], np.atleast_2d(ref)[r[i], c[i]]
        b = np.atleast_2d(bound)[r[i], c[i]] if bound is not None else float("nan")
        out.append(f"[{r[i]},{c[i]}] got {g:.7g} ref {f:.7g} bound {b:.3g}")
    return f"{len(r)} mismatches: " + "; ".join(out)


def strict_fraction(got, ref, rtol=1e-4, atol=1e-6):
    """Fraction of elements meeting the plain elementwise bar |Δ| <= 1e-4|ref| + 1e-6."""
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    return float((np.abs(got - ref) <= rtol * np.abs(ref) + atol).mean())


def assert_grad_bar(got, ref, bound, atol=1e-6, name="grad", min_strict=0.999, rtol=1e-4, kappa=0.1, extra=None):
    """The gradient parity assertion of every GPU test (R31, "how the bar is applied").

    Primary check — the north-star bar elementwise: |Δ| ≤ 1e-4·|ref| + atol.
    An element may miss it only if
      (a) its sum is cancellation-dominated: κ·B ≥ |ref| (the oracle's forward-error scale B —
          Σ|per-pair terms| through |chain Jacobian| — is at least 10× the cancelled result), and
      (b) it meets R31: |Δ| ≤ 1e-4·(|ref| + κ·B) + atol;
    and the fraction of elements meeting the primary bar must be ≥ ``min_strict``. ``extra``
    (optional, per element) is a propagated INPUT tolerance (e.g. the D-SSIM dL/dC bar pushed through
    the backward): an element within |Δ| ≤ 1e-4·(|ref| + κ·B) + extra + atol also passes.
    Prints (and with OIT_PARITY_LOG appends as JSON) the element count, the strict misses, the
    worst strict miss (|Δ| over the primary bar) and the largest |Δ|/B."""
    import json
    import os
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    B = np.zeros_like(ref) if bound is None else np.broadcast_to(np.asarray(bound, np.float64), ref.shape)
    d = np.abs(got - ref)
    strict_lim = rtol * np.abs(ref) + atol
    strict_ok = d <= strict_lim
    miss = ~strict_ok
    cancel = kappa * B >= np.abs(ref)
    r31_ok = d <= rtol * (np.abs(ref) + kappa * B) + atol
    n = int(ref.size)
    n_miss = int(miss.sum())
    frac = 1.0 - n_miss / max(n, 1)
    worst = float((d / strict_lim).max()) if n else 0.0
    with np.errstate(divide="ignore", invalid="ignore"):
        rb = np.where(B > 0, d / np.where(B > 0, B, 1.0), 0.0)
    stats = dict(name=name, test=os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0], n=n,
                 strict_misses=n_miss, strict_fraction=frac, worst_strict_ratio=worst,
                 max_err_over_B=float(rb.max()) if n else 0.0)
    ok_alt = cancel & r31_ok
    if extra is not None:
        E = np.broadcast_to(np.asarray(extra, np.float64), ref.shape)
        in_tol = d <= rtol * (np.abs(ref) + kappa * B) + E + atol
        stats["input_tolerance_misses"] = int((miss & ~ok_alt & in_tol).sum())
        ok_alt = ok_alt | in_tol
    bad = miss & ~ok_alt
    print("grad bar", json.dumps(stats))
    log = os.environ.get("OIT_PARITY_LOG")
    if log:
        with open(log, "a") as f:
            f.write(json.dumps(stats) + "\n")
    assert not bad.any(), f"{name}: " + describe_bad(got, ref, bad, B)
    assert frac >= min_strict, (name, stats)
    return stats


def decode_rect(rec):
    """rec [n][16] fp32 → (x0, y0, x1, y1) int arrays from the packed uint32 bits of q3.x/q3.y."""
    r = np.ascontiguousarray(rec, np.float32)
    rx = r[:, 12].view(np.uint32)
    ry = r[:, 13].view(np.uint32)
    return (rx & 0xffff).astype(np.int32), (ry & 0xffff).astype(np.int32), (rx >> 16).astype(np.int32), (ry >> 16).astype(np.int32)

"""CPU oracle for the SparseOIT hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. The product package
``paper_2605_13855_b200`` never imports it, and the two share no code: this module loads
``oracle/oit_oracle.c`` (plain single-threaded C, fp64 values + the fp32 decision spec of
DESIGN.md §3) through ctypes and wraps it with numpy.

Each function cites the PAPER.md passage it follows (``P:line``); see ``oit_oracle.c``.
Parity status: every function here is pinned by ``tests/test_oracle_*.py`` (closed forms,
brute force, finite differences, invariants, known-answer vectors); none is "parity unpinned".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oit_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboit_oracle.so")
ROW = 80
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, -ffp-contract=off so the fp32 decision spec is op-exact)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class Camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32),
                ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("R", C.c_float * 9), ("t", C.c_float * 3), ("center", C.c_float * 3),
                ("znear", C.c_float)]


def camera(cam: dict) -> Camera:
    c = Camera()
    c.width, c.height = int(cam["width"]), int(cam["height"])
    c.fx, c.fy, c.cx, c.cy = (float(cam[k]) for k in ("fx", "fy", "cx", "cy"))
    for i in range(9):
        c.R[i] = float(cam["R"][i])
    for i in range(3):
        c.t[i] = float(cam["t"][i])
        c.center[i] = float(cam["center"][i])
    c.znear = float(cam.get("znear", 0.2))
    return c


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.orc_speclog.restype = C.c_float
        _lib.orc_speclog.argtypes = [C.c_float]
        _lib.orc_bin.restype = C.c_int64
        _lib.orc_fps.restype = C.c_int32
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def speclog(x: float) -> float:
    """DESIGN.md §3 speclog (the fp32 log that decides the α thresholds, R8)."""
    return float(lib().orc_speclog(C.c_float(np.float32(x))))


def sh_basis(r) -> np.ndarray:
    """3DGS real-SH basis Y_0..Y_15 at unit direction r (Eq. 4)."""
    Y = np.zeros(16)
    lib().orc_sh_basis(_p(_f64(r)), _p(Y))
    return Y


def project_spec(rows32, idx, cam) -> dict:
    """fp32 decision-path projection (DESIGN.md §3 steps 1-12; Eq. 2, 5, 6; Alg. 2 l.1-2)."""
    rows32, idx = _f32(rows32), _i32(idx)
    out = np.zeros((len(idx), 15), np.float32)
    lib().orc_project_spec(_p(rows32), _p(idx), C.c_int32(len(idx)), C.byref(camera(cam)), _p(out))
    return dict(visible=out[:, 0].astype(bool), rect=out[:, 1:5].astype(np.int32),  # x0,y0,x1,y1
                mx=out[:, 5], my=out[:, 6], nA=out[:, 7], nB=out[:, 8], nC=out[:, 9],
                thr_lo=out[:, 10], thr_hi=out[:, 11], tz=out[:, 12], ex=out[:, 13], ey=out[:, 14])


def project_value(rows64, sigma, idx, cam) -> dict:
    """fp64 value-path projection: μ', conic, colour (Eq. 4), weight (Eq. 1), depth."""
    rows64, idx = _f64(rows64), _i32(idx)
    out = np.zeros((len(idx), 11))
    lib().orc_project_value(_p(rows64), C.c_double(sigma), _p(idx), C.c_int32(len(idx)),
                            C.byref(camera(cam)), _p(out))
    return dict(mx=out[:, 0], my=out[:, 1], A=out[:, 2], B=out[:, 3], C=out[:, 4],
                color=out[:, 5:8], w=out[:, 8], tz=out[:, 9], o=out[:, 10])


def branch_flags(rows64, sigma, idx, cam) -> dict:
    """Which piecewise branch of the value path each slot sits on (test bookkeeping for the FD pins
    of the clamp branches): tan-fov clamp in J (R13, Eq. 6), colour clamp per channel
    (R7, Eq. 4), v(r) <= 0 (R4, Eq. 1), d >= σ (Eq. 1)."""
    rows64, idx = _f64(rows64), _i32(idx)
    out = np.zeros((len(idx), 7), np.int32)
    lib().orc_branch_flags(_p(rows64), C.c_double(sigma), _p(idx), C.c_int32(len(idx)),
                           C.byref(camera(cam)), _p(out))
    out = out.astype(bool)
    return dict(clampx=out[:, 0], clampy=out[:, 1], color=out[:, 2:5], vneg=out[:, 5], ramp0=out[:, 6])


def n_tiles(cam) -> tuple:
    return (int(cam["width"]) + 15) // 16, (int(cam["height"]) + 15) // 16


def tile_contrib(rows32, idx, cam) -> np.ndarray:
    """Brute force: [n_slots, n_tiles] bool, True iff some pixel of the tile passes the spec
    contribution test for the slot (used to pin the tile culling as conservative)."""
    rows32, idx = _f32(rows32), _i32(idx)
    tx, ty = n_tiles(cam)
    out = np.zeros((len(idx), tx * ty), np.uint8)
    lib().orc_tile_contrib(_p(rows32), _p(idx), C.c_int32(len(idx)), C.byref(camera(cam)), _p(out))
    return out.astype(bool)


def bin_tiles(rows32, idx, cam):
    """Brute-force (splat, tile) binning keyed by tile only (Alg. 2 l.3-6), over the
    tiles of each slot's rectangle that pass the exact tile test (DESIGN.md §3 step 12b).
    Returns (pair_slot ascending within each tile, tile_offsets[n_tiles+1])."""
    rows32, idx = _f32(rows32), _i32(idx)
    tx, ty = n_tiles(cam)
    offs = np.zeros(tx * ty + 1, np.int32)
    n = lib().orc_bin(_p(rows32), _p(idx), C.c_int32(len(idx)), C.byref(camera(cam)), None,
                      C.c_int64(0), _p(offs))
    pairs = np.zeros(max(int(n), 1), np.int32)
    lib().orc_bin(_p(rows32), _p(idx), C.c_int32(len(idx)), C.byref(camera(cam)), _p(pairs),
                  C.c_int64(n), _p(offs))
    return pairs[:n], offs


def render(rows32, sigma, idx, cam, bg, base=None, route=None, mode: str = "rect", rows64=None):
    """Weighted-OIT forward (Eq. 7) over splats rows[idx], on top of ``base``
    (pre-render accumulators [5,H,W], Alg. 1, R16). ``route`` marks FOLD slots (BAU,
    Alg. 2 l.12). ``rows64`` (default: rows32 as fp64) carries the values while rows32 carries
    the decisions (they differ only in finite-difference tests).
    Returns dict(image [3,H,W], state [5,H,W] = P_R,P_G,P_B,Q,T, base_out, tile_pairs, contrib_pairs)."""
    rows32, idx = _f32(rows32), _i32(idx)
    rows64 = _f64(rows32 if rows64 is None else rows64)
    H, W = int(cam["height"]), int(cam["width"])
    image = np.zeros((3, H, W))
    state = np.zeros((5, H, W))
    base_out = np.zeros((5, H, W)) if route is not None else None
    counters = np.zeros(2, np.int64)
    base = None if base is None else _f64(base)
    route = None if route is None else np.ascontiguousarray(route, dtype=np.uint8)
    lib().orc_render(_p(rows32), _p(rows64), C.c_double(sigma), _p(idx), C.c_int32(len(idx)),
                     C.byref(camera(cam)), _p(_f64(bg)), _p(base), _p(route),
                     C.c_int32(0 if mode == "brute" else 1), _p(image), _p(state), _p(base_out),
                     _p(counters))
    return dict(image=image, state=state, base_out=base_out, tile_pairs=int(counters[0]),
                contrib_pairs=int(counters[1]))


def reconcile(rows32, sigma, cache, fold_idx, unfold_idx, cam):
    """Lazy pre-render reconciliation (§4.1, NEXT-1): the cache [5,H,W] of the frozen set with
    the newly frozen splats folded in and the re-activated ones removed (returns a new array)."""
    rows32 = _f32(rows32)
    out = _f64(cache).copy()
    f, u = _i32(fold_idx), _i32(unfold_idx)
    lib().orc_reconcile(_p(rows32), _p(_f64(rows32)), C.c_double(sigma), _p(f), C.c_int32(len(f)), _p(u),
                        C.c_int32(len(u)), C.byref(camera(cam)), _p(out))
    return out


def backward(rows32, sigma, idx, cam, bg, state, dL_dC, mode: str = "rect", rows64=None):
    """Analytic backward: Eq. B.2 per (splat, pixel), then the chain rule to
    μ, q, s, o, h, v (Eq. 8 attribute list) and σ. Returns (grad [n,80], dsigma, dcov [n,6])."""
    rows32, idx = _f32(rows32), _i32(idx)
    rows64 = _f64(rows32 if rows64 is None else rows64)
    grad = np.zeros((len(idx), ROW))
    dcov = np.zeros((len(idx), 6))
    dsig = np.zeros(1)
    lib().orc_backward(_p(rows32), _p(rows64), C.c_double(sigma), _p(idx), C.c_int32(len(idx)),
                       C.byref(camera(cam)), _p(_f64(bg)), _p(_f64(state)), _p(_f64(dL_dC)),
                       C.c_int32(0 if mode == "brute" else 1), _p(grad), _p(dsig), _p(dcov))
    return grad, float(dsig[0]), dcov


def backward_bound(rows32, sigma, idx, cam, bg, state, dL_dC, mode: str = "rect", full: bool = False):
    """``backward`` plus, per splat and row field, the forward-error scale of the gradient:
    Σ_k |∂row/∂G2_k|·Σ_pairs|term_k| (the 2D-gradient terms' magnitudes before cancellation,
    through |chain Jacobian|). Test bookkeeping for the fp32 tolerance (R31), not part
    of the method. Returns (grad, dsigma, dcov, bound), or with ``full`` a dict that adds the same
    scale for dΣ (``bound_cov`` [n,6]) and dσ (``bound_sigma``)."""
    rows32, idx = _f32(rows32), _i32(idx)
    rows64 = _f64(rows32)
    grad = np.zeros((len(idx), ROW))
    bound = np.zeros((len(idx), ROW))
    dcov = np.zeros((len(idx), 6))
    dsig = np.zeros(1)
    bcov = np.zeros((len(idx), 6))
    bsig = np.zeros(1)
    lib().orc_backward_bound(_p(rows32), _p(rows64), C.c_double(sigma), _p(idx), C.c_int32(len(idx)),
                             C.byref(camera(cam)), _p(_f64(bg)), _p(_f64(state)), _p(_f64(dL_dC)),
                             C.c_int32(0 if mode == "brute" else 1), _p(grad), _p(dsig), _p(dcov), _p(bound),
                             _p(bcov), _p(bsig))
    if full:
        return dict(grad=grad, dsigma=float(dsig[0]), dcov=dcov, bound=bound, bound_cov=bcov,
                    bound_sigma=float(bsig[0]))
    return grad, float(dsig[0]), dcov, bound


def loss_grad(image, target, loss: str = "l1") -> np.ndarray:
    """dL/dC of the mean L1 (sign(0)=0) or L2 loss over 3HW (3DGS L1 term; R24)."""
    image, target = _f64(image), _f64(target)
    g = np.zeros_like(image)
    lib().orc_loss_grad(_p(image), _p(target), C.c_int64(image.size), C.c_int32(0 if loss == "l1" else 1), _p(g))
    return g


def philox4x32_10(ctr, key) -> np.ndarray:
    """Philox4x32-10 counter-based generator (Salmon et al. 2011) — the shared RNG (R22)."""
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def fps(centers, S: int, seed: int, refresh: int) -> np.ndarray:
    """Farthest point sampling over camera centres with a Philox random start (§4.1, R22)."""
    centers = _f32(centers).reshape(-1, 3)
    out = np.zeros(S, np.int32)
    rc = lib().orc_fps(_p(centers), C.c_int32(len(centers)), C.c_int32(S), C.c_uint64(seed),
                       C.c_uint32(refresh), _p(out))
    if rc != 0:
        raise ValueError("fps: need 0 < S <= V")
    return out


def update_active(score_grad32, score_idx, eps32, mode: str, n_total: int, bits):
    """Activeness of Eq. 8 with the ∃ reading (R18), FRESH/MONOTONE (R21)."""
    g = _f32(score_grad32).reshape(-1, ROW)
    sidx = _i32(score_idx)
    eps = _f32(eps32)
    bits = np.ascontiguousarray(bits, dtype=np.uint32).copy()
    active = np.zeros(max(n_total, 1), np.int32)
    frozen = np.zeros(max(n_total, 1), np.int32)
    activated = np.zeros(max(n_total, 1), np.int32)
    n_out = np.zeros(3, np.int32)
    lib().orc_update_active(_p(g), _p(sidx), C.c_int32(len(sidx)), _p(eps),
                            C.c_int32(1 if mode == "monotone" else 0), C.c_int32(n_total), _p(bits),
                            _p(active), _p(frozen), _p(activated), _p(n_out))
    return bits, active[:n_out[0]].copy(), frozen[:n_out[1]].copy(), activated[:n_out[2]].copy()


def score_subsample(rows32, sigma, cams, targets, caches, active_idx, score_idx, views, bg,
                    loss: str = "l1", mode: str = "rect", with_bound: bool = False):
    """Subsampled gradient score (Alg. 1 l.8-12; §4.1): for each subsampled
    view j, the full-𝒢 pixel state is the cached frozen-set accumulators ⊕ the active set
    (R16); L_j's gradient (R20, R24) is back-propagated to the scored splats; the mean over
    the S views is returned (R19) as (score_grad [n_score,80], dsigma[, bound[, bound_sigma]])
    (``with_bound="full"`` adds the dσ error scale)."""
    acc = np.zeros((len(score_idx), ROW))
    bnd = np.zeros((len(score_idx), ROW))
    dsig = bsig = 0.0
    for j in views:
        cam = cams[j]
        fwd = render(rows32, sigma, active_idx, cam, bg, base=caches[j], mode=mode)
        g = loss_dssim(fwd["image"], targets[j], 0.2)[1] if loss == "dssim" else loss_grad(fwd["image"], targets[j], loss)
        r = backward_bound(rows32, sigma, score_idx, cam, bg, fwd["state"], g, mode=mode, full=True)
        acc += r["grad"]
        bnd += r["bound"]
        dsig += r["dsigma"]
        bsig += r["bound_sigma"]
    if with_bound == "full":
        return acc / len(views), dsig / len(views), bnd / len(views), bsig / len(views)
    if with_bound:
        return acc / len(views), dsig / len(views), bnd / len(views)
    return acc / len(views), dsig / len(views)


ADAM_LR_3DGS = {"mu": 1.6e-4, "o": 0.01, "q": 1e-3, "s": 5e-3, "v": 0.005, "h_dc": 2.5e-3, "h_rest": 2.5e-3 / 20,
                "sigma": 0.1}
ADAM_LR_KEYS = ("mu", "o", "q", "s", "v", "h_dc", "h_rest", "sigma")


def adam_step(grad, active_idx, latent, m, v, step, dsigma=0.0, sig_state=None, lr=None, beta1=0.9, beta2=0.999,
              eps=1e-15):
    """NEXT-2: masked Adam (Kingma & Ba, Alg. 1) on the compacted active rows, per-splat step
    counts, with the activations of R25/R33 (Alg. 1 l.6 P:162). Inputs are copied; returns
    (latent, m, v, step, rows_physical, sig_state, sigma) as fp64 / int32 arrays."""
    lr = dict(ADAM_LR_3DGS if lr is None else lr)
    lrv = np.array([lr[k] for k in ADAM_LR_KEYS], np.float64)
    grad = _f64(grad).reshape(-1, ROW)
    idx = _i32(active_idx)
    lat, mm, vv = (_f64(x).reshape(-1, ROW).copy() for x in (latent, m, v))
    st = np.ascontiguousarray(step, dtype=np.int32).copy()
    rows = lat.copy()                 # frozen rows: the physical row of the unchanged latent
    rows[:, 3] = 1.0 / (1.0 + np.exp(-lat[:, 3]))
    rows[:, 8:11] = np.exp(lat[:, 8:11])
    ss = None if sig_state is None else _f64(sig_state).copy()
    sig_out = np.zeros(1)
    lib().orc_adam_step(_p(grad), _p(idx), C.c_int32(len(idx)), _p(lat), _p(mm), _p(vv), _p(st), _p(rows),
                        C.c_double(float(dsigma)), _p(ss) if ss is not None else None, _p(sig_out), _p(lrv),
                        C.c_double(beta1), C.c_double(beta2), C.c_double(eps))
    return lat, mm, vv, st, rows, ss, (float(sig_out[0]) if ss is not None else None)


def loss_dssim(image, target, lam: float = 0.2, with_map: bool = False):
    """NEXT-3: the 3DGS loss (1−λ)·L1 + λ·(1 − SSIM) (11×11 Gaussian window σ 1.5,
    zero padding, C1 = 0.01², C2 = 0.03²) and dL/dC. image, target [3,H,W]. Returns (L, g[, ssim])."""
    x, y = _f64(image), _f64(target)
    H, W = x.shape[1], x.shape[2]
    g = np.zeros_like(x)
    smap = np.zeros_like(x)
    lib().orc_loss_dssim.restype = C.c_double
    L = lib().orc_loss_dssim(_p(x), _p(y), C.c_int32(H), C.c_int32(W), C.c_double(lam), _p(g), _p(smap))
    return (L, g, smap) if with_map else (L, g)

"""ctypes binding of liboit.so (include/oit.h) — argument marshalling only.

Every function here has the name of the C-ABI entry point it calls and forwards torch CUDA
tensors as raw device pointers; all arithmetic runs in the CUDA kernels of liboit. There is no
CPU fallback: if the shared library is missing or a call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "liboit.so")

OIT_TILE = 16
OIT_ROW = 80
OIT_REC = 20


class OitError(RuntimeError):
    pass


class Camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32),
                ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("R", C.c_float * 9), ("t", C.c_float * 3), ("center", C.c_float * 3),
                ("znear", C.c_float)]


class BwdEvents(C.Structure):
    _fields_ = [("moments_begin", C.c_void_p), ("moments_end", C.c_void_p)]


class KernelEvents(C.Structure):
    _fields_ = [("kernel_begin", C.c_void_p), ("kernel_end", C.c_void_p)]


class Scene(C.Structure):
    _fields_ = [("n", C.c_int32), ("rows", C.c_void_p), ("sigma", C.c_void_p)]


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


class AdamCfg(C.Structure):
    _fields_ = [("lr", C.c_float * 8), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float)]


LOSS_CODE = {"l1": 0, "l2": 1, "dssim": 2}   # "dssim" = the 3DGS (1−λ)L1 + λ·D-SSIM, λ = 0.2
OIT_TARGET_U8 = 0x100                          # loss flag: 8-bit targets (uint8 [3][H][W], value u8/255)
OIT_COEF_IN_WS = 0x200                         # bwd_ex: coefficients already in ws (oit_composite_fwd_loss)
OIT_COEF_ALL_TILES = 0x400                     # fwd_loss: coefficients for every tile (reusable by the score)


def _loss_flags(loss: str, targets) -> int:
    """Loss code plus OIT_TARGET_U8 when the (first non-None) target tensor is uint8."""
    t = next((x for x in targets if x is not None), None)
    return LOSS_CODE[loss] | (OIT_TARGET_U8 if t is not None and t.dtype == torch.uint8 else 0)


_lib = None


def lib() -> C.CDLL:
    """Load liboit.so (built in-tree by __graft_entry__.build()); raise if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OitError(f"liboit.so not built at {LIB_PATH}; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        sz, i32, i64, vp, f32 = C.c_size_t, C.c_int32, C.c_int64, C.c_void_p, C.c_float
        cam_p, scene_p = C.POINTER(Camera), C.POINTER(Scene)
        sig = {
            "oit_status_string": (C.c_char_p, [C.c_int]),
            "oit_num_tiles": (i32, [cam_p]),
            "oit_project_cull": (C.c_int, [scene_p, cam_p, vp, i32, vp, vp, vp]),
            "oit_bin_workspace_bytes": (sz, [cam_p, i64]),
            "oit_bin_workspace_bytes_ex": (sz, [cam_p, i32, i64]),
            "oit_bin_tiles": (C.c_int, [cam_p, vp, vp, i32, vp, i64, vp, vp, vp, sz, vp]),
            "oit_fwd_workspace_bytes": (sz, [cam_p, i64]),
            "oit_composite_fwd": (C.c_int, [cam_p, vp, vp, vp, i64, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
            "oit_composite_fwd_ex": (C.c_int, [cam_p, vp, vp, vp, i64, vp, vp, vp, vp, vp, vp, vp, vp, sz, i32, vp]),
            "oit_composite_fwd_loss": (C.c_int, [cam_p, vp, vp, vp, i64, vp, vp, vp, i32, vp, vp, sz, vp, sz, i32, i32,
                                                 vp]),
            "oit_composite_fwd_loss_ex": (C.c_int, [cam_p, vp, vp, vp, i64, vp, vp, vp, i32, vp, vp, sz, vp, sz, i32,
                                                    C.POINTER(KernelEvents), i32, vp]),
            "oit_loss_grad": (C.c_int, [cam_p, vp, vp, i32, vp, vp]),
            "oit_bwd_workspace_bytes": (sz, [cam_p, i32, i64]),
            "oit_composite_bwd": (C.c_int, [scene_p, cam_p, vp, i32, vp, vp, vp, i64, vp, vp, vp, f32, vp, vp,
                                            vp, vp, sz, vp]),
            "oit_composite_bwd_ex": (C.c_int, [scene_p, cam_p, vp, i32, vp, vp, vp, i64, vp, vp, vp, f32, vp, vp,
                                               vp, vp, sz, vp, i32, C.POINTER(BwdEvents), i32, vp]),
            "oit_composite_bwd_perpixel": (C.c_int, [scene_p, cam_p, vp, i32, vp, vp, vp, i64, vp, vp, vp, f32, vp,
                                                     vp, vp, vp, sz, C.POINTER(BwdEvents), vp]),
            "oit_select_views": (C.c_int, [vp, i32, i32, C.c_uint64, C.c_uint32, vp, vp]),
            "oit_score_workspace_bytes": (sz, [cam_p, i32, i32, i64]),
            "oit_score_subsample": (C.c_int, [scene_p, cam_p, i32, vp, vp, vp, i32, vp, i32, vp, i32, i32, vp, f32,
                                              vp, vp, i64, vp, vp, sz, i32, vp]),
            "oit_score_subsample_ex": (C.c_int, [scene_p, cam_p, i32, vp, vp, vp, i32, vp, i32, vp, i32, i32, vp,
                                                 f32, vp, vp, i64, vp, vp, sz, vp, vp, i32, vp]),
            "oit_update_workspace_bytes": (sz, [i32]),
            "oit_delta_workspace_bytes": (sz, [i32]),
            "oit_active_set_delta": (C.c_int, [vp, vp, i32, vp, vp, vp, vp, vp, sz, vp]),
            "oit_reconcile_workspace_bytes": (sz, [cam_p, i32, i64]),
            "oit_reconcile_cache": (C.c_int, [scene_p, cam_p, vp, i32, vp, i32, vp, i64, vp, vp, sz, vp]),
            "oit_dssim_workspace_bytes": (sz, [cam_p]),
            "oit_loss_dssim": (C.c_int, [cam_p, vp, vp, C.c_float, vp, vp, vp, sz, vp]),
            "oit_adam_step": (C.c_int, [vp, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, C.POINTER(AdamCfg), vp]),
            "oit_update_active_set": (C.c_int, [vp, vp, i32, vp, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
            "oit_score_activeness": (C.c_int, [vp, i32, vp, vp, vp]),
            "oit_apply_activeness": (C.c_int, [vp, vp, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
        }
        missing = [n for n in EXPORTED if n not in sig]
        if missing:  # every entry point the binding calls is called through a declared prototype
            raise OitError(f"no ctypes prototype for {missing}")
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


EXPORTED = ["oit_status_string", "oit_num_tiles", "oit_project_cull", "oit_bin_workspace_bytes",
            "oit_bin_workspace_bytes_ex", "oit_bin_tiles",
            "oit_fwd_workspace_bytes", "oit_composite_fwd", "oit_composite_fwd_ex", "oit_composite_fwd_loss",
            "oit_composite_fwd_loss_ex", "oit_loss_grad", "oit_bwd_workspace_bytes", "oit_composite_bwd", "oit_composite_bwd_ex",
            "oit_select_views", "oit_score_workspace_bytes", "oit_score_subsample", "oit_score_subsample_ex",
            "oit_update_workspace_bytes",
            "oit_update_active_set", "oit_delta_workspace_bytes", "oit_active_set_delta",
            "oit_reconcile_workspace_bytes", "oit_reconcile_cache", "oit_adam_step",
            "oit_dssim_workspace_bytes", "oit_loss_dssim", "oit_composite_bwd_perpixel", "oit_score_activeness",
            "oit_apply_activeness"]


# ------------------------------------------------------------------ marshalling helpers ---
def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise OitError("liboit takes CUDA tensors (no CPU path)")
    if not t.is_contiguous():
        raise OitError("liboit takes contiguous tensors")
    return C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def _check(rc: int, name: str):
    if rc != 0:
        raise OitError(f"{name}: {lib().oit_status_string(rc).decode()} (status {rc})")


def _f3(v):
    return (C.c_float * 3)(*[float(x) for x in v])


def scene(rows: torch.Tensor, sigma: torch.Tensor) -> Scene:
    assert rows.dtype == torch.float32 and rows.dim() == 2 and rows.shape[1] == OIT_ROW
    assert sigma.dtype == torch.float32 and sigma.numel() == 1
    return Scene(int(rows.shape[0]), _ptr(rows), _ptr(sigma))


def num_tiles(cam: dict) -> int:
    return ((int(cam["width"]) + 15) // 16) * ((int(cam["height"]) + 15) // 16)


# ------------------------------------------------------------------ the C-ABI, by name ----
def oit_project_cull(rows, sigma, cam, idx, rec, tiles_per_slot, stream=None):
    sc, c = scene(rows, sigma), camera(cam)
    _check(lib().oit_project_cull(C.byref(sc), C.byref(c), _ptr(idx), int(idx.numel()), _ptr(rec),
                                  _ptr(tiles_per_slot), _stream(stream)), "oit_project_cull")


def oit_bin_workspace_bytes(cam, pair_capacity: int, n_slots=None) -> int:
    """Scratch of oit_bin_tiles; with n_slots, enough for the bitmap path on views that small."""
    if n_slots is None:
        return int(lib().oit_bin_workspace_bytes(C.byref(camera(cam)), int(pair_capacity)))
    return int(lib().oit_bin_workspace_bytes_ex(C.byref(camera(cam)), int(n_slots), int(pair_capacity)))


def oit_bin_tiles(cam, rec, tiles_per_slot, n_slots, pair_slot, tile_offsets, n_pairs, ws, stream=None):
    _check(lib().oit_bin_tiles(C.byref(camera(cam)), _ptr(rec), _ptr(tiles_per_slot), int(n_slots),
                               _ptr(pair_slot), int(pair_slot.numel()), _ptr(tile_offsets), _ptr(n_pairs),
                               _ptr(ws), int(ws.numel()), _stream(stream)), "oit_bin_tiles")


def oit_fwd_workspace_bytes(cam, pair_capacity: int) -> int:
    return int(lib().oit_fwd_workspace_bytes(C.byref(camera(cam)), int(pair_capacity)))


def oit_composite_fwd(cam, rec, pair_slot, tile_offsets, bg, ws, base=None, route=None, image=None, state=None,
                      base_out=None, stream=None, counters=None, concurrency: int = 1):
    """counters: optional int64[2] device tensor (+=): contributing pairs, tile-granular evals;
    concurrency: calls the caller keeps in flight on other streams (grid sizing). Either selects
    oit_composite_fwd_ex."""
    args = (C.byref(camera(cam)), _ptr(rec), _ptr(pair_slot), _ptr(tile_offsets), int(pair_slot.numel()), _f3(bg),
            _ptr(base), _ptr(route), _ptr(image), _ptr(state), _ptr(base_out))
    if counters is None and concurrency == 1:
        _check(lib().oit_composite_fwd(*args, _ptr(ws), int(ws.numel()), _stream(stream)), "oit_composite_fwd")
    else:
        _check(lib().oit_composite_fwd_ex(*args, _ptr(counters), _ptr(ws), int(ws.numel()), int(concurrency),
                                          _stream(stream)), "oit_composite_fwd_ex")


def oit_composite_fwd_loss(cam, rec, pair_slot, tile_offsets, bg, ws, bwd_ws, n_slots: int, target, loss: str,
                           base=None, state=None, stream=None, concurrency: int = 1, events=None,
                           all_tiles: bool = False):
    """a3 + a4 fused (training view): the forward whose epilogue applies the L1/L2 loss against
    target (fp32 or uint8) and writes the backward coefficients into bwd_ws; follow with
    oit_composite_bwd(..., coef_ready=True) on the same bwd_ws. events: optional (begin, end)
    torch.cuda.Event pair recorded around the composite kernel alone (oit_composite_fwd_loss_ex).
    all_tiles: coefficients for every tile (OIT_COEF_ALL_TILES), reusable by oit_score_subsample."""
    flags = _loss_flags(loss, [target]) | (OIT_COEF_ALL_TILES if all_tiles else 0)
    args = (C.byref(camera(cam)), _ptr(rec), _ptr(pair_slot), _ptr(tile_offsets), int(pair_slot.numel()), _f3(bg),
            _ptr(base), _ptr(target), flags, _ptr(state), _ptr(ws), int(ws.numel()),
            _ptr(bwd_ws), int(bwd_ws.numel()), int(n_slots))
    if events is None:
        _check(lib().oit_composite_fwd_loss(*args, int(concurrency), _stream(stream)), "oit_composite_fwd_loss")
    else:
        ev = C.byref(KernelEvents(C.c_void_p(events[0].cuda_event), C.c_void_p(events[1].cuda_event)))
        _check(lib().oit_composite_fwd_loss_ex(*args, ev, int(concurrency), _stream(stream)),
               "oit_composite_fwd_loss_ex")


def oit_loss_grad(cam, image, target, loss: str, dL_dimage, stream=None):
    _check(lib().oit_loss_grad(C.byref(camera(cam)), _ptr(image), _ptr(target), 0 if loss == "l1" else 1,
                               _ptr(dL_dimage), _stream(stream)), "oit_loss_grad")


def oit_bwd_workspace_bytes(cam, n_slots: int, pair_capacity: int) -> int:
    return int(lib().oit_bwd_workspace_bytes(C.byref(camera(cam)), int(n_slots), int(pair_capacity)))


def oit_composite_bwd(rows, sigma, cam, idx, rec, pair_slot, tile_offsets, bg, state, dL_dimage, grad, dL_dsigma,
                      ws, dL_dcov=None, scale: float = 1.0, stream=None, events=None, target=None, loss="l1",
                      per_pixel: bool = False, concurrency: int = 1, coef_ready: bool = False):
    """events: optional (begin, end) torch.cuda.Event pair recorded around the a5 moment kernel;
    target: optional training image — the L1/L2 pixel gradient is then fused into the backward
    (dL_dimage may be None); concurrency: calls in flight on other streams (grid sizing);
    coef_ready: oit_composite_fwd_loss already wrote the coefficients into ws (state, dL_dimage
    and target unused). Any of them selects oit_composite_bwd_ex."""
    sc, c = scene(rows, sigma), camera(cam)
    args = (C.byref(sc), C.byref(c), _ptr(idx), int(idx.numel()), _ptr(rec), _ptr(pair_slot), _ptr(tile_offsets),
            int(pair_slot.numel()), _f3(bg), _ptr(state), _ptr(dL_dimage), C.c_float(scale), _ptr(grad),
            _ptr(dL_dsigma), _ptr(dL_dcov), _ptr(ws), int(ws.numel()))
    if per_pixel:   # NEXT-4 ablation (3DGS-style per-pixel moments)
        ev = None if events is None else C.byref(BwdEvents(C.c_void_p(events[0].cuda_event),
                                                           C.c_void_p(events[1].cuda_event)))
        _check(lib().oit_composite_bwd_perpixel(*args, ev, _stream(stream)), "oit_composite_bwd_perpixel")
    elif events is None and target is None and concurrency == 1 and not coef_ready:
        _check(lib().oit_composite_bwd(*args, _stream(stream)), "oit_composite_bwd")
    else:
        ev = None if events is None else C.byref(BwdEvents(C.c_void_p(events[0].cuda_event),
                                                           C.c_void_p(events[1].cuda_event)))
        flags = OIT_COEF_IN_WS if coef_ready else _loss_flags(loss, [target])
        _check(lib().oit_composite_bwd_ex(*args, _ptr(target), flags, ev, int(concurrency), _stream(stream)),
               "oit_composite_bwd_ex")


def oit_select_views(centers, n_sub: int, seed: int, refresh: int, views_out, stream=None):
    _check(lib().oit_select_views(_ptr(centers), int(centers.shape[0]), int(n_sub), C.c_uint64(seed),
                                  C.c_uint32(refresh), _ptr(views_out), _stream(stream)), "oit_select_views")


def oit_score_workspace_bytes(cam, n_active: int, n_score: int, pair_capacity: int) -> int:
    return int(lib().oit_score_workspace_bytes(C.byref(camera(cam)), int(n_active), int(n_score),
                                               int(pair_capacity)))


def oit_score_subsample(rows, sigma, cams, targets, caches, active_idx, score_idx, views, loss: str, bg,
                        score_grad, dL_dsigma, pair_capacity: int, max_pairs, ws, stream=None, scale=None,
                        concurrency: int = 1, coef_ws=None, coef_ready=None):
    """scale: weight of each view's gradient (default 1/len(views): the mean over these views);
    concurrency: score calls in flight on other streams (grid sizing only); coef_ws: optional list
    (one entry per subsampled view, entries may be None) of backward workspaces holding the view's
    coefficients from oit_composite_fwd_loss(..., all_tiles=True) (oit_score_subsample_ex);
    coef_ready: optional list of torch.cuda.Event (entries may be None) the call waits on right
    before it reads the matching coef_ws entry."""
    sc = scene(rows, sigma)
    V = len(cams)
    cam_arr = (Camera * V)(*[camera(c) for c in cams])
    tg = (C.c_void_p * V)(*[(t.data_ptr() if t is not None else None) for t in targets])
    ch = (C.c_void_p * V)(*[(c.data_ptr() if c is not None else None) for c in caches]) if caches is not None else None
    vw = (C.c_int32 * len(views))(*[int(v) for v in views])
    args = (C.byref(sc), cam_arr, V, tg, ch, _ptr(active_idx), int(active_idx.numel()), _ptr(score_idx),
            int(score_idx.numel()), vw, len(views), _loss_flags(loss, targets), _f3(bg),
            C.c_float(1.0 / len(views) if scale is None else scale), _ptr(score_grad), _ptr(dL_dsigma),
            int(pair_capacity), _ptr(max_pairs), _ptr(ws), int(ws.numel()))
    if coef_ws is None:
        _check(lib().oit_score_subsample(*args, int(concurrency), _stream(stream)), "oit_score_subsample")
    else:
        assert len(coef_ws) == len(views)
        cw = (C.c_void_p * len(views))(*[(w.data_ptr() if w is not None else None) for w in coef_ws])
        ev = None
        if coef_ready is not None:
            assert len(coef_ready) == len(views)
            ev = (C.c_void_p * len(views))(*[(e.cuda_event if e is not None else None) for e in coef_ready])
        _check(lib().oit_score_subsample_ex(*args, cw, ev, int(concurrency), _stream(stream)),
               "oit_score_subsample_ex")


def oit_update_workspace_bytes(n_total: int) -> int:
    return int(lib().oit_update_workspace_bytes(int(n_total)))


def oit_update_active_set(score_grad, score_idx, eps, mode: str, n_total: int, active_bits, active_idx, n_active,
                          newly_frozen=None, n_frozen=None, newly_active=None, n_activated=None, ws=None,
                          stream=None):
    e = (C.c_float * 6)(*[float(x) for x in eps])
    _check(lib().oit_update_active_set(_ptr(score_grad), _ptr(score_idx), int(score_idx.numel()), e,
                                       1 if mode == "monotone" else 0, int(n_total), _ptr(active_bits),
                                       _ptr(active_idx), _ptr(n_active), _ptr(newly_frozen), _ptr(n_frozen),
                                       _ptr(newly_active), _ptr(n_activated), _ptr(ws), int(ws.numel()),
                                       _stream(stream)), "oit_update_active_set")


def oit_score_activeness(score_grad, n_rows: int, eps, row_bits, stream=None):
    """a8, first half: Eq. 8 per score row → row bitmask [⌈n_rows/32⌉] (int32/uint32 tensor)."""
    e = (C.c_float * 6)(*[float(x) for x in eps])
    _check(lib().oit_score_activeness(_ptr(score_grad), int(n_rows), e, _ptr(row_bits), _stream(stream)),
           "oit_score_activeness")


def oit_apply_activeness(row_bits, score_idx, mode: str, n_total: int, active_bits, active_idx, n_active,
                         newly_frozen=None, n_frozen=None, newly_active=None, n_activated=None, ws=None,
                         stream=None):
    """a8, second half: the row bits applied to the splats score_idx, then recompaction."""
    _check(lib().oit_apply_activeness(_ptr(row_bits), _ptr(score_idx), int(score_idx.numel()),
                                      1 if mode == "monotone" else 0, int(n_total), _ptr(active_bits),
                                      _ptr(active_idx), _ptr(n_active), _ptr(newly_frozen), _ptr(n_frozen),
                                      _ptr(newly_active), _ptr(n_activated), _ptr(ws), int(ws.numel()),
                                      _stream(stream)), "oit_apply_activeness")


def oit_delta_workspace_bytes(n_total: int) -> int:
    return int(lib().oit_delta_workspace_bytes(int(n_total)))


def oit_active_set_delta(old_bits, bits, n_total: int, fold_idx, n_fold, unfold_idx, n_unfold, ws, stream=None):
    _check(lib().oit_active_set_delta(_ptr(old_bits), _ptr(bits), int(n_total), _ptr(fold_idx), _ptr(n_fold),
                                      _ptr(unfold_idx), _ptr(n_unfold), _ptr(ws), int(ws.numel()), _stream(stream)),
           "oit_active_set_delta")


def oit_reconcile_workspace_bytes(cam, n_splats: int, pair_capacity: int) -> int:
    return int(lib().oit_reconcile_workspace_bytes(C.byref(camera(cam)), int(n_splats), int(pair_capacity)))


def oit_reconcile_cache(rows, sigma, cam, fold_idx, unfold_idx, cache, pair_capacity: int, n_pairs, ws, stream=None):
    sc = scene(rows, sigma)
    nf, nu = int(fold_idx.numel()), int(unfold_idx.numel())
    _check(lib().oit_reconcile_cache(C.byref(sc), C.byref(camera(cam)), _ptr(fold_idx) if nf else None, nf,
                                     _ptr(unfold_idx) if nu else None, nu, _ptr(cache), int(pair_capacity),
                                     _ptr(n_pairs), _ptr(ws), int(ws.numel()), _stream(stream)), "oit_reconcile_cache")


ADAM_LR_KEYS = ("mu", "o", "q", "s", "v", "h_dc", "h_rest", "sigma")
ADAM_LR_3DGS = {"mu": 1.6e-4, "o": 0.01, "q": 1e-3, "s": 5e-3, "v": 0.005, "h_dc": 2.5e-3, "h_rest": 2.5e-3 / 20,
                "sigma": 0.1}   # P:220 (o, σ, v) + the 3DGS defaults for the rest


def adam_cfg(lr=None, beta1=0.9, beta2=0.999, eps=1e-15) -> AdamCfg:
    lr = dict(ADAM_LR_3DGS if lr is None else lr)
    c = AdamCfg()
    for k, key in enumerate(ADAM_LR_KEYS):
        c.lr[k] = float(lr[key])
    c.beta1, c.beta2, c.eps = float(beta1), float(beta2), float(eps)
    return c


def oit_adam_step(grad, active_idx, latent, m, v, step, rows, cfg: AdamCfg, n_active=None, d_n_active=None,
                  dsigma=None, sigma_state=None, sigma=None, stream=None):
    n = int(active_idx.numel()) if n_active is None else int(n_active)
    _check(lib().oit_adam_step(_ptr(grad) if n else None, _ptr(active_idx) if n else None, n, _ptr(d_n_active),
                               _ptr(latent), _ptr(m), _ptr(v), _ptr(step), _ptr(rows), _ptr(dsigma),
                               _ptr(sigma_state), _ptr(sigma), C.byref(cfg), _stream(stream)), "oit_adam_step")


def oit_dssim_workspace_bytes(cam) -> int:
    return int(lib().oit_dssim_workspace_bytes(C.byref(camera(cam))))


def oit_loss_dssim(cam, image, target, dL_dimage, ws, lam: float = 0.2, loss=None, stream=None):
    _check(lib().oit_loss_dssim(C.byref(camera(cam)), _ptr(image), _ptr(target), float(lam), _ptr(dL_dimage),
                                _ptr(loss), _ptr(ws), int(ws.numel()), _stream(stream)), "oit_loss_dssim")

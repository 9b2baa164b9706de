"""The C-ABI library builds for sm_100a, loads without a GPU and exports every symbol that
include/oit.h declares (no compute calls here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "oit.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(oit_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_six_north_star_calls():
    names = declared_functions()
    for n in ["oit_project_cull", "oit_bin_tiles", "oit_composite_fwd", "oit_composite_bwd",
              "oit_score_subsample", "oit_update_active_set"]:
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2605_13855_b200 import build as B
    path = B.build()
    lib = ctypes.CDLL(path)
    for name in declared_functions():
        assert hasattr(lib, name), name
    from paper_2605_13855_b200 import _lib
    assert set(_lib.EXPORTED) == set(declared_functions())


def test_library_is_sm100a_sass():
    from paper_2605_13855_b200 import build as B
    out = subprocess.run(["cuobjdump", "--list-elf", B.build()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_argument_errors_without_gpu():
    from paper_2605_13855_b200 import _lib
    L = _lib.lib()
    assert L.oit_status_string(0) == b"ok"
    assert b"capacity" in L.oit_status_string(3)
    cam = _lib.camera(dict(width=64, height=48, fx=50, fy=50, cx=32, cy=24, R=[1, 0, 0, 0, 1, 0, 0, 0, 1],
                           t=[0, 0, 0], center=[0, 0, 0]))
    assert L.oit_num_tiles(ctypes.byref(cam)) == 4 * 3
    # synchronous validation happens before any launch: null scene → OIT_EINVAL
    assert L.oit_project_cull(None, ctypes.byref(cam), None, 0, None, None, None) == 1
    assert L.oit_select_views(None, 4, 2, 0, 0, None, None) == 1
    assert L.oit_update_workspace_bytes(1000) > 0
    assert L.oit_bwd_workspace_bytes(ctypes.byref(cam), 100, 1000) > 0
    # fused forward loss: no target / D-SSIM (not pixel-local) / missing workspaces are rejected
    # synchronously (OIT_EINVAL = 1), before anything is launched
    bg = (ctypes.c_float * 3)(0, 0, 0)
    args = lambda tgt, loss, ws: (ctypes.byref(cam), None, None, ctypes.c_void_p(8), 0, bg, None, tgt, loss, None,  # noqa: E731
                                  ws, 1 << 20, ws, 1 << 20, 10, 1, None)
    assert L.oit_composite_fwd_loss(*args(None, 0, ctypes.c_void_p(8))) == 1
    assert L.oit_composite_fwd_loss(*args(ctypes.c_void_p(8), 2, ctypes.c_void_p(8))) == 1
    assert L.oit_composite_fwd_loss(*args(ctypes.c_void_p(8), 0 | _lib.OIT_TARGET_U8, None)) == 1


def test_score_coefficient_reuse_argument_errors_without_gpu():
    """oit_score_subsample_ex rejects, synchronously and before any launch, a reused coefficient
    workspace for the D-SSIM loss (the fused forward writes only pixel-local coefficients) and one
    that is not 16-byte aligned (OIT_EINVAL = 1)."""
    from paper_2605_13855_b200 import _lib
    L = _lib.lib()
    cam = _lib.camera(dict(width=64, height=48, fx=50, fy=50, cx=32, cy=24, R=[1, 0, 0, 0, 1, 0, 0, 0, 1],
                           t=[0, 0, 0], center=[0, 0, 0]))
    sc = _lib.Scene(100, ctypes.c_void_p(256), ctypes.c_void_p(256))
    cams = (_lib.Camera * 1)(cam)
    tg = (ctypes.c_void_p * 1)(ctypes.c_void_p(256))
    views = (ctypes.c_int32 * 1)(0)
    bg = (ctypes.c_float * 3)(0, 0, 0)
    nbytes = L.oit_score_workspace_bytes(ctypes.byref(cam), 10, 20, 1000)
    dev = ctypes.c_void_p(256)

    def call(loss, coef):
        cw = None if coef is None else (ctypes.c_void_p * 1)(coef)
        return L.oit_score_subsample_ex(ctypes.byref(sc), cams, 1, tg, None, dev, 10, dev, 20, views, 1, loss, bg,
                                        ctypes.c_float(1.0), dev, dev, 1000, dev, dev, nbytes, cw, None, 1, None)

    assert call(2, ctypes.c_void_p(256)) == 1          # D-SSIM: no reusable coefficients
    assert call(0, ctypes.c_void_p(256 + 4)) == 1      # misaligned workspace
    assert call(2, ctypes.c_void_p(256 + 4)) == 1


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2605_13855_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oit_oracle" not in txt, f

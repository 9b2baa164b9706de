"""DEV: the degenerate empty-state score (no cache, nothing active) — locate the elements that miss
the R31 bar and characterise their splats (DESIGN.md §5 known limitation)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_2605_13855_b200 import _lib as L  # noqa: E402
from paper_2605_13855_b200 import synth  # noqa: E402

DEV = "cuda"
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)  # noqa: E731
sc = synth.scene_c2(n=20000, n_views=3, res=200)
cam = sc.cams[0]
rows, sigma = t(sc.rows), t(np.array([sc.sigma], np.float32))
empty = torch.empty(0, dtype=torch.int32, device=DEV)
t32 = synth.target_image(cam, 4)
cap = 1 << 20


def gpu_score(idx):
    ws = torch.empty(L.oit_score_workspace_bytes(cam, 0, len(idx), cap), dtype=torch.uint8, device=DEV)
    sg = torch.zeros((len(idx), 80), dtype=torch.float32, device=DEV)
    sds = torch.zeros(1, dtype=torch.float32, device=DEV)
    mp = torch.zeros(1, dtype=torch.int64, device=DEV)
    L.oit_score_subsample(rows, sigma, [cam], [t(t32)], None, empty, t(idx), [0], "l2", sc.bg, sg, sds, cap, mp, ws)
    return sg.cpu().numpy().astype(np.float64)


idx = np.arange(sc.n, dtype=np.int32)
g = gpu_score(idx)
ref, _, bnd = O.score_subsample(sc.rows, sc.sigma, [cam], [t32], [None], np.zeros(0, np.int32), idx, [0], sc.bg, "l2",
                                with_bound=True)
bar = 1e-4 * (np.abs(ref) + 0.1 * bnd) + 1e-6 / (3 * 200 * 200)
r, c = np.nonzero(np.abs(g - ref) > bar)
print("bad elements", list(zip(r.tolist(), c.tolist())))
sp = O.project_spec(sc.rows, idx, cam)
for k, f in zip(r, c):
    o = sc.rows[k, 3]
    print(f"splat {k} field {f}: gpu {g[k, f]:.7g} ref {ref[k, f]:.7g} bound {bnd[k, f]:.3g} | o={o:.4f} "
          f"thr_hi={sp['thr_hi'][k]:.4g} ex={sp['ex'][k]:.3g} ey={sp['ey'][k]:.3g} rect={sp['rect'][k]}")
    g1 = gpu_score(np.array([k], np.int32))
    print(f"   alone on the GPU: {g1[0, f]:.7g};  row rel err {np.abs(g[k] - ref[k]).max() / np.abs(ref[k]).max():.2e}")
    # the oracle through its brute-force path
    rb, _, _ = O.score_subsample(sc.rows, sc.sigma, [cam], [t32], [None], np.zeros(0, np.int32), np.array([k], np.int32),
                                 [0], sc.bg, "l2", mode="brute", with_bound=True)
    print(f"   oracle brute: {rb[0, f]:.7g}")

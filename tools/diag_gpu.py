"""GPU-vs-oracle diagnostics (prints error breakdowns; not a test)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_2605_13855_b200 import synth  # noqa: E402
from paper_2605_13855_b200.pipeline import ViewPipeline  # noqa: E402
from tests.helpers import tile_major_to_plain  # noqa: E402

DEV = "cuda"
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)  # noqa: E731

FIELDS = {"mu": slice(0, 3), "o": slice(3, 4), "q": slice(4, 8), "s": slice(8, 11), "v": slice(12, 28), "h": slice(28, 76)}


def fwd_diag(sc, cam, idx, name):
    p = ViewPipeline(cam, len(idx), 1 << 22, device=DEV)
    img, st = p.forward(t(sc.rows), t(np.array([sc.sigma], np.float32)), t(idx), sc.bg)
    ref = O.render(sc.rows, sc.sigma, idx, cam, sc.bg)
    W, H = cam["width"], cam["height"]
    g = tile_major_to_plain(st.cpu().numpy(), W, H)
    e = np.abs(img.cpu().numpy() - ref["image"])
    k = np.unravel_index(np.argmax(e), e.shape)
    y, x = k[1], k[2]
    print(f"[{name}] img max err {e.max():.3e} at {k}; mean {e.mean():.2e}; n>1e-5: {(e > 1e-5).sum()}")
    print(f"   state gpu P,Q,T = {g[:, y, x]}  oracle = {ref['state'][:, y, x]}")
    rel = np.abs(g - ref["state"]) / (np.abs(ref["state"]) + 1e-30)
    for c, nm in enumerate(["P0", "P1", "P2", "Q", "T"]):
        print(f"   {nm}: max rel err {rel[c].max():.2e}  (median {np.median(rel[c]):.2e})")
    return p, img, st, ref


def bwd_diag(sc, cam, idx, name, seed=5):
    p, img, st, ref = fwd_diag(sc, cam, idx, name)
    gimg = synth.dl_dimage(cam, seed)
    grad = torch.zeros((len(idx), 80), dtype=torch.float32, device=DEV)
    ds = torch.zeros(1, dtype=torch.float32, device=DEV)
    p.backward(t(sc.rows), t(np.array([sc.sigma], np.float32)), t(idx), sc.bg, st, t(gimg), grad, ds)
    gg = grad.cpu().numpy()
    gref, dsref, _ = O.backward(sc.rows, sc.sigma, idx, cam, sc.bg, ref["state"], gimg)
    print(f"   dsigma gpu {ds.item():.6g} oracle {dsref:.6g}")
    for nm, sl in FIELDS.items():
        a, b = gg[:, sl], gref[:, sl]
        err = np.abs(a - b)
        bad = err > 1e-4 * np.abs(b) + 1e-6
        rel = err / (np.abs(b) + 1e-12)
        scale = np.abs(b).max()
        print(f"   {nm:3s}: |ref|max {scale:.3e} bad {bad.sum():5d}/{bad.size}  max err {err.max():.3e}  "
              f"worst rel (|ref|>1e-3) {rel[np.abs(b) > 1e-3].max() if (np.abs(b) > 1e-3).any() else 0:.2e}")
        if bad.any():
            r, c = np.nonzero(bad)
            j = np.argmax(err[bad] / (np.abs(b[bad]) + 1e-6))
            print(f"        worst row {r[j]} col {c[j]}: gpu {a[r[j], c[j]]:.6e} ref {b[r[j], c[j]]:.6e}")


if __name__ == "__main__":
    sc = synth.scene_c1()
    bwd_diag(sc, sc.cams[0], np.arange(sc.n, dtype=np.int32), "C1 v0")
    sc2 = synth.scene_c2(n=20000, n_views=3, res=200)
    bwd_diag(sc2, sc2.cams[0], np.arange(sc2.n, dtype=np.int32), "C2s v0")
    # permutation
    p = ViewPipeline(sc.cams[1], sc.n, 1 << 20, device=DEV)
    rows, sig = t(sc.rows), t(np.array([sc.sigma], np.float32))
    a, _ = p.forward(rows, sig, t(np.arange(sc.n, dtype=np.int32)), sc.bg)
    a = a.cpu().numpy().copy()
    b, _ = p.forward(rows, sig, t(np.random.default_rng(1).permutation(sc.n).astype(np.int32)), sc.bg)
    print("perm max diff", np.abs(a - b.cpu().numpy()).max())
    e, _ = p.forward(rows, sig, torch.empty(0, dtype=torch.int32, device=DEV), sc.bg)
    print("empty image unique", np.unique(e.cpu().numpy().reshape(3, -1), axis=1).T)

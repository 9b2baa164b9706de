"""Isolate fp32 error sources of the forward/backward against the fp64 oracle (diagnostic)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_2605_13855_b200 import _lib as L  # noqa: E402
from paper_2605_13855_b200 import synth  # noqa: E402
from paper_2605_13855_b200.pipeline import ViewPipeline  # noqa: E402
from tests.helpers import plain_to_tile_major, tile_major_to_plain  # noqa: E402

DEV = "cuda"
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)  # noqa: E731


def run(sc, cam, idx, tag):
    W, H = cam["width"], cam["height"]
    rows, sig = t(sc.rows), t(np.array([sc.sigma], np.float32))
    p = ViewPipeline(cam, len(idx), 1 << 23, device=DEV)
    img, st = p.forward(rows, sig, t(idx), sc.bg)
    ref = O.render(sc.rows, sc.sigma, idx, cam, sc.bg)
    e0 = np.abs(img.cpu().numpy() - ref["image"])
    k = np.unravel_index(np.argmax(e0), e0.shape)
    y, x = k[1], k[2]
    pv = O.project_value(sc.rows, sc.sigma, idx, cam)
    print(f"[{tag}] E0 (gpu) max {e0.max():.3e} at {k}, n>1e-5 {(e0 > 1e-5).sum()}")
    print(f"    oracle state there {ref['state'][:, y, x]}, gpu {tile_major_to_plain(st.cpu().numpy(), W, H)[:, y, x]}")
    # replace colour and weight with the oracle's fp64 values (rounded to fp32)
    rec = p.rec[:len(idx)]
    r = rec.cpu().numpy()
    vis = (r[:, 12].view(np.uint32) != 0) | (r[:, 13].view(np.uint32) != 0)
    werr = np.abs(r[vis, 11] - pv["w"][vis]) / np.maximum(pv["w"][vis], 1e-12)
    print(f"    w rel err max {werr.max():.2e}; ramp<0.01 count {(pv['w'][vis] < 0.01).sum()}")
    r2 = r.copy()
    r2[vis, 8:11] = pv["color"][vis]
    r2[vis, 11] = pv["w"][vis]
    rec.copy_(t(r2))
    L.oit_composite_fwd(cam, rec, p.pairs, p.offs, sc.bg, p.fwd_ws, image=p.image, state=p.state)
    e1 = np.abs(p.image.cpu().numpy() - ref["image"])
    print(f"    E1 (oracle c,w) max {e1.max():.3e}, n>1e-5 {(e1 > 1e-5).sum()}")
    # backward: GPU state vs oracle state as input, oracle c,w in rec
    g = synth.dl_dimage(cam, 5)
    gref, _, _, bnd = O.backward_bound(sc.rows, sc.sigma, idx, cam, sc.bg, ref["state"], g)
    assert np.all(bnd >= np.abs(gref) * (1 - 1e-9))
    for name, state in [("gpu-state", p.state.clone()),
                        ("oracle-state", t(plain_to_tile_major(ref["state"], W, H).astype(np.float32)))]:
        grad = torch.zeros((len(idx), 80), dtype=torch.float32, device=DEV)
        ds = torch.zeros(1, dtype=torch.float32, device=DEV)
        L.oit_composite_bwd(rows, sig, cam, t(idx), rec, p.pairs, p.offs, sc.bg, state, t(g), grad, ds, p.bwd_ws)
        gg = grad.cpu().numpy()
        bad = np.abs(gg - gref) > 1e-4 * np.abs(gref) + 1e-6
        nrm = np.linalg.norm(gg - gref) / np.linalg.norm(gref)
        print(f"    bwd with {name}: bad {bad.sum()}/{bad.size}, normwise rel {nrm:.2e}")
        for nm, sl in [("mu", slice(0, 3)), ("o", slice(3, 4)), ("q", slice(4, 8)), ("s", slice(8, 11)), ("v", slice(12, 28)), ("h", slice(28, 76))]:
            a, b = gg[:, sl], gref[:, sl]
            err = np.abs(a - b)
            mx = np.abs(b).max()
            rown = np.abs(b).max(1, keepdims=True)
            c1 = (err > 1e-4 * np.abs(b) + 1e-6).sum()
            c2 = (err > 1e-4 * np.abs(b) + 1e-6 * max(1.0, mx)).sum()
            c3 = (err > 1e-4 * np.maximum(np.abs(b), 1e-2 * rown) + 1e-6).sum()
            bb = bnd[:, sl]
            ratio = err / np.maximum(bb, 1e-30)
            q = np.quantile(ratio[bb > 0], [0.5, 0.99, 0.9999, 1.0])
            c4 = (err > 1e-4 * np.abs(b) + 1e-6 + 1e-5 * bb).sum()
            print(f"      {nm:3s} max|ref| {mx:.2e} strict {c1} floor*max {c2} bound1e-5 {c4}  q(err/bound) {q}")


if __name__ == "__main__":
    sc = synth.scene_c2(n=20000, n_views=3, res=200)
    run(sc, sc.cams[0], np.arange(sc.n, dtype=np.int32), "C2s")
    sc = synth.scene_c2(n_views=2)
    act = np.flatnonzero(synth.active_mask(sc, 0.2, "clustered")).astype(np.int32)
    run(sc, sc.cams[1], act, "C2 full rho=0.2")

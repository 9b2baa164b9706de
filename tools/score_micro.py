"""DEV: the C4 score (1M inactive splats scored over a 111k-active state, C3 rig) through
oit_score_subsample for S views in ONE call (CUDA events, one stream); prints ms per scored view.
OIT_DEV_LIB=<path> times another build of the library (A/B).
usage: python tools/score_micro.py [--views 4 8] [--reps 3]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_13855_b200 import _lib as L  # noqa: E402
from paper_2605_13855_b200 import synth  # noqa: E402

if os.environ.get("OIT_DEV_LIB"):
    L.LIB_PATH = os.environ["OIT_DEV_LIB"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", type=int, nargs="+", default=[1, 4, 8])
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    from paper_2605_13855_b200.pipeline import ViewPipeline
    dev = "cuda"
    n_ina, n_act = 1_000_000, 111_000
    sc = synth.scene_c3(n=n_ina + n_act, n_views=300)
    mask = synth.active_mask(sc, n_act / sc.n, "clustered")
    act = torch.from_numpy(np.flatnonzero(mask).astype(np.int32)).to(dev)
    ina = torch.from_numpy(np.flatnonzero(~mask).astype(np.int32)).to(dev)
    rows = torch.from_numpy(sc.rows).to(dev)
    sigma = torch.tensor([sc.sigma], dtype=torch.float32, device=dev)
    V = max(a.views)
    views = list(range(0, 300, 300 // V))[:V]
    big = ViewPipeline(sc.cams[0], n_ina, 1 << 24, device=dev)
    caches, targets = [None] * 300, [None] * 300
    for j in views:
        big.set_camera(sc.cams[j])
        _, st = big.forward(rows, sigma, ina, sc.bg, image=False)
        caches[j] = st.clone()
        targets[j] = torch.randint(0, 256, (3, 1064, 1600), device=dev, dtype=torch.uint8)
    del big
    cap = 1 << 24
    ws = torch.empty(L.oit_score_workspace_bytes(sc.cams[0], n_act, n_ina, cap), dtype=torch.uint8, device=dev)
    sg = torch.zeros((n_ina, 80), dtype=torch.float32, device=dev)
    sds = torch.zeros(1, dtype=torch.float32, device=dev)
    mp = torch.zeros(1, dtype=torch.int64, device=dev)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for S in a.views:
        part = views[:S]
        L.oit_score_subsample(rows, sigma, sc.cams, targets, caches, act, ina, part, "l1", sc.bg, sg, sds, cap, mp, ws,
                              scale=1.0 / S)
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            t0.record()
            L.oit_score_subsample(rows, sigma, sc.cams, targets, caches, act, ina, part, "l1", sc.bg, sg, sds, cap, mp,
                                  ws, scale=1.0 / S)
            t1.record()
            torch.cuda.synchronize()
            ts.append(t0.elapsed_time(t1))
        print(f"S={S}: {np.median(ts):.3f} ms per call, {np.median(ts) / S:.3f} ms per scored view "
              f"(max pairs {int(mp.item())})")


if __name__ == "__main__":
    main()

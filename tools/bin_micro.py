"""DEV: a2 binning alone on the bench workload (C2, 300k splats, 800², ρ = 0.2 clustered): per-view
oit_bin_tiles time (CUDA events, one stream, records precomputed) and the tile-length distribution.
Run under `ncu --metrics gpu__time_duration.sum` for the per-kernel split.
usage: python tools/bin_micro.py [--views 20] [--rho 0.2] [--c3]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_13855_b200 import _lib as L  # noqa: E402
from paper_2605_13855_b200 import synth  # noqa: E402
from paper_2605_13855_b200.pipeline import ViewPipeline  # noqa: E402

if os.environ.get("OIT_DEV_LIB"):  # A/B against another build of the library (dev only)
    L.LIB_PATH = os.environ["OIT_DEV_LIB"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", type=int, default=20)
    ap.add_argument("--rho", type=float, default=0.2)
    ap.add_argument("--c3", action="store_true")
    a = ap.parse_args()
    dev = "cuda"
    sc = synth.scene_c3(n_views=a.views) if a.c3 else synth.scene_c2(n_views=a.views)
    mask = synth.active_mask(sc, a.rho, "clustered")
    act = torch.from_numpy(np.flatnonzero(mask).astype(np.int32)).to(dev)
    rows = torch.from_numpy(sc.rows).to(dev)
    sigma = torch.tensor([sc.sigma], dtype=torch.float32, device=dev)
    n = int(act.numel())
    pipes = []
    for cam in sc.cams:
        p = ViewPipeline(cam, n, 1 << 23, device=dev)
        p.project_bin(rows, sigma, act)
        pipes.append(p)
    torch.cuda.synchronize()
    lens = np.concatenate([np.diff(p.offs.cpu().numpy()) for p in pipes])
    print(f"slots {n}, pairs/view {lens.sum() / len(pipes):.0f}, tiles {len(lens) // len(pipes)}, "
          f"L: nonzero {np.mean(lens > 0):.2f}, mean(nz) {lens[lens > 0].mean():.0f}, p50 {np.percentile(lens, 50):.0f}, "
          f"p90 {np.percentile(lens, 90):.0f}, p99 {np.percentile(lens, 99):.0f}, max {lens.max()}, "
          f">64 {np.mean(lens > 64):.2f}")
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(3):
        t0.record()
        for p in pipes:
            L.oit_bin_tiles(p.cam, p.rec, p.tps, n, p.pairs, p.offs, p.n_pairs, p.bin_ws, None)
        t1.record()
        torch.cuda.synchronize()
        print(f"bin us/view {1e3 * t0.elapsed_time(t1) / len(pipes):.1f}")


if __name__ == "__main__":
    main()

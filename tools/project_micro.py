"""DEV: a1 projection alone (oit_project_cull, CUDA events, one stream) on the bench shapes: C2 training
views (60k active of 300k, ρ = 0.2 clustered), the C2 cache build (240k frozen) and C3 (300k active of
3M); prints µs per call and the algorithmic HBM rate (320 B row + 4 B index + 84 B out per slot)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_13855_b200 import _lib as L  # noqa: E402
from paper_2605_13855_b200 import synth  # noqa: E402

if os.environ.get("OIT_DEV_LIB"):  # A/B against another build of the library (dev only)
    L.LIB_PATH = os.environ["OIT_DEV_LIB"]


def run(name, sc, idx_np, reps=20):
    dev = "cuda"
    rows = torch.from_numpy(sc.rows).to(dev)
    sigma = torch.tensor([sc.sigma], dtype=torch.float32, device=dev)
    idx = torch.from_numpy(idx_np.astype(np.int32)).to(dev)
    n = len(idx_np)
    rec = torch.empty((n, L.OIT_REC), dtype=torch.float32, device=dev)
    tps = torch.empty(n, dtype=torch.int32, device=dev)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for r in range(reps + 3):
        cam = sc.cams[r % len(sc.cams)]
        flush.zero_()
        t0.record()
        L.oit_project_cull(rows, sigma, cam, idx, rec, tps)
        t1.record()
        torch.cuda.synchronize()
        if r >= 3:
            ts.append(t0.elapsed_time(t1))
    ms = float(np.median(ts))
    vis = float((tps > 0).float().mean().item())
    print(f"{name}: {n} slots, visible {vis:.2f}, {1e3 * ms:.1f} us, {n * 408 / (ms * 1e-3) / 1e9:.0f} GB/s algorithmic")


def main():
    sc = synth.scene_c2(n_views=8)
    m = synth.active_mask(sc, 0.2, "clustered")
    run("C2 train (60k)", sc, np.flatnonzero(m))
    run("C2 cache (240k)", sc, np.flatnonzero(~m))
    sc3 = synth.scene_c3(n_views=8)
    m3 = synth.active_mask(sc3, 0.1, "clustered")
    run("C3 train (300k)", sc3, np.flatnonzero(m3))
    run("C3 all (3M)", sc3, np.arange(sc3.n))


if __name__ == "__main__":
    main()

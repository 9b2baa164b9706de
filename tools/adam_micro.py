"""Micro-benchmark of oit_adam_step (NEXT-2): n_total splats, fraction rho active; L2 flushed
(write + read back) before each timed call; prints ms and GB/s of algorithmic bytes."""
import sys

import numpy as np
import torch

from paper_2605_13855_b200 import _lib as L

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300_000
rho = float(sys.argv[2]) if len(sys.argv) > 2 else 0.2
dev = "cuda"
g = np.random.default_rng(0)
act = torch.from_numpy(np.flatnonzero(g.random(n) < rho).astype(np.int32)).to(dev)
na = act.numel()
grad = torch.randn((na, 80), device=dev)
lat = torch.randn((n, 80), device=dev)
m, v, rows = torch.zeros_like(lat), torch.zeros_like(lat), torch.zeros_like(lat)
step = torch.zeros(n, dtype=torch.int32, device=dev)
cfg = L.adam_cfg()
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for k in range(25):
    flush.zero_(); flush.sum()
    torch.cuda.synchronize()
    t0.record()
    L.oit_adam_step(grad, act, lat, m, v, step, rows, cfg)
    t1.record()
    torch.cuda.synchronize()
    if k >= 5:
        ts.append(t0.elapsed_time(t1))
ms = float(np.median(ts))
print(f"n={n} rows={na} ms={ms:.4f} GB/s={na * 2572 / ms / 1e6:.0f}")

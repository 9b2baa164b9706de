"""Micro-benchmark of oit_loss_dssim (NEXT-3) at W×H: L2 flushed before each timed call."""
import sys

import numpy as np
import torch

from paper_2605_13855_b200 import _lib as L

W = int(sys.argv[1]) if len(sys.argv) > 1 else 800
H = int(sys.argv[2]) if len(sys.argv) > 2 else W
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 25
dev = "cuda"
cam = {"width": W, "height": H, "fx": 1.0, "fy": 1.0, "cx": 0.0, "cy": 0.0, "R": np.eye(3).ravel(),
       "t": np.zeros(3), "center": np.zeros(3)}
img, tgt = torch.rand((3, H, W), device=dev), torch.rand((3, H, W), device=dev)
g = torch.empty_like(img)
loss = torch.zeros(1, device=dev)
ws = torch.empty(L.oit_dssim_workspace_bytes(cam), dtype=torch.uint8, device=dev)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts, hot = [], []
for k in range(reps):
    flush.zero_(); flush.sum()
    torch.cuda.synchronize()
    t0.record()
    L.oit_loss_dssim(cam, img, tgt, g, ws, 0.2, loss)
    t1.record()
    torch.cuda.synchronize()
    ts.append(t0.elapsed_time(t1))
    t0.record()
    L.oit_loss_dssim(cam, img, tgt, g, ws, 0.2, loss)
    t1.record()
    torch.cuda.synchronize()
    hot.append(t0.elapsed_time(t1))
print(f"{W}x{H} cold ms={np.median(ts[3:]):.4f} warm-L2 ms={np.median(hot[3:]):.4f}")

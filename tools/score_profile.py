"""DEV: one C4 score view (1M inactive splats scored over a 111k-active state) for ncu launch lists."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_13855_b200 import _lib as L  # noqa: E402
from paper_2605_13855_b200 import synth  # noqa: E402
from paper_2605_13855_b200.pipeline import ViewPipeline  # noqa: E402

dev = "cuda"
n_ina, n_act = 1_000_000, 111_000
sc = synth.scene_c3(n=n_ina + n_act, n_views=300)
mask = synth.active_mask(sc, n_act / sc.n, "clustered")
act = torch.from_numpy(np.flatnonzero(mask).astype(np.int32)).to(dev)
ina = torch.from_numpy(np.flatnonzero(~mask).astype(np.int32)).to(dev)
rows = torch.from_numpy(sc.rows).to(dev)
sigma = torch.tensor([sc.sigma], dtype=torch.float32, device=dev)
cam = sc.cams[7]
big = ViewPipeline(cam, n_ina, 1 << 24, device=dev)
_, st = big.forward(rows, sigma, ina, sc.bg, image=False)
cache = st.clone()
print("inactive pairs", big.pairs_used())
big.forward(rows, sigma, act, sc.bg, image=False)
print("active pairs", big.pairs_used())
del big
tgt = torch.randint(0, 256, (3, cam["height"], cam["width"]), device=dev, dtype=torch.uint8)
cap = 1 << 24
ws = torch.empty(L.oit_score_workspace_bytes(cam, n_act, n_ina, cap), dtype=torch.uint8, device=dev)
sg = torch.zeros((n_ina, 80), dtype=torch.float32, device=dev)
sds = torch.zeros(1, dtype=torch.float32, device=dev)
mp = torch.zeros(1, dtype=torch.int64, device=dev)
for _ in range(3):
    L.oit_score_subsample(rows, sigma, [cam], [tgt], [cache], act, ina, [0], "l1", sc.bg, sg, sds, cap, mp, ws)
torch.cuda.synchronize()
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0.record()
for _ in range(5):
    L.oit_score_subsample(rows, sigma, [cam], [tgt], [cache], act, ina, [0], "l1", sc.bg, sg, sds, cap, mp, ws)
t1.record()
torch.cuda.synchronize()
print("score ms/view", t0.elapsed_time(t1) / 5, "max pairs", int(mp.item()))

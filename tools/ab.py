"""DEV: in-process A/B timing of kernel variants on the bench workload. Variants are selected by an
`oit_dev_set_variant(int)` export that experimental builds add temporarily (the product library has
none: variant 0 only).

Prepares C2 (300k splats, 800², ρ = 0.2 clustered) views over their pre-render caches, then times
the a3 composite (fwd) and a5 moments (bwd) kernels with CUDA events, single stream, alternating
the variants round-robin so clock/thermal drift hits all of them alike.
usage: python tools/ab.py --variants 0 2 [--views 20] [--rounds 5]
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_13855_b200 import _lib as L  # noqa: E402
from paper_2605_13855_b200 import synth  # noqa: E402
from paper_2605_13855_b200.pipeline import ViewPipeline  # noqa: E402
from bench import event_ms  # noqa: E402

if os.environ.get("OIT_DEV_LIB"):  # A/B against another build of the library (dev only)
    L.LIB_PATH = os.environ["OIT_DEV_LIB"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variants", type=int, nargs="+", default=[0])
    ap.add_argument("--views", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--rho", type=float, default=0.2)
    a = ap.parse_args()
    dev = "cuda"
    sc = synth.scene_c2(n_views=a.views)
    mask = synth.active_mask(sc, a.rho, "clustered")
    act = torch.from_numpy(np.flatnonzero(mask).astype(np.int32)).to(dev)
    ina = torch.from_numpy(np.flatnonzero(~mask).astype(np.int32)).to(dev)
    rows = torch.from_numpy(sc.rows).to(dev)
    sigma = torch.tensor([sc.sigma], dtype=torch.float32, device=dev)
    p = ViewPipeline(sc.cams[0], sc.n, 1 << 23, device=dev)
    caches, grads = [], []
    for v, cam in enumerate(sc.cams):
        p.set_camera(cam)
        _, st = p.forward(rows, sigma, ina, sc.bg, image=False)
        caches.append(st.clone())
        grads.append(torch.from_numpy(synth.dl_dimage(cam, v)).to(dev))
    grad = torch.zeros((len(act), 80), dtype=torch.float32, device=dev)
    dsig = torch.zeros(1, dtype=torch.float32, device=dev)
    lib = L.lib()
    set_variant = getattr(lib, "oit_dev_set_variant", None)
    if set_variant is None:
        assert a.variants == [0], "this library has no kernel variants"
        set_variant = lambda v: None  # noqa: E731
    else:
        set_variant.argtypes = [ctypes.c_int]
    res = {v: {"fwd": [], "bwd": []} for v in a.variants}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for e in ev:
        e.record()  # creates the underlying cudaEvent_t
    for r in range(a.rounds):
        for var in a.variants:
            set_variant(var)
            tf = tb = 0.0
            for v, cam in enumerate(sc.cams):
                p.set_camera(cam)
                _, st = p.forward(rows, sigma, act, sc.bg, base=caches[v], image=False, events=(ev[0], ev[1]))
                p.backward(rows, sigma, act, sc.bg, st, grads[v], grad, dsig, events=(ev[2], ev[3]))
                torch.cuda.synchronize()
                tf += event_ms(ev[0], ev[1])
                tb += event_ms(ev[2], ev[3])
            if r > 0:
                res[var]["fwd"].append(tf / len(sc.cams) * 1e3)
                res[var]["bwd"].append(tb / len(sc.cams) * 1e3)
    set_variant(0)
    for var in a.variants:
        f, b = np.array(res[var]["fwd"]), np.array(res[var]["bwd"])
        print(f"variant {var}: fwd {np.median(f):7.2f} us/view (min {f.min():.2f})   "
              f"bwd moments {np.median(b):7.2f} us/view (min {b.min():.2f})")


if __name__ == "__main__":
    main()

"""Buffer management around the C-ABI for one camera shape (PyTorch = device memory + streams).

``ViewPipeline`` owns the per-view scratch of the hot path (records, pair lists, pixel state,
workspaces) and runs a1 → a2 → a3 (forward) and a4 → a5 → a6 (backward) for one view by
calling the ``oit_*`` entry points. It performs no arithmetic of its own.
"""
from __future__ import annotations

import torch

from . import _lib as L


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


class ViewPipeline:
    def __init__(self, cam: dict, max_slots: int, pair_capacity: int, device="cuda"):
        self.cam = cam
        self.device = device
        self.W, self.H = int(cam["width"]), int(cam["height"])
        self.n_tiles = L.num_tiles(cam)
        self.max_slots = int(max_slots)
        self.capacity = int(pair_capacity)
        dev = device
        self.rec = torch.empty((max(self.max_slots, 1), L.OIT_REC), dtype=torch.float32, device=dev)
        self.tps = torch.empty(max(self.max_slots, 1), dtype=torch.int32, device=dev)
        self.pairs = torch.empty(max(self.capacity, 1), dtype=torch.int32, device=dev)
        self.offs = torch.empty(self.n_tiles + 1, dtype=torch.int32, device=dev)
        self.n_pairs = torch.zeros(1, dtype=torch.int64, device=dev)
        self.bin_ws = _ws(L.oit_bin_workspace_bytes(cam, self.capacity, n_slots=self.max_slots), dev)
        self.fwd_ws = _ws(L.oit_fwd_workspace_bytes(cam, self.capacity), dev)
        self.bwd_ws = _ws(L.oit_bwd_workspace_bytes(cam, self.max_slots, self.capacity), dev)
        self.state = torch.empty((5, self.n_tiles, 256), dtype=torch.float32, device=dev)
        self.image = torch.empty((3, self.H, self.W), dtype=torch.float32, device=dev)

    def set_camera(self, cam: dict):
        assert int(cam["width"]) == self.W and int(cam["height"]) == self.H
        self.cam = cam

    def project_bin(self, rows, sigma, idx, stream=None):
        n = int(idx.numel())
        assert n <= self.max_slots
        # (an empty slice may carry a null data pointer; hand the full buffers to the ABI then)
        rec, tps = (self.rec[:n], self.tps[:n]) if n > 0 else (self.rec, self.tps)
        L.oit_project_cull(rows, sigma, self.cam, idx, rec[:n], tps[:n], stream) if n > 0 else None
        L.oit_bin_tiles(self.cam, rec, tps, n, self.pairs, self.offs, self.n_pairs, self.bin_ws, stream)
        return rec

    def forward(self, rows, sigma, idx, bg, base=None, route=None, base_out=None, image=True, stream=None,
                counters=None, events=None, concurrency=1):
        """a1-a3: returns (image or None, state). ``state`` is this pipeline's buffer. ``events``:
        optional (begin, end) torch events recorded around the a3 composite kernel."""
        rec = self.project_bin(rows, sigma, idx, stream)
        if events is not None:
            events[0].record()
        L.oit_composite_fwd(self.cam, rec, self.pairs, self.offs, bg, self.fwd_ws, base=base, route=route,
                            image=self.image if image else None, state=self.state, base_out=base_out,
                            stream=stream, counters=counters, concurrency=concurrency)
        if events is not None:
            events[1].record()
        return (self.image if image else None), self.state

    def new_bwd_ws(self):
        """A backward workspace of this pipeline's shape (e.g. one that keeps a view's coefficients
        for oit_score_subsample after the pipeline has moved on to other views)."""
        return _ws(L.oit_bwd_workspace_bytes(self.cam, self.max_slots, self.capacity), self.device)

    def forward_loss(self, rows, sigma, idx, bg, target, loss="l1", base=None, state=False, stream=None, events=None,
                     concurrency=1, bwd_ws=None, all_tiles=False):
        """a1-a3 + a4 fused (training view): the forward whose epilogue writes the L1/L2 backward
        coefficients into this pipeline's backward workspace (or bwd_ws); follow with backward(...,
        coef_ready=True) on the same workspace. Returns the state buffer if state=True (else None,
        not written). all_tiles: coefficients for every tile (reusable by oit_score_subsample)."""
        rec = self.project_bin(rows, sigma, idx, stream)
        # events (optional): recorded by the library around the composite kernel alone
        L.oit_composite_fwd_loss(self.cam, rec, self.pairs, self.offs, bg, self.fwd_ws,
                                 self.bwd_ws if bwd_ws is None else bwd_ws, self.max_slots, target, loss, base=base,
                                 state=self.state if state else None, stream=stream, concurrency=concurrency,
                                 events=events, all_tiles=all_tiles)
        return self.state if state else None

    def backward(self, rows, sigma, idx, bg, state, dL_dimage, grad, dL_dsigma, dL_dcov=None, scale=1.0,
                 reuse_bins=True, stream=None, events=None, target=None, loss="l1", per_pixel=False, concurrency=1,
                 coef_ready=False, bwd_ws=None):
        """a4-a6 for the splats idx (grad rows += ...). With reuse_bins the records/pairs of the
        preceding forward over the same idx are reused."""
        n = int(idx.numel())
        rec = (self.rec[:n] if n > 0 else self.rec) if reuse_bins else self.project_bin(rows, sigma, idx, stream)
        L.oit_composite_bwd(rows, sigma, self.cam, idx, rec, self.pairs, self.offs, bg, state, dL_dimage, grad,
                            dL_dsigma, self.bwd_ws if bwd_ws is None else bwd_ws, dL_dcov=dL_dcov, scale=scale, stream=stream, events=events,
                            target=target, loss=loss, per_pixel=per_pixel, concurrency=concurrency,
                            coef_ready=coef_ready)

    def pairs_used(self) -> int:
        return int(self.n_pairs.item())

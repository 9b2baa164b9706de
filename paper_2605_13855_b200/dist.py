"""View-sharded data parallelism: one process per GPU, replicated splat
parameters, training views partitioned across ranks, and ONE exchange per step — the sum of the
compacted active-set gradient rows and dσ, held in one contiguous buffer (``GradBuffer``) so it is
one all-reduce (NCCL over NVLink on B200; gloo in the CPU tests).

The refresh (a7/a8, every I iterations) exchanges less than the gradient: each rank scores its own
share of the S subsampled views into the score rows (scale 1/S, so the sum over ranks is the mean
over all S views, R19); a reduce-scatter sums the rows by row range, each rank applies Eq. 8 to
its range only (``oit_score_activeness``: one bit per row), an all-gather of those bits
(n_score/8 bytes) gives every rank the whole membership vector, and every rank applies it and
recompacts (``oit_apply_activeness``) — so the replicas' active sets stay bit-identical and the
Eq. 8 norm work is divided by the world size.

The paper is single-GPU; this module is the north star's multi-GPU extension. It holds no
arithmetic of the method: the sums are collectives over device tensors and the thresholding runs in
liboit's kernels.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib as L

ROW = 80


def views_of_rank(views_per_rank: int, rank: int) -> range:
    """Weak scaling: rank r owns the contiguous block [r·V, (r+1)·V) of the global view list."""
    return range(rank * views_per_rank, (rank + 1) * views_per_rank)


def shard_views(n_views: int, rank: int, world: int) -> range:
    """Strong scaling: a fixed view list split into `world` contiguous blocks (sizes differ ≤ 1)."""
    q, r = divmod(n_views, world)
    start = rank * q + min(rank, r)
    return range(start, start + q + (1 if rank < r else 0))


def _world(group=None) -> int:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group)
    return 1


def _rank(group=None) -> int:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group)
    return 0


def _via_host(t: torch.Tensor, group=None) -> bool:
    # gloo moves CUDA tensors through the host for some collectives only; the CPU tests and the
    # one-GPU multi-rank test hook stage them explicitly (NCCL takes device tensors directly)
    return t.is_cuda and dist.get_backend(group) == "gloo"


class GradBuffer:
    """The per-step exchange buffer: ``rows`` [n_rows][80] (the compacted gradient rows, C-ABI
    layout) and ``dsigma`` [1] are views of ONE contiguous fp32 tensor ``flat`` (dσ at offset
    n_rows·80, padded to 16 B), so a9 is a single all-reduce."""

    def __init__(self, n_rows: int, device="cuda"):
        n = int(n_rows) * ROW
        self.flat = torch.zeros(n + 4, dtype=torch.float32, device=device)
        self.rows = self.flat[:n].view(int(n_rows), ROW)
        self.dsigma = self.flat[n:n + 1]

    def zero_(self):
        self.flat.zero_()
        return self


def all_reduce_(t: torch.Tensor, group=None) -> None:
    """In-place sum over ranks (no-op on one process)."""
    if _world(group) <= 1:
        return
    if _via_host(t, group):
        h = t.cpu()
        dist.all_reduce(h, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, group=group)


def combine_gradients(grad, dsigma: torch.Tensor | None = None, group=None) -> None:
    """a9: in-place sum over ranks of the compacted gradient rows and dσ. ``grad`` is a
    ``GradBuffer`` (one collective) or a rows tensor with ``dsigma`` separately (two)."""
    if isinstance(grad, GradBuffer):
        all_reduce_(grad.flat, group)
        return
    all_reduce_(grad, group)
    if dsigma is not None:
        all_reduce_(dsigma, group)


def combine_scores(score_grad: torch.Tensor, n_views_total: int, n_views_local: int, group=None) -> None:
    """All-reduce form of the refresh combine (kept for callers that need every row on every rank):
    per-rank score rows that are means over the rank's own views become the mean over all
    subsampled views (Σ_r n_r·mean_r / Σ_r n_r)."""
    if _world(group) > 1:
        if n_views_total > 0:
            score_grad.mul_(float(n_views_local) / float(n_views_total))
        all_reduce_(score_grad, group)


def score_rows_per_rank(n_score: int, world: int) -> int:
    """Rows of the score buffer each rank thresholds in the sharded refresh (a multiple of 32, so
    every rank's row bits are whole 32-bit words)."""
    per = -(-int(n_score) // max(world, 1))
    return -(-per // 32) * 32


def score_buffer_rows(n_score: int, world: int) -> int:
    """Rows to allocate for the score buffer of the sharded refresh (padding rows stay zero)."""
    return max(score_rows_per_rank(n_score, world) * max(world, 1), 32)


def sharded_refresh_update(score_rows: torch.Tensor, score_idx: torch.Tensor, eps, mode: str, n_total: int,
                           active_bits: torch.Tensor, active_idx: torch.Tensor, n_active: torch.Tensor, ws: torch.Tensor,
                           newly_frozen=None, n_frozen=None, newly_active=None, n_activated=None, group=None,
                           stream=None) -> None:
    """The refresh exchange + a8. ``score_rows`` [score_buffer_rows(n, world)][80]:
    this rank's contribution to the score rows of the n = score_idx.numel() scored splats (rows
    beyond n are zero padding), already scaled so that the sum over ranks is the mean over all
    subsampled views. Reduce-scatter by row range → Eq. 8 on this rank's range → all-gather of the
    row bits → membership update and recompaction on every rank (identical on all ranks)."""
    world, rank = _world(group), _rank(group)
    n = int(score_idx.numel())
    chunk = score_rows_per_rank(n, world)
    assert score_rows.shape[0] >= chunk * world and score_rows.shape[1] == ROW
    dev = score_rows.device
    if world > 1:
        mine = torch.empty((chunk, ROW), dtype=torch.float32, device=dev)
        src = score_rows[:chunk * world]
        if _via_host(src, group):
            h = torch.empty((chunk, ROW), dtype=torch.float32)
            dist.reduce_scatter_tensor(h, src.cpu().contiguous(), group=group)
            mine.copy_(h)
        else:
            dist.reduce_scatter_tensor(mine, src.contiguous(), group=group)
    else:
        mine = score_rows[:chunk]
    valid = max(0, min(chunk, n - rank * chunk))
    bits_mine = torch.zeros(chunk // 32, dtype=torch.int32, device=dev)
    L.oit_score_activeness(mine, valid, eps, bits_mine, stream=stream)
    if world > 1:
        bits_all = torch.empty(chunk // 32 * world, dtype=torch.int32, device=dev)
        if _via_host(bits_mine, group):
            h = torch.empty(chunk // 32 * world, dtype=torch.int32)
            dist.all_gather_into_tensor(h, bits_mine.cpu(), group=group)
            bits_all.copy_(h)
        else:
            dist.all_gather_into_tensor(bits_all, bits_mine, group=group)
    else:
        bits_all = bits_mine
    L.oit_apply_activeness(bits_all, score_idx, mode, n_total, active_bits, active_idx, n_active,
                           newly_frozen=newly_frozen, n_frozen=n_frozen, newly_active=newly_active,
                           n_activated=n_activated, ws=ws, stream=stream)

"""View-sharded data parallelism: one process per GPU, replicated splat
parameters, training views partitioned across ranks, and ONE exchange per step — the sum of the
compacted active-set gradient rows (+ dσ) with an all-reduce (NCCL over NVLink on B200; gloo in
the CPU tests). The refresh (a7/a8) combines the per-rank score rows the same way, so every rank
applies the identical Eq. 8 update and the replicas' active sets stay bit-identical.

The paper is single-GPU; this module is the north star's multi-GPU extension. It holds no
arithmetic of the method (the sums are plain collectives over device tensors).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def views_of_rank(views_per_rank: int, rank: int) -> range:
    """Weak scaling: rank r owns the contiguous block [r·V, (r+1)·V) of the global view list."""
    return range(rank * views_per_rank, (rank + 1) * views_per_rank)


def shard_views(n_views: int, rank: int, world: int) -> range:
    """Strong scaling: a fixed view list split into `world` contiguous blocks (sizes differ ≤ 1)."""
    q, r = divmod(n_views, world)
    start = rank * q + min(rank, r)
    return range(start, start + q + (1 if rank < r else 0))


def combine_gradients(grad: torch.Tensor, dsigma: torch.Tensor, group=None) -> None:
    """a9: in-place sum over ranks of the compacted gradient rows [n_A][80] and dσ [1]."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(grad, group=group)
        dist.all_reduce(dsigma, group=group)


def combine_scores(score_grad: torch.Tensor, n_views_total: int, n_views_local: int, group=None) -> None:
    """Refresh: the per-rank score rows are means over the rank's subsampled views; turn them into
    the mean over all subsampled views (Σ_r n_r·mean_r / Σ_r n_r) with one all-reduce."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        if n_views_total > 0:
            score_grad.mul_(float(n_views_local) / float(n_views_total))
        dist.all_reduce(score_grad, group=group)

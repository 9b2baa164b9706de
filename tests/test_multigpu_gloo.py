"""N > 1 host logic on CPU (world_size 2, gloo): view sharding + the gradient / score all-reduce
of paper_2605_13855_b200.dist, with the oracle standing in for the per-view compute. The result
must equal the single-process sum over all views, and every rank must derive the identical
active-set bitmask from the combined score."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2605_13855_b200 import dist as D
from paper_2605_13855_b200 import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    return synth.scene_c1(n=300, n_views=4, res=32)


def _view_grad(sc, v, idx):
    cam = sc.cams[v]
    st = O.render(sc.rows, sc.sigma, idx, cam, sc.bg)["state"]
    g = synth.dl_dimage(cam, 100 + v).astype(np.float64)
    gr, ds, _ = O.backward(sc.rows, sc.sigma, idx, cam, sc.bg, st, g)
    return gr, ds


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc = _scene()
        idx = np.arange(sc.n)
        views = list(D.views_of_rank(2, rank))
        grad = torch.zeros((sc.n, 80), dtype=torch.float64)
        dsig = torch.zeros(1, dtype=torch.float64)
        for v in views:
            gr, ds = _view_grad(sc, v, idx)
            grad += torch.from_numpy(gr)
            dsig += ds
        # refresh: each rank scores its own views (local mean), combined into the global mean
        score = grad.clone() / len(views)
        D.combine_gradients(grad, dsig)
        D.combine_scores(score, n_views_total=2 * world, n_views_local=len(views))
        bits0 = synth.bits_from_mask(np.ones(sc.n, bool))
        eps = np.full(6, 1e-3, np.float32)
        bits, act, _, _ = O.update_active(score.numpy().astype(np.float32), idx, eps, "fresh", sc.n, bits0)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), grad=grad.numpy(), dsig=dsig.numpy(), score=score.numpy(),
                 bits=bits)
    finally:
        dist.destroy_process_group()


def test_shard_views_partition():
    for n, w in [(100, 1), (100, 2), (100, 8), (7, 3), (3, 4)]:
        parts = [list(D.shard_views(n, r, w)) for r in range(w)]
        assert sum(parts, []) == list(range(n))
        assert max(map(len, parts)) - min(map(len, parts)) <= 1
    assert list(D.views_of_rank(100, 2)) == list(range(200, 300))


@pytest.mark.timeout(300)
def test_two_rank_gradient_and_score_allreduce(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    r = [np.load(tmp_path / f"rank{k}.npz") for k in range(world)]
    sc = _scene()
    idx = np.arange(sc.n)
    ref = np.zeros((sc.n, 80))
    ref_ds = 0.0
    for v in range(4):
        gr, ds = _view_grad(sc, v, idx)
        ref += gr
        ref_ds += ds
    for k in range(world):
        assert np.allclose(r[k]["grad"], ref, rtol=1e-12, atol=1e-14)
        assert abs(r[k]["dsig"][0] - ref_ds) <= 1e-12 * max(1.0, abs(ref_ds))
        assert np.allclose(r[k]["score"], ref / 4, rtol=1e-12, atol=1e-14)
    assert np.array_equal(r[0]["bits"], r[1]["bits"])
    assert np.abs(ref).max() > 0

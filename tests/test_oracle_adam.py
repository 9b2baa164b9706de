"""Pins of the oracle's masked Adam + activations (NEXT-2, Alg. 1 l.6 P:162) against
torch.optim.Adam in fp64 with autograd through the activations (a library routine the oracle does
not call), and closed forms of Adam's bias-corrected first step and of a constant gradient."""
import numpy as np
import pytest
import torch

import oracle as O

ROW = 80
GROUPS = {"mu": [0, 1, 2], "o": [3], "q": [4, 5, 6, 7], "s": [8, 9, 10], "v": list(range(12, 28)),
          "h_dc": [28, 29, 30], "h_rest": list(range(31, 76))}


def _latent(n, g):
    lat = g.normal(size=(n, ROW)) * 0.5
    lat[:, [11, 76, 77, 78, 79]] = 0.0
    return lat


def _act(lat):
    out = lat.clone()
    out[:, 3] = torch.sigmoid(lat[:, 3])
    out[:, 8:11] = torch.exp(lat[:, 8:11])
    return out


def test_adam_matches_torch_adam_through_activations():
    g = np.random.default_rng(3)
    n = 7
    lat0 = _latent(n, g)
    lr = {k: float(x) for k, x in zip(O.ADAM_LR_KEYS, [1e-3, 0.05, 2e-3, 0.01, 0.02, 3e-3, 1e-4, 0.1])}
    params = {k: torch.tensor(lat0[:, c], dtype=torch.float64, requires_grad=True) for k, c in GROUPS.items()}
    lsig = torch.tensor([np.log(0.7)], dtype=torch.float64, requires_grad=True)
    opt = torch.optim.Adam([{"params": [params[k]], "lr": lr[k]} for k in GROUPS] + [{"params": [lsig], "lr": lr["sigma"]}],
                           betas=(0.9, 0.999), eps=1e-15)
    lat, m, v = lat0.copy(), np.zeros((n, ROW)), np.zeros((n, ROW))
    step = np.zeros(n, np.int32)
    ss = np.array([np.log(0.7), 0.0, 0.0, 0.0])
    idx = np.arange(n, dtype=np.int32)
    for it in range(4):
        gphys = g.normal(size=(n, ROW)) * 10.0 ** g.integers(-4, 1, size=(n, 1))
        gphys[:, [11, 76, 77, 78, 79]] = 0.0
        gsig = float(g.normal())
        # torch: latent → physical, loss = <gphys, physical> + gsig·σ  ⇒ autograd = the chain rule
        full = torch.zeros((n, ROW), dtype=torch.float64)
        for k, c in GROUPS.items():
            full[:, c] = params[k]
        loss = (_act(full) * torch.from_numpy(gphys)).sum() + gsig * torch.exp(lsig).sum()
        opt.zero_grad()
        loss.backward()
        opt.step()
        lat, m, v, step, rows, ss, sig = O.adam_step(gphys, idx, lat, m, v, step, gsig, ss, lr)
        for k, c in GROUPS.items():
            assert np.allclose(lat[:, c], params[k].detach().numpy(), rtol=1e-13, atol=1e-15), (it, k)
            assert np.allclose(m[:, c], opt.state[params[k]]["exp_avg"].numpy(), rtol=1e-12, atol=1e-300)
            assert np.allclose(v[:, c], opt.state[params[k]]["exp_avg_sq"].numpy(), rtol=1e-12, atol=1e-300)
        with torch.no_grad():
            full = torch.zeros((n, ROW), dtype=torch.float64)
            for k, c in GROUPS.items():
                full[:, c] = params[k]
            assert np.allclose(rows, _act(full).numpy(), rtol=1e-13, atol=1e-15)
        assert abs(ss[0] - lsig.item()) < 1e-13 and abs(sig - np.exp(lsig.item())) < 1e-13
        assert np.all(step == it + 1) and ss[3] == it + 1


def test_adam_first_step_is_lr_sign_and_frozen_rows_untouched():
    """t = 1: m̂ = g, v̂ = g² ⇒ Δℓ = −lr·g/(|g|+ε) (closed form); rows outside the active list keep
    latent, moments and step bit-for-bit; a splat first activated later starts at t = 1."""
    g = np.random.default_rng(5)
    n = 6
    lat0 = _latent(n, g)
    lr = dict(O.ADAM_LR_3DGS)
    gr = g.normal(size=(n, ROW))
    gr[:, [11, 76, 77, 78, 79]] = 0.0
    act1 = np.array([0, 2, 5], np.int32)
    lat, m, v, step, rows, _, _ = O.adam_step(gr[act1], act1, lat0, np.zeros((n, ROW)), np.zeros((n, ROW)),
                                              np.zeros(n, np.int32))
    fro = np.setdiff1d(np.arange(n), act1)
    assert np.array_equal(lat[fro], lat0[fro]) and not m[fro].any() and not v[fro].any() and not step[fro].any()
    lrf = np.zeros(ROW)
    for k, c in GROUPS.items():
        lrf[c] = lr[k]
    gl = gr[act1].copy()
    o = 1 / (1 + np.exp(-lat0[act1, 3]))
    gl[:, 3] *= o * (1 - o)
    gl[:, 8:11] *= np.exp(lat0[act1, 8:11])
    assert np.allclose(lat[act1], lat0[act1] - lrf * gl / (np.abs(gl) + 1e-15), rtol=1e-14, atol=1e-17)
    # splat 1 joins at the second call: its own t = 1 (same closed form), splat 0 is at t = 2
    act2 = np.array([0, 1], np.int32)
    lat2, _, _, step2, _, _, _ = O.adam_step(gr[act2], act2, lat, m, v, step)
    assert list(step2) == [2, 1, 1, 0, 0, 1]
    g1 = gr[1].copy()
    o1 = 1 / (1 + np.exp(-lat0[1, 3]))
    g1[3] *= o1 * (1 - o1)
    g1[8:11] *= np.exp(lat0[1, 8:11])
    assert np.allclose(lat2[1], lat0[1] - lrf * g1 / (np.abs(g1) + 1e-15), rtol=1e-14, atol=1e-17)


def test_adam_constant_gradient_steps_lr_sign_every_step():
    """Constant g: m_t = (1−β1^t)g and v_t = (1−β2^t)g² exactly, so every step moves the latent by
    lr·g/(|g|+ε) (Adam's bias correction; the μ field has the identity activation)."""
    n = 1
    lat = np.zeros((n, ROW))
    m = np.zeros((n, ROW))
    v = np.zeros((n, ROW))
    step = np.zeros(n, np.int32)
    gr = np.zeros((n, ROW))
    gr[0, 0], gr[0, 1] = 0.3, -2e-3
    lr = dict(O.ADAM_LR_3DGS)
    for t in range(1, 51):
        lat, m, v, step, rows, _, _ = O.adam_step(gr, [0], lat, m, v, step, lr=lr)
        assert lat[0, 0] == pytest.approx(-t * lr["mu"], rel=1e-12)
        assert lat[0, 1] == pytest.approx(t * lr["mu"], rel=1e-12)
        assert lat[0, 2] == 0.0
        assert rows[0, 3] == 0.5 and rows[0, 8] == 1.0

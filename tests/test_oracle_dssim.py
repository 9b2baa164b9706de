"""Pins of the oracle's 3DGS loss (1−λ)L1 + λ(1−SSIM) and its gradient (NEXT-3)
against an independent evaluation (torch conv2d with the Gaussian window, fp64 autograd), closed
forms (identical images; constant images at interior pixels) and central differences."""
import numpy as np
import torch
import torch.nn.functional as F

import oracle as O


def _torch_loss(x, y, lam):
    g = torch.exp(-((torch.arange(11, dtype=torch.float64) - 5) ** 2) / (2 * 1.5 ** 2))
    g = g / g.sum()
    w = (g[:, None] * g[None, :]).expand(3, 1, 11, 11).contiguous()
    c = lambda t: F.conv2d(t[None], w, padding=5, groups=3)[0]  # noqa: E731
    mx, my = c(x), c(y)
    sx, sy, sxy = c(x * x) - mx * mx, c(y * y) - my * my, c(x * y) - mx * my
    C1, C2 = 0.01 ** 2, 0.03 ** 2
    s = ((2 * mx * my + C1) * (2 * sxy + C2)) / ((mx * mx + my * my + C1) * (sx + sy + C2))
    return (1 - lam) * (x - y).abs().mean() + lam * (1 - s.mean()), s


def test_dssim_matches_torch_conv_autograd():
    g = np.random.default_rng(11)
    for H, W, lam in [(24, 31, 0.2), (7, 5, 0.5), (40, 16, 1.0)]:
        x = g.random((3, H, W))
        y = np.clip(x + g.normal(size=x.shape) * 0.2, 0, 1)
        L, gr, smap = O.loss_dssim(x, y, lam, with_map=True)
        xt = torch.tensor(x, requires_grad=True)
        Lt, st = _torch_loss(xt, torch.tensor(y), lam)
        Lt.backward()
        assert abs(L - Lt.item()) < 1e-13
        assert np.allclose(smap, st.detach().numpy(), rtol=0, atol=1e-13)
        assert np.allclose(gr, xt.grad.numpy(), rtol=1e-10, atol=1e-16)


def test_dssim_identical_images_zero_loss_and_gradient():
    x = np.random.default_rng(2).random((3, 20, 18))
    L, gr = O.loss_dssim(x, x.copy(), 0.2)
    assert abs(L) < 1e-14 and np.abs(gr).max() < 1e-15


def test_dssim_constant_images_closed_form():
    """x ≡ a, y ≡ b: at pixels ≥ 5 from the border the window is complete, σ = 0, and
    S = (2ab + C1)/(a² + b² + C1)."""
    a, b = 0.7, 0.2
    H = W = 16
    _, _, smap = O.loss_dssim(np.full((3, H, W), a), np.full((3, H, W), b), 0.2, with_map=True)
    C1 = 1e-4
    assert np.allclose(smap[:, 5:-5, 5:-5], (2 * a * b + C1) / (a * a + b * b + C1), rtol=1e-13)
    assert np.all(np.abs(smap[:, 0, 0] - (2 * a * b + C1) / (a * a + b * b + C1)) > 1e-3)   # border differs


def test_dssim_gradient_central_differences():
    g = np.random.default_rng(4)
    x = g.random((3, 9, 8))
    y = g.random((3, 9, 8))
    L, gr = O.loss_dssim(x, y, 0.2)
    h = 1e-6
    for _ in range(25):
        k = tuple(int(g.integers(0, s)) for s in x.shape)
        xp, xm = x.copy(), x.copy()
        xp[k] += h
        xm[k] -= h
        fd = (O.loss_dssim(xp, y, 0.2)[0] - O.loss_dssim(xm, y, 0.2)[0]) / (2 * h)
        assert abs(fd - gr[k]) <= 1e-7 * max(1.0, abs(gr[k]) * 1e3), (k, fd, gr[k])

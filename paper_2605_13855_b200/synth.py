"""Seeded synthetic inputs shaped like the paper's workloads.

This module is the ONLY code shared by the oracle tests and the CUDA path. It draws random
numbers (numpy Philox bit generator, fixed seeds) and builds look-at cameras; it contains none
of the method's arithmetic (no projection, no compositing, no gradients).

Parameter rows follow DESIGN.md §2: ``[N][80]`` fp32 — 0-2 μ, 3 o, 4-7 q (raw, w,x,y,z),
8-10 s, 12-27 v (weight SH), 28-75 h (16×3 coefficient-major).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

ROW = 80
MU, O, Q, S, V, H = 0, 3, 4, 8, 12, 28


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(int(seed)))


def look_at(center, target=(0.0, 0.0, 0.0), up=(0.0, 0.0, 1.0), *, width, height, f, cx, cy,
            znear=0.2) -> dict:
    """OpenCV-style camera (x right, y down, z forward) at ``center`` looking at ``target``."""
    c = np.asarray(center, np.float64)
    fwd = np.asarray(target, np.float64) - c
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, np.float64))
    if np.linalg.norm(right) < 1e-9:
        right = np.cross(fwd, np.array([0.0, 1.0, 0.0]))
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    R = np.stack([right, down, fwd])
    t = -R @ c
    return dict(width=int(width), height=int(height), fx=float(f), fy=float(f), cx=float(cx),
                cy=float(cy), R=R.astype(np.float32).reshape(9), t=t.astype(np.float32),
                center=c.astype(np.float32), znear=float(znear))


def ring_cameras(n, radius, elevation_deg, *, width, height, f, cx, cy, azimuth0=0.0,
                 height_jitter=0.0, z=None, seed=0) -> list:
    g = rng(seed + 7001)
    cams = []
    el = math.radians(elevation_deg)
    for k in range(n):
        az = azimuth0 + 2 * math.pi * k / n
        zz = radius * math.sin(el) if z is None else z + (g.uniform(-height_jitter, height_jitter) if height_jitter else 0.0)
        rr = radius * math.cos(el) if z is None else radius
        cams.append(look_at((rr * math.cos(az), rr * math.sin(az), zz), width=width, height=height,
                            f=f, cx=cx, cy=cy))
    return cams


def fibonacci_hemisphere_cameras(n, radius, *, width, height, f, cx, cy) -> list:
    cams = []
    golden = math.pi * (3.0 - math.sqrt(5.0))
    for k in range(n):
        zc = 0.05 + 0.9 * (k + 0.5) / n          # upper hemisphere, avoid the exact pole/horizon
        r = math.sqrt(1.0 - zc * zc)
        az = golden * k
        cams.append(look_at((radius * r * math.cos(az), radius * r * math.sin(az), radius * zc),
                            width=width, height=height, f=f, cx=cx, cy=cy))
    return cams


def _appearance(g: np.random.Generator, n: int, rows: np.ndarray) -> None:
    """q ~ 4-normal (raw, unnormalised), o ~ U[0.1,1.0], h DC ~ U[-1.2,1.2], h rest clipped
    N(0,0.01); v DC ~ U[3,6], v rest clipped N(0,0.02) to ±0.03 (v(r) ≥ 0.3, R4)."""
    rows[:, Q:Q + 4] = g.standard_normal((n, 4)).astype(np.float32)
    rows[:, O] = g.uniform(0.1, 1.0, n).astype(np.float32)
    h = np.clip(g.normal(0.0, 0.01, (n, 16, 3)), -0.01, 0.01)
    h[:, 0, :] = g.uniform(-1.2, 1.2, (n, 3))
    rows[:, H:H + 48] = h.reshape(n, 48).astype(np.float32)
    v = np.clip(g.normal(0.0, 0.02, (n, 16)), -0.03, 0.03)
    v[:, 0] = g.uniform(3.0, 6.0, n)
    rows[:, V:V + 16] = v.astype(np.float32)


@dataclass
class Scene:
    name: str
    rows: np.ndarray            # [N][80] fp32
    sigma: float
    cams: list
    bg: np.ndarray              # [3]
    meta: dict = field(default_factory=dict)

    def __post_init__(self):
        # σ lives in an fp32 device scalar: keep the host copy fp32-representable so the oracle
        # and the GPU see the same value (the ramp 1 - d/σ amplifies any difference near d ≈ σ)
        self.sigma = float(np.float32(self.sigma))

    @property
    def n(self) -> int:
        return int(self.rows.shape[0])


def scene_c1(seed: int = 1, n: int = 1000, n_views: int = 4, res: int = 64) -> Scene:
    """C1 tiny: μ ~ U[-1,1]³, log s ~ N(ln 0.05, 0.4); 4 views 64×64 on a ring r=4, elev 20°,
    f=80 (scaled with res), c0=(0.1,0.2,0.3); σ = 4.75 (≈10% of (splat, view) pairs have d ≥ σ)."""
    g = rng(seed)
    rows = np.zeros((n, ROW), np.float32)
    rows[:, MU:MU + 3] = g.uniform(-1.0, 1.0, (n, 3)).astype(np.float32)
    rows[:, S:S + 3] = np.exp(g.normal(math.log(0.05), 0.4, (n, 3))).astype(np.float32)
    _appearance(g, n, rows)
    f = 80.0 * res / 64.0
    cams = ring_cameras(n_views, 4.0, 20.0, width=res, height=res, f=f, cx=res / 2, cy=res / 2, seed=seed)
    return Scene("C1", rows, 4.75, cams, np.array([0.1, 0.2, 0.3]), dict(seed=seed))


def scene_c2(seed: int = 2, n: int = 300_000, n_views: int = 100, res: int = 800) -> Scene:
    """C2 NeRF-synthetic-shaped: N on a unit sphere shell (5% radial noise), log s ~ N(ln 0.01, 0.5);
    views on a Fibonacci upper hemisphere r=4, res×res, f=1111.1·res/800; white background; σ = 4.8."""
    g = rng(seed)
    rows = np.zeros((n, ROW), np.float32)
    d = g.standard_normal((n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    rad = 1.0 + 0.05 * g.standard_normal(n)
    rows[:, MU:MU + 3] = (d * rad[:, None]).astype(np.float32)
    rows[:, S:S + 3] = np.exp(g.normal(math.log(0.01), 0.5, (n, 3))).astype(np.float32)
    _appearance(g, n, rows)
    f = 1111.1 * res / 800.0
    cams = fibonacci_hemisphere_cameras(n_views, 4.0, width=res, height=res, f=f, cx=res / 2, cy=res / 2)
    return Scene("C2", rows, 4.8, cams, np.array([1.0, 1.0, 1.0]), dict(seed=seed))


def scene_c3(seed: int = 3, n: int = 3_000_000, n_views: int = 200, width: int = 1600, height: int = 1064) -> Scene:
    """C3 Mip-NeRF360-shaped: 60% ~U([-2,2]²×[-0.8,0.8]), 40% on an upper-hemisphere shell with
    radius log-U[8,40]; log s ~ N(ln 0.01, 0.6)·max(1, r/4); views on a ring r=3.5, height
    0.6±0.1 looking at the origin; f=1150 (scaled), c=(W/2,H/2); black background; σ = 25."""
    g = rng(seed)
    rows = np.zeros((n, ROW), np.float32)
    n_in = int(round(0.6 * n))
    mu = np.empty((n, 3))
    mu[:n_in, 0:2] = g.uniform(-2.0, 2.0, (n_in, 2))
    mu[:n_in, 2] = g.uniform(-0.8, 0.8, n_in)
    d = g.standard_normal((n - n_in, 3))
    d[:, 2] = np.abs(d[:, 2])
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    r = np.exp(g.uniform(math.log(8.0), math.log(40.0), n - n_in))
    mu[n_in:] = d * r[:, None]
    rows[:, MU:MU + 3] = mu.astype(np.float32)
    rad = np.linalg.norm(mu, axis=1)
    logs = g.normal(math.log(0.01), 0.6, (n, 3))
    rows[:, S:S + 3] = (np.exp(logs) * np.maximum(1.0, rad / 4.0)[:, None]).astype(np.float32)
    _appearance(g, n, rows)
    f = 1150.0 * width / 1600.0
    cams = ring_cameras(n_views, 3.5, 0.0, width=width, height=height, f=f, cx=width / 2, cy=height / 2,
                        z=0.6, height_jitter=0.1, seed=seed)
    return Scene("C3", rows, 25.0, cams, np.array([0.0, 0.0, 0.0]), dict(seed=seed))


def scene_degenerate(seed: int = 5) -> Scene:
    """C1 (300 splats, 4 views 64×64) plus hand-set edge-case splats: zero quaternion, opacity at
    and just above 1/255, opacity 1 and 0.995 (the 0.99 clamp at the centre), a splat at the look-at
    point (centre on the principal point), one huge splat covering every view, needle-thin and
    flat splats, a splat behind/at the near plane of every view, far off-screen splats whose extent
    reaches the border, exact duplicates, a colour channel clamped at 0 (h DC very negative), a
    weight SH that is negative in some directions (the v⁺ guard, R4) and splats beyond σ (w = 0)."""
    base = scene_c1(seed=seed, n=300, n_views=4)
    rows = [r for r in base.rows]

    def splat(mu, s=(0.05, 0.05, 0.05), o=0.7, q=(1.0, 0.0, 0.0, 0.0), dc=(0.3, 0.2, -0.1), vdc=4.0, vrest=None):
        r = np.zeros(ROW, np.float32)
        r[MU:MU + 3] = mu
        r[O] = o
        r[Q:Q + 4] = q
        r[S:S + 3] = s
        r[H:H + 3] = dc
        r[V] = vdc
        if vrest is not None:
            r[V + 1:V + 4] = vrest
        rows.append(r)

    splat((0.1, 0.1, 0.1), q=(0.0, 0.0, 0.0, 0.0))                  # zero quaternion → culled
    splat((0.2, -0.1, 0.0), o=np.float32(1.0 / 255.0))              # 255·o ≤ 1 → culled
    splat((0.2, -0.2, 0.1), o=np.nextafter(np.float32(1.0 / 255.0), np.float32(1)) * np.float32(1.001))
    splat((-0.3, 0.2, 0.0), o=1.0)                                  # α clamped to 0.99 near the centre
    splat((0.3, 0.3, -0.2), o=0.995)
    splat((0.0, 0.0, 0.0), s=(0.08, 0.08, 0.08))                    # on the look-at point: centre on (cx, cy)
    splat((0.0, 0.0, 0.0), s=(3.0, 3.0, 3.0), o=0.05)               # covers every view (huge extent)
    splat((0.4, 0.0, 0.2), s=(1e-4, 0.3, 0.3))                      # flat disc
    splat((-0.4, 0.1, 0.2), s=(1e-4, 1e-4, 0.4), q=(0.7, 0.1, 0.7, 0.1))   # needle
    for c in base.cams:                                             # at / behind every camera centre
        ctr = np.asarray(c["center"], np.float64)
        splat(tuple(ctr * 1.0001))
        splat(tuple(ctr * 1.3))
    splat((6.0, 0.0, 0.3), s=(0.6, 0.6, 0.6))                       # off-screen centre, extent on screen
    splat((0.0, -6.0, 0.3), s=(0.6, 0.6, 0.6))
    for _ in range(2):
        splat((0.15, 0.25, -0.05), o=0.6, dc=(0.1, 0.4, 0.2))       # exact duplicates
    splat((-0.1, -0.3, 0.1), dc=(-3.0, 0.5, 0.5))                   # red channel clamped at 0
    splat((0.25, -0.25, -0.1), vdc=0.3, vrest=(2.0, 2.0, 2.0))      # v(r) < 0 for some directions
    for c in base.cams:                                             # on the view axis beyond σ: w = 0, still in T
        splat(tuple(-0.35 * np.asarray(c["center"], np.float64)), s=(0.15, 0.15, 0.15))
    return Scene("degenerate", np.stack(rows).astype(np.float32), base.sigma, base.cams, base.bg, dict(seed=seed))


BRANCH_KINDS = ("fov", "color", "vneg", "ramp")


def scene_branch(kind: str, seed: int = 0, n: int = 10) -> Scene:
    """Tiny scenes whose splats sit on the piecewise branches of the value path, for the
    finite-difference pins and the GPU parity of those branches. One 16×16 camera at the origin
    with the identity rotation (camera space = world space, f = 12, c = (8, 8)), so every position
    below is directly camera-space; μ_z ~ U[2.5, 4].

    * ``fov``: 6 of the n splats at |t_x/t_z| (or |t_y/t_z|) ∈ [1.08, 1.5]·1.3·tan(fov/2) — the J
      clamp of R13 active — with s ~ U[0.6, 1.0] so the α = 1/255 ellipse still reaches the image;
    * ``color``: 6 splats with one or two colour channels' DC ~ U[-3.5, -2.2] (SH + 0.5 < 0: R7 clamp);
    * ``vneg``: 5 splats with v DC ~ U[-6, -3] (v(r) < 0: w = 0 through R4, still in T per R11);
    * ``ramp``: σ fixed at 3.2; 3 splats at d ∈ σ·[1.01, 1.3] (d ≥ σ: w = 0), 4 at d ∈ σ·[0.98, 0.999]
      (within 2% below σ), the rest nearer.
    The other splats are ordinary (in-frustum, positive colour and weight)."""
    assert kind in BRANCH_KINDS
    g = rng(7700 + 97 * BRANCH_KINDS.index(kind) + seed)
    width = height = 16
    f = 12.0
    cam = dict(width=width, height=height, fx=f, fy=f, cx=8.0, cy=8.0, R=np.eye(3, dtype=np.float32).reshape(9),
               t=np.zeros(3, np.float32), center=np.zeros(3, np.float32), znear=0.2)
    rows = np.zeros((n, ROW), np.float32)
    z = g.uniform(2.5, 4.0, n)
    u = g.uniform(-0.45, 0.45, (n, 2))                 # in-frustum t_x/t_z, t_y/t_z
    s = np.exp(g.normal(math.log(0.25), 0.3, (n, 3)))
    _appearance(g, n, rows)
    rows[:, O] = g.uniform(0.3, 0.95, n).astype(np.float32)
    sigma = 4.75
    if kind == "fov":
        lim = 1.3 * (0.5 * width / f)
        for k in range(6):
            ax = k % 2                                  # x for even k, y for odd k
            sign = 1.0 if (k // 2) % 2 == 0 else -1.0
            u[k, ax] = sign * lim * g.uniform(1.08, 1.5)
            s[k] = g.uniform(0.6, 1.0, 3)
    elif kind == "color":
        for k in range(6):
            chans = [k % 3] if k < 3 else [k % 3, (k + 1) % 3]
            for ch in chans:
                rows[k, H + ch] = g.uniform(-3.5, -2.2)
    elif kind == "vneg":
        rows[:5, V] = g.uniform(-6.0, -3.0, 5)
    else:  # ramp
        sigma = 3.2
        z[:3] = sigma * g.uniform(1.01, 1.3, 3)
        z[3:7] = sigma * g.uniform(0.98, 0.999, 4)
        z[7:] = sigma * g.uniform(0.7, 0.9, n - 7)
    rows[:, MU] = (u[:, 0] * z).astype(np.float32)
    rows[:, MU + 1] = (u[:, 1] * z).astype(np.float32)
    rows[:, MU + 2] = z.astype(np.float32)
    rows[:, S:S + 3] = s.astype(np.float32)
    return Scene(f"branch-{kind}", rows, sigma, [cam], np.array([0.1, 0.2, 0.3]), dict(seed=seed, kind=kind))


def active_mask(scene: Scene, rho: float, kind: str = "clustered", seed: int = 11) -> np.ndarray:
    """Forced active set of fraction ρ: 'uniform' (Bernoulli(ρ)) or 'clustered' (μ_x in the top ρ
    quantile — the paper's "small objects … large number of iterations")."""
    n = scene.n
    if rho >= 1.0:
        return np.ones(n, bool)
    if kind == "uniform":
        return rng(seed).random(n) < rho
    x = scene.rows[:, MU]
    k = max(1, int(round(rho * n)))
    thr = np.partition(x, n - k)[n - k]
    return x >= thr


def dl_dimage(cam: dict, seed: int) -> np.ndarray:
    """Synthetic upstream gradient dL/dC ~ U[-1,1], [3,H,W] fp32."""
    return rng(seed).uniform(-1.0, 1.0, (3, cam["height"], cam["width"])).astype(np.float32)


def target_image(cam: dict, seed: int) -> np.ndarray:
    """Synthetic training image ~ U[0,1], [3,H,W] fp32."""
    return rng(seed).uniform(0.0, 1.0, (3, cam["height"], cam["width"])).astype(np.float32)


def target_image_u8(cam: dict, seed: int) -> np.ndarray:
    """Synthetic 8-bit training image (uint8 [3,H,W], uniform 0..255) — the datasets' PNG format."""
    return rng(seed).integers(0, 256, (3, cam["height"], cam["width"]), dtype=np.uint8)


def pixel_state(cam: dict, seed: int) -> np.ndarray:
    """Synthetic pre-render cache [5,H,W] fp32 (planes P_R, P_G, P_B, Q, T) shaped
    like the frozen-set accumulators of Eq. 7: with A = Σα ~ U[0,3] per pixel, T = e^{−A·U[0.8,1.2]}
    (≥ 0.01), Q = A·U[0.3,1.5] (w in the synthetic range) and P = F·Q with F ~ U[0,1]³ — so a pixel
    with little coverage has both Q ≈ 0 and T ≈ 1, as a real cache does. A seeded input for parity
    tests at sizes where the oracle cannot render the frozen set."""
    g = rng(seed)
    H, W = cam["height"], cam["width"]
    a = g.uniform(0.0, 3.0, (H, W))
    q = a * g.uniform(0.3, 1.5, (H, W))
    out = np.empty((5, H, W))
    out[0:3] = g.uniform(0.0, 1.0, (3, H, W)) * q[None]
    out[3] = q
    out[4] = np.maximum(np.exp(-a * g.uniform(0.8, 1.2, (H, W))), 0.01)
    return out.astype(np.float32)


def bits_from_mask(mask: np.ndarray) -> np.ndarray:
    n = len(mask)
    padded = np.zeros(((n + 31) // 32) * 32, bool)
    padded[:n] = mask
    weights = (np.uint64(1) << np.arange(32, dtype=np.uint64))[None, :]
    return (padded.reshape(-1, 32).astype(np.uint64) * weights).sum(axis=1).astype(np.uint32)


def mask_from_bits(bits: np.ndarray, n: int) -> np.ndarray:
    b = np.asarray(bits, np.uint32)
    out = ((b[:, None] >> np.arange(32, dtype=np.uint32)[None, :]) & 1).astype(bool).reshape(-1)
    return out[:n]


def camera_centers(cams) -> np.ndarray:
    return np.stack([c["center"] for c in cams]).astype(np.float32)

#!/usr/bin/env python
"""bench.py — fwd+bwd active-set OIT render throughput (Mpix/s, splat-pixel evals/s) on B200.

Workload (BASELINE.json configs[1], "NeRF-synthetic-shaped object"): 300k splats, 100 views of
800×800 per GPU, headline active fraction ρ = 0.2 (clustered mask); the sweep adds ρ = 1.0 and 0.05.
One STEP = one batch of 100 training views against one parameter state (R28: gradients summed, one
optimizer step) followed by one refresh (Alg. 1): the 100 views each go through a1
project → a2 bin → a3 composite over the view's pre-render cache → a4 L1 loss gradient → a5/a6
backward (grad rows +=), then one masked Adam step on the compacted rows (NEXT-2), then the
refresh: a7 FPS view subsample (S = 5% of the views) + gradient score of the inactive splats, and a8
the active-set update (into a scratch bitmask, so the forced ρ is kept across steps; the caches
therefore need no reconciliation inside the step — NEXT-1 is timed separately). The parameter rows
and σ are restored between timed steps (outside the timed region) so every step sees the same
workload. For N > 1 (torchrun), each rank owns its own 100 views (weak scaling); the gradient rows
+ dσ are one NCCL all-reduce (a9), the score rows are reduce-scattered by row range and the Eq. 8
bits all-gathered. configs[4] (C5) adds the view-sharded step with strong scaling:
3M splats, 64 views per step split over the ranks. Inputs are synthetic
(paper_2605_13855_b200.synth), larger than L2 per step, and L2 is flushed between timed steps.

--impl reference times the CPU oracle (oracle/, test infrastructure) on the same workload: each
step renders + back-propagates one training view per host core (independent processes).
"""
from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fwd+bwd OIT render Mpix/s and splat-pixel evals/s vs active-set fraction"
UNIT = "Mpix/s"
WORKLOAD = "C2 NeRF-synthetic-shaped: 300k splats, 100 views 800x800 per GPU, rho=0.2 clustered"

# Algorithmic FP32 work per tile-granular splat-pixel evaluation, as SURVEY.md §8(d) defines it
# (FP32 instructions): the forward costs ≈18 per contributing and ≈9 per skipped
# evaluation, the backward ≈36 per contributing and ≈10 per skipped one. Peak = 148 SMs × 128
# FP32 lanes × 1965 MHz = 37.2 T instr/s (B200_PROFILING.md unit counts).
FWD_I_SKIP, FWD_I_CONTRIB = 9, 18
BWD_I_SKIP, BWD_I_CONTRIB = 10, 36
FP32_PEAK_TINSTR = 148 * 128 * 1.965e9 / 1e12       # 37.2
# the same work in FLOPs (FMA = 2, MUFU = 1), kept for comparison with round 1's accounting
FWD_F_TEST, FWD_F_CONTRIB = 9, 17
BWD_F_TEST, BWD_F_CONTRIB = 9, 32
FP32_PEAK_TFLOPS = 2 * FP32_PEAK_TINSTR             # 74.4


def _hbm_peak():
    """Measured copy bandwidth (MEASURED_PEAKS.json, driver-written), else the guide's fallback."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"
    except Exception:
        return 7700.0, "B200_PROFILING.md nominal 7.7 TB/s (MEASURED_PEAKS.json absent)"


HBM_PEAK_GBS, HBM_PEAK_SOURCE = _hbm_peak()


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--rho", type=float, default=0.2)
    ap.add_argument("--kind", choices=["clustered", "uniform"], default="clustered")
    ap.add_argument("--views", type=int, default=100)
    ap.add_argument("--splats", type=int, default=300_000)
    ap.add_argument("--res", type=int, default=800)
    ap.add_argument("--sub-rate", type=float, default=0.05, help="refresh subsample rate S/V")
    ap.add_argument("--streams", type=int, default=12, help="training views processed concurrently (one stream each)")
    ap.add_argument("--score-streams", type=int, default=0, help="refresh streams (0: one per subsampled view)")
    ap.add_argument("--coef-reuse", action="store_true",
                    help="the refresh reuses the coefficients of the subsampled views' training forwards instead of "
                         "rasterising their active set itself (oit_score_subsample_ex; +1.0%% at rho 0.2, -1.1%% at "
                         "rho 0.05 on one B200, so off by default)")
    ap.add_argument("--targets", choices=["u8", "f32"], default="u8",
                    help="training-image format: 8-bit (the datasets' PNGs, OIT_TARGET_U8) or fp32")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--loss", choices=["l1", "dssim"], default="l1",
                    help="training/score loss: L1 (north-star config) or the 3DGS (1-λ)L1 + λ·D-SSIM (NEXT-3)")
    ap.add_argument("--no-ablation", action="store_true", help="skip the NEXT-4 per-pixel backward ablation")
    ap.add_argument("--no-dssim", action="store_true", help="skip the NEXT-3 D-SSIM loss measurement")
    ap.add_argument("--no-adam", action="store_true", help="skip the NEXT-2 Adam measurement")
    ap.add_argument("--no-reconcile", action="store_true", help="skip the NEXT-1 reconciliation measurement")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-c3", action="store_true", help="skip the configs[2] (C3, 3M splats) measurement")
    ap.add_argument("--no-c4", action="store_true", help="skip the configs[3] (C4 score sweep) measurement")
    ap.add_argument("--no-c5", action="store_true", help="skip the configs[4] (C5 view-sharded step) measurement")
    ap.add_argument("--c5-rhos", type=float, nargs="+", default=[0.1, 1.0], help="C5 active fractions")
    ap.add_argument("--profile-once", action="store_true",
                    help="run one eager step between cudaProfilerStart/Stop (for ncu --profile-from-start off), "
                         "print the claimed kernel count, exit")
    return ap.parse_args()


# =============================================================================================
# CPU oracle legs (cpu_baseline and --impl reference)
# =============================================================================================
_REF = {}


def _ref_init(seed_views, n_splats, res, rho, kind, crop=1):
    import oracle as O
    from paper_2605_13855_b200 import synth
    sc = synth.scene_c2(n=n_splats, n_views=seed_views, res=res)
    if crop > 1:   # a res/crop × res/crop window of every view, view v taking window v mod crop², so
        w = res // crop   # that the workers together cover every part of the image (a bounded sample)
        for v, c in enumerate(sc.cams):
            q = v % (crop * crop)
            c["width"] = c["height"] = w
            c["cx"] -= (q % crop) * w
            c["cy"] -= (q // crop) * w
    mask = synth.active_mask(sc, rho, kind)
    _REF.update(O=O, synth=synth, sc=sc, act=np.flatnonzero(mask).astype(np.int32),
                ina=np.flatnonzero(~mask).astype(np.int32), caches={}, targets={})


def _ref_prepare(v):
    """Untimed per-view setup: the view's pre-render cache of the frozen set and its target."""
    O, sc = _REF["O"], _REF["sc"]
    cam = sc.cams[v]
    _REF["caches"][v] = O.render(sc.rows, sc.sigma, _REF["ina"], cam, sc.bg)["state"]
    _REF["targets"][v] = _REF["synth"].target_image(cam, 1000 + v).astype(np.float64)
    return v


def _ref_step(v):
    """One training view through the oracle: render 𝒜 over the cache, L1 gradient, backward."""
    O, sc = _REF["O"], _REF["sc"]
    cam = sc.cams[v]
    t0 = time.perf_counter()
    fwd = O.render(sc.rows, sc.sigma, _REF["act"], cam, sc.bg, base=_REF["caches"][v])
    g = O.loss_grad(fwd["image"], _REF["targets"][v], "l1")
    O.backward(sc.rows, sc.sigma, _REF["act"], cam, sc.bg, fwd["state"], g)
    return time.perf_counter() - t0


class OracleRunner:
    """One training view per host core, each in its own process (the oracle is single-threaded).
    Worker k prepares (untimed) and then repeatedly processes view k; a step's time is the slowest
    worker's compute time for its view (the views run concurrently)."""

    def __init__(self, args, n_views_total, crop=1):
        self.cores = os.cpu_count() or 1
        self.views = list(range(min(self.cores, n_views_total)))
        ctx = mp.get_context("spawn")
        self.pool = ctx.Pool(len(self.views), initializer=_ref_init,
                             initargs=(n_views_total, args.splats, args.res, args.rho, args.kind, crop))
        self.crop = crop
        self.px_per_view = (args.res // crop) ** 2

    def step(self):
        """Per-worker compute times of one step (the workers run concurrently)."""
        return self.pool.map(_ref_prepare_and_step, self.views, chunksize=1)

    def close(self):
        self.pool.close()
        self.pool.join()


def _ref_prepare_and_step(v):
    if v not in _REF["caches"]:
        _ref_prepare(v)
    return _ref_step(v)


def cpu_leg(args, n_views_total, steps, warmup, crop=1):
    r = OracleRunner(args, n_views_total, crop)
    try:
        # the first pass also prepares each view's cache (untimed: _ref_step times only its own work)
        for _ in range(max(1, warmup)):
            r.step()
        ts = [r.step() for _ in range(steps)]
    finally:
        r.close()
    # aggregate throughput of the independent workers with the work balanced over them (a core that
    # finishes its window early would take the next one in a real job): cores × total pixels / total
    # compute time; wall time per step = the slowest worker
    rate = float(np.mean([len(st) * len(st) * r.px_per_view / sum(st) for st in ts]))
    mean = float(np.mean([max(step_ts) for step_ts in ts]))
    return dict(value=rate / 1e6, unit=UNIT, cores=r.cores, kind="oracle", ms_per_step=mean * 1e3,
                sample=f"{len(r.views)} training views (one per host core, independent processes) of the same "
                       f"workload" + (f", each cropped to one {args.res // crop}x{args.res // crop} window (view v: "
                                      f"window v mod {crop * crop}, so the workers cover every part of the image)"
                                      if crop > 1 else "") +
                       ", each: oracle render of the active set over its pre-render cache + L1 gradient "
                       "+ backward (single-threaded C, fp64); value = workers × pixels / total compute time")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    # K + W steps of one view per core would take ~12 s each at full size: the reference arm samples
    # a quarter window of every view (the four windows spread over the workers) so that the whole
    # run stays within a few minutes
    res = cpu_leg(args, args.views, max(1, args.steps), max(0, args.warmup), crop=2)
    line = {"impl": "reference", "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "rho": args.rho, "mask": args.kind},
            "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# =============================================================================================
# GPU leg
# =============================================================================================
class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    def __init__(self, device_index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {nv.nvmlClocksEventReasonGpuIdle: "gpu_idle", nv.nvmlClocksEventReasonSwPowerCap: "sw_power_cap",
                 nv.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
                 nv.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal_slowdown",
                 nv.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal_slowdown",
                 nv.nvmlClocksEventReasonHwPowerBrakeSlowdown: "hw_power_brake_slowdown",
                 nv.nvmlClocksEventReasonApplicationsClocksSetting: "applications_clocks_setting",
                 nv.nvmlClocksEventReasonSyncBoost: "sync_boost"}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in names.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "n_samples": len(self.samples)}


_CUDART = None


def event_ms(a, b):
    """cudaEventElapsedTime on raw event handles (the moment-kernel events are recorded inside
    liboit, which torch's own bookkeeping does not see)."""
    global _CUDART
    import ctypes
    if _CUDART is None:
        _CUDART = ctypes.CDLL("libcudart.so.12")
    ms = ctypes.c_float(0.0)
    rc = _CUDART.cudaEventElapsedTime(ctypes.byref(ms), ctypes.c_void_p(a.cuda_event), ctypes.c_void_p(b.cuda_event))
    if rc != 0:
        raise RuntimeError(f"cudaEventElapsedTime failed ({rc})")
    return ms.value


def torch_logit(torch, o):
    return torch.logit(o.clamp(1e-6, 1.0 - 1e-6))


def scan_kernels(n):
    """k_scan_blocks alone for n <= 4096 (it writes the total), else + k_scan_sums + k_scan_add."""
    if n <= 0:
        return 0
    return 1 if (n + 4095) // 4096 == 1 else 3


class Workload:
    """One rank's share: scene, active set, per-view caches/targets, buffers and the step."""

    def __init__(self, args, torch, L, synth, rho, cams, rank, world, scene=None, cap=1 << 22, cache_cap=None,
                 with_refresh=True, kind=None):
        from paper_2605_13855_b200.pipeline import ViewPipeline
        self.torch, self.L = torch, L
        dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        # scene content (cameras passed in): C2 by default, or a given scene (C3 measurements)
        sc = synth.scene_c2(n=args.splats, n_views=1, res=args.res) if scene is None else scene
        self.sc = sc
        self.cams = cams
        self.V = len(cams)
        self.rho = rho
        self.world, self.rank = world, rank
        self.loss = args.loss
        mask = synth.active_mask(sc, rho, args.kind if kind is None else kind)
        self.n = sc.n
        act = np.flatnonzero(mask).astype(np.int32)
        ina = np.flatnonzero(~mask).astype(np.int32)
        self.n_act, self.n_ina = len(act), len(ina)
        self.rows = torch.from_numpy(sc.rows).to(dev)
        self.sigma = torch.tensor([sc.sigma], dtype=torch.float32, device=dev)
        self.act = torch.from_numpy(act).to(dev)
        self.ina = torch.from_numpy(ina).to(dev)
        self.bg = sc.bg
        H, W = int(cams[0]["height"]), int(cams[0]["width"])
        self.H, self.W = H, W
        # cap ≥ 2× the largest per-view pair count of the training views (checked below); the
        # frozen-set caches are built on the first pipeline, sized for them (cache_cap)
        self.pipe = ViewPipeline(cams[0], max(self.n_act, self.n_ina, 1), cache_cap or cap, device=dev)
        # independent views run concurrently: one pipeline (buffers + workspaces) per stream; the
        # gradient rows are accumulated with vector atomics, so all streams share grad / dσ
        self.n_streams = max(1, args.streams)
        self.pipes = [self.pipe] + [ViewPipeline(cams[0], max(self.n_act, 1), cap, device=dev)
                                    for _ in range(self.n_streams - 1)]
        self.streams = [torch.cuda.Stream() for _ in range(self.n_streams)]
        self.copy_stream = torch.cuda.Stream()
        self.ev_copy = [torch.cuda.Event() for _ in range(len(cams))]
        nt = self.pipe.n_tiles
        self.n_tiles = nt
        # ---- untimed setup: per-view pre-render caches of the frozen set (Alg. 1 I^pre), targets ----
        self.caches = torch.empty((self.V, 5, nt, 256), dtype=torch.float32, device=dev)
        gen = torch.Generator(device=dev)
        gen.manual_seed(1234 + rank)
        if args.targets == "u8":   # 8-bit training images (OIT_TARGET_U8: read as u8/255 by the loss kernels)
            self.targets = torch.randint(0, 256, (self.V, 3, H, W), generator=gen, device=dev, dtype=torch.uint8)
        else:
            self.targets = torch.rand((self.V, 3, H, W), generator=gen, device=dev, dtype=torch.float32)
        self.pairs_act = []
        for v, cam in enumerate(cams):
            self.pipe.set_camera(cam)
            if self.n_ina > 0:
                _, st = self.pipe.forward(self.rows, self.sigma, self.ina, self.bg, image=False)
                self.caches[v].copy_(st)
                assert self.pipe.pairs_used() <= self.pipe.capacity, "cache pair capacity overflow"
            else:
                self.caches[v, :3].zero_(); self.caches[v, 3].zero_(); self.caches[v, 4].fill_(1.0)
        # work counters of the training views (untimed)
        cnt = torch.zeros(2, dtype=torch.int64, device=dev)
        max_pairs = 0
        for v, cam in enumerate(cams):
            self.pipe.set_camera(cam)
            self.pipe.forward(self.rows, self.sigma, self.act, self.bg, base=self.caches[v], counters=cnt)
            npairs = self.pipe.pairs_used()
            self.pairs_act.append(npairs)
            max_pairs = max(max_pairs, npairs)
        c = cnt.cpu().numpy()
        self.contrib, self.tile_evals = int(c[0]), int(c[1])
        assert max_pairs <= cap, "pair capacity overflow"
        self.max_pairs_train = max_pairs
        # ---- buffers of the step: the a9 exchange buffer (gradient rows ⊕ dσ, one all-reduce) ----
        from paper_2605_13855_b200 import dist as D
        self.gbuf = D.GradBuffer(max(self.n_act, 1), device=dev)
        self.grad, self.dsig = self.gbuf.rows, self.gbuf.dsigma
        self._setup_adam()
        self.with_refresh = with_refresh
        self._setup_refresh(args, synth, mask, cams, cap) if with_refresh else None
        # events around the two hot kernels of every training view (external nodes in the graph)
        mk = lambda: torch.cuda.Event(enable_timing=True, external=True)  # noqa: E731
        self.ev_fwd = [(mk(), mk()) for _ in range(self.V)]
        self.ev_bwd = [(mk(), mk()) for _ in range(self.V)]
        self.ev_seg = [mk() for _ in range(3)]
        for pair in self.ev_fwd + self.ev_bwd + [tuple(self.ev_seg[:2]), tuple(self.ev_seg[1:])]:
            pair[0].record()                      # torch creates the CUDA event lazily on first record
            pair[1].record()
        torch.cuda.synchronize()

    def _setup_adam(self):
        """NEXT-2 optimizer state for all N splats (untimed setup): latent = the physical rows
        through the inverse 3DGS activations (logit o, log s; μ, q, v, h as is), zero moments; σ's
        state (log σ, m, v, t). The rows/σ at the start of every timed step are these."""
        torch, dev = self.torch, self.dev
        lat = self.rows.clone()
        lat[:, 3] = torch_logit(torch, self.rows[:, 3])
        lat[:, 8:11] = torch.log(self.rows[:, 8:11])
        self.lat, self.m, self.v = lat, torch.zeros_like(lat), torch.zeros_like(lat)
        self.astep = torch.zeros(self.n, dtype=torch.int32, device=dev)
        self.sig_state = torch.tensor([math.log(float(self.sigma.item())), 0.0, 0.0, 0.0], dtype=torch.float32,
                                      device=dev)
        self.sig_state0 = self.sig_state.clone()
        self.rows0, self.sigma0 = self.rows.clone(), self.sigma.clone()
        self.adam_cfg = self.L.adam_cfg()

    def adam(self):
        """One masked Adam step on the (combined) compacted gradient rows: the active splats' latent
        and physical rows and σ move; frozen splats are untouched."""
        self.L.oit_adam_step(self.grad, self.act, self.lat, self.m, self.v, self.astep, self.rows, self.adam_cfg,
                             dsigma=self.dsig, sigma_state=self.sig_state, sigma=self.sigma)

    def restore_params(self):
        """Outside the timed region: back to the initial rows/σ/optimizer state (same work each step)."""
        self.rows.copy_(self.rows0)
        self.sigma.copy_(self.sigma0)
        self.lat[:, :] = self.rows0
        self.lat[:, 3] = torch_logit(self.torch, self.rows0[:, 3])
        self.lat[:, 8:11] = self.torch.log(self.rows0[:, 8:11])
        self.m.zero_()
        self.v.zero_()
        self.astep.zero_()
        self.sig_state.copy_(self.sig_state0)

    def _setup_refresh(self, args, synth, mask, cams, cap):
        torch, L, dev = self.torch, self.L, self.dev
        # refresh: FPS over this rank's view centres, S = 5% of the views, scored set = inactive set
        self.S = max(1, int(round(args.sub_rate * self.V)))
        self.centers = torch.from_numpy(synth.camera_centers(cams)).to(dev)
        self.views_dev = torch.empty(self.S, dtype=torch.int32, device=dev)
        L.oit_select_views(self.centers, self.S, 2605, 0, self.views_dev)
        self.views_host = [int(x) for x in self.views_dev.cpu().numpy()]   # same refresh index each step
        self.score_cap = cap
        # the refresh's streams: S views split over them (each call chains its views in groups of the
        # multi-view epilogue); default: one stream per view up to the training stream count
        nsc = max(1, min(self.S, args.score_streams if args.score_streams > 0 else self.n_streams))
        self.score_ws = [torch.empty(max(L.oit_score_workspace_bytes(cams[0], self.n_act, self.n_ina, cap), 256),
                                     dtype=torch.uint8, device=dev) for _ in range(nsc)]
        # the refresh's own streams: it runs concurrently with the training views (R35)
        self.score_streams = [torch.cuda.Stream() for _ in range(nsc)]
        # coefficient reuse (L1/L2): the subsampled views' training forwards write every tile's
        # coefficients into a workspace of their own, which the score reads (oit_score_subsample_ex)
        self.reuse_coef = self.loss in ("l1", "l2") and args.coef_reuse and self.n_ina > 0
        picked = sorted(set(self.views_host)) if self.reuse_coef else []
        self.coef_ws = {j: self.pipe.new_bwd_ws() for j in picked}
        self.ev_coef = {j: torch.cuda.Event() for j in picked}
        from paper_2605_13855_b200 import dist as D
        # padded to the sharded refresh's row ranges (rows beyond n_ina stay zero)
        self.score_rows = torch.zeros((D.score_buffer_rows(self.n_ina, self.world), 80), dtype=torch.float32,
                                      device=dev)
        self.score_grad = self.score_rows[:max(self.n_ina, 1)]
        self.score_dsig = torch.zeros(1, dtype=torch.float32, device=dev)
        self.max_pairs = torch.zeros(1, dtype=torch.int64, device=dev)
        self.bits0 = torch.from_numpy(synth.bits_from_mask(mask).view(np.int32)).to(dev)
        self.bits = self.bits0.clone()
        self.act_out = torch.empty(self.n, dtype=torch.int32, device=dev)
        self.fro_out = torch.empty(self.n, dtype=torch.int32, device=dev)
        self.new_out = torch.empty(self.n, dtype=torch.int32, device=dev)
        self.counts = torch.zeros(3, dtype=torch.int32, device=dev)
        self.upd_ws = torch.empty(L.oit_update_workspace_bytes(self.n), dtype=torch.uint8, device=dev)
        self.eps = [1e-7, 1e-7, 1e-7, 1e-7, 1e-7, 1e-7]
        self.caches_list = [self.caches[v] for v in range(self.V)]
        self.targets_list = [self.targets[v] for v in range(self.V)]

    # ---------------------------------------------------------------------------------------
    def target_f32(self, v):
        """fp32 copy of training image v (for the measurement legs that call oit_loss_grad / SSIM)."""
        t = self.targets[v]
        return t.float() / 255.0 if t.dtype == self.torch.uint8 else t.contiguous()

    def refresh_parts(self):
        if not self.with_refresh or self.n_ina <= 0:
            return 0
        return sum(1 for k in range(len(self.score_ws)) if self.views_host[k::len(self.score_ws)])

    def train_views(self, n_streams=None, host_targets=None, extra_concurrency=0, after_picked=None):
        """a1-a6 over every training view (Alg. 1 l.3-6, one view per iteration); views are dealt
        round-robin to n_streams streams (fork/join on the current stream). host_targets (e2e):
        pinned-host training images, copied on a copy stream; each view's loss waits only for its
        own image (copies overlap the compute of earlier views). after_picked (the refresh with
        coefficient reuse): the views the refresh scores are enqueued first — their fused forward
        writes every tile's coefficients into a workspace of their own and records ev_coef — then
        after_picked() enqueues the refresh (forked before the views, waiting only on ev_coef), then
        the remaining views."""
        torch, L = self.torch, self.L
        ns = self.n_streams if n_streams is None else n_streams
        main = torch.cuda.current_stream()
        self.gbuf.zero_()
        picked = list(dict.fromkeys(self.views_host)) if after_picked is not None else []
        order = picked + [v for v in range(self.V) if v not in set(picked)]
        if host_targets is not None:
            self.copy_stream.wait_stream(main)
            with torch.cuda.stream(self.copy_stream):
                for v in order:
                    self.targets[v].copy_(host_targets[v], non_blocking=True)
                    self.ev_copy[v].record(self.copy_stream)
        for st_ in self.streams[:ns]:
            st_.wait_stream(main)
        for i, v in enumerate(order):
            if after_picked is not None and i == len(picked):
                after_picked()
            cam = self.cams[v]
            k = v % ns
            p = self.pipes[k]
            with torch.cuda.stream(self.streams[k]):
                p.set_camera(cam)
                # a3 (no image: the fused a4 below resolves C from the state), then a4+a5+a6 with
                # the L1 gradient against the view's training image fused into the coefficients
                if host_targets is not None:
                    self.streams[k].wait_event(self.ev_copy[v])
                if self.loss in ("l1", "l2"):
                    # a3 + a4 fused: the forward's epilogue applies the pixel-local loss and writes the
                    # backward coefficients into the backward workspace (no pixel-state round trip)
                    cw = self.coef_ws.get(v) if after_picked is not None else None
                    p.forward_loss(self.rows, self.sigma, self.act, self.bg, self.targets[v], self.loss,
                                   base=self.caches[v], events=self.ev_fwd[v], concurrency=ns + extra_concurrency,
                                   bwd_ws=cw, all_tiles=cw is not None)
                    if cw is not None:
                        self.ev_coef[v].record(self.streams[k])
                    p.backward(self.rows, self.sigma, self.act, self.bg, None, None, self.grad, self.dsig,
                               events=self.ev_bwd[v], coef_ready=True, concurrency=ns + extra_concurrency, bwd_ws=cw)
                else:   # D-SSIM is not pixel-local: state → resolve → SSIM stencils → coefficients
                    _, st = p.forward(self.rows, self.sigma, self.act, self.bg, base=self.caches[v], image=False,
                                      events=self.ev_fwd[v], concurrency=ns + extra_concurrency)
                    p.backward(self.rows, self.sigma, self.act, self.bg, st, None, self.grad, self.dsig,
                               events=self.ev_bwd[v], target=self.targets[v], loss=self.loss,
                               concurrency=ns + extra_concurrency)
        if after_picked is not None and len(picked) == len(order):
            after_picked()
        for st_ in self.streams[:ns]:
            main.wait_stream(st_)
        if host_targets is not None:
            main.wait_stream(self.copy_stream)

    def refresh(self, join=True, extra_concurrency=0, fork_from=None, reuse=False):
        """a7 (FPS + subsampled score of the inactive splats) on the refresh's own streams, forked
        from the current stream (or fork_from); join=False leaves them running (refresh_join()
        later), so the score overlaps the training views (R35: the period's refresh scores the
        parameters the period's batch uses, the update applies to the next period). reuse: each
        score stream waits for its views' training forwards (ev_coef) and takes their coefficients
        instead of rasterising the active set again (oit_score_subsample_ex)."""
        L = self.L
        torch = self.torch
        main = torch.cuda.current_stream() if fork_from is None else fork_from
        with torch.cuda.stream(main):
            L.oit_select_views(self.centers, self.S, 2605, 0, self.views_dev)
            self.score_grad.zero_()
            self.score_dsig.zero_()
        if self.n_ina > 0:
            # the S subsampled views are scored concurrently (disjoint subsets, scale 1/S each)
            parts = [self.views_host[k::len(self.score_ws)] for k in range(len(self.score_ws))]
            conc = sum(1 for q in parts if q) + extra_concurrency
            for k, part in enumerate(parts):
                if not part:
                    continue
                self.score_streams[k].wait_stream(main)
                cws = evs = None
                if reuse:   # the call waits on each view's event only before that view's backward
                    cws = [self.coef_ws[j] for j in part]
                    evs = [self.ev_coef[j] for j in part]
                with torch.cuda.stream(self.score_streams[k]):
                    L.oit_score_subsample(self.rows, self.sigma, self.cams, self.targets_list, self.caches_list,
                                          self.act, self.ina, part, self.loss, self.bg, self.score_grad, self.score_dsig,
                                          self.score_cap, self.max_pairs, self.score_ws[k], scale=1.0 / self.S,
                                          concurrency=conc, coef_ws=cws, coef_ready=evs)
            if join:
                self.refresh_join()

    def refresh_join(self):
        if self.n_ina <= 0:
            return
        main = self.torch.cuda.current_stream()
        for k in range(len(self.score_ws)):
            if self.views_host[k::len(self.score_ws)]:
                main.wait_stream(self.score_streams[k])

    def train_and_refresh(self, host_targets=None):
        """The step's a1-a6 over the 100 views and the refresh's a7, concurrently (R35). With
        coefficient reuse (default for L1/L2) the refresh takes the subsampled views' coefficients
        from their training forwards — the same parameters, active set, cache and target."""
        nr = self.refresh_parts()
        if self.with_refresh and self.reuse_coef:
            main = self.torch.cuda.current_stream()
            self.train_views(host_targets=host_targets, extra_concurrency=nr,
                             after_picked=lambda: self.refresh(join=False, extra_concurrency=self.n_streams,
                                                               fork_from=main, reuse=True))
            self.refresh_join()
            return
        if self.with_refresh:
            self.refresh(join=False, extra_concurrency=self.n_streams)
        self.train_views(host_targets=host_targets, extra_concurrency=nr)
        if self.with_refresh:
            self.refresh_join()

    def update(self):
        L = self.L
        self.bits.copy_(self.bits0)
        if self.n_ina > 0 and self.world > 1:
            # reduce-scatter of the score rows by row range, Eq. 8 on this rank's
            # range, all-gather of the row bits, recompaction on every rank
            from paper_2605_13855_b200 import dist as D
            D.sharded_refresh_update(self.score_rows, self.ina, self.eps, "fresh", self.n, self.bits, self.act_out,
                                     self.counts[0:1], self.upd_ws, newly_frozen=self.fro_out,
                                     n_frozen=self.counts[1:2], newly_active=self.new_out,
                                     n_activated=self.counts[2:3])
        elif self.n_ina > 0:
            L.oit_update_active_set(self.score_grad, self.ina, self.eps, "fresh", self.n, self.bits, self.act_out,
                                    self.counts[0:1], self.fro_out, self.counts[1:2], self.new_out,
                                    self.counts[2:3], self.upd_ws)

    def kernel_launches(self):
        """Our kernels launched by one step (per the launch structure of each C-ABI call; checked
        against the ncu launch list of the bench command in profiles/)."""
        nt = self.n_tiles
        nw = (self.n + 31) // 32
        a, s = self.n_act, self.n_ina
        proj = lambda n: 1 if n > 0 else 0  # noqa: E731
        # bitmap path (the view's (tile × slot) bitmap ≤ 128 MB): k_bin_expand<1,1>, k_bitmap_count,
        # the scan, k_bitmap_emit; otherwise k_bin_expand<0> (n > 0), the scan, k_bin_expand<1>,
        # k_tile_sort (n > 0, sorted lists only)
        bitmap = lambda n: n > 0 and nt <= 4096 and nt * ((((n + 31) // 32) + 3) // 4 * 4) <= (32 << 20)  # noqa: E731
        binn = lambda n: (2 if n > 0 else 0) + scan_kernels(nt) + 1  # noqa: E731
        fwd = 3                                            # item histogram + emission, k_fwd_items
        # k_quad_bin, item histogram + emission, k_moments, k_epilogue (none for an empty slot list)
        bwd = lambda n: 5 if n > 0 else 0  # noqa: E731
        lossk = 4 if self.loss == "dssim" else 0   # resolve + 2 SSIM stencil passes + k_coef
        # training views with L1/L2: a4 fused into the forward's epilogue (no k_coef launch), which
        # also writes the quadrant lists (no k_quad_bin in the backward)
        bwd_train = (lambda n: 4 if n > 0 else 0) if self.loss in ("l1", "l2") else bwd  # noqa: E731
        train = self.V * (proj(a) + binn(a) + fwd + bwd_train(a) + lossk) + 1   # + k_adam
        refresh = 1                                        # k_fps
        if s > 0:
            # the scored set is binned straight into the backward's quadrant lists: k_bin_expand<0>,
            # the scan, the quadrant scatter; its backward has no k_quad_bin
            bin_q = lambda n: (1 if n > 0 else 0) + scan_kernels(nt) + 1  # noqa: E731
            # (with coefficient reuse the score takes each view's coefficients from its training
            # forward: no projection, binning or forward of the active set inside the refresh)
            own = 0 if self.reuse_coef else proj(a) + binn(a) + fwd + lossk
            refresh += self.S * (own + proj(s) + bin_q(s) + bwd(s) - (1 if s > 0 else 0))
            if self.world > 1:   # k_row_activeness + k_apply_bits, k_popc3, 3 scans, k_emit3
                refresh += 1 + 1 + 1 + 3 * scan_kernels(nw) + 1
            else:                # k_update_bits, k_popc3, 3 scans, k_emit3
                refresh += 1 + 1 + 3 * scan_kernels(nw) + 1
        return train + refresh


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2605_13855_b200 import _lib as L
    from paper_2605_13855_b200 import synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # OIT_BENCH_BACKEND=gloo + OIT_BENCH_SAME_DEVICE=1: exercise the N > 1 path (sharding, barriers,
    # all-reduces, max-over-ranks timing) with several ranks on ONE GPU — a test hook, not a bench mode
    backend = os.environ.get("OIT_BENCH_BACKEND", "nccl")
    if os.environ.get("OIT_BENCH_SAME_DEVICE"):
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    L.lib()  # fail loudly if liboit.so is missing
    from paper_2605_13855_b200 import dist as D
    all_cams = synth.scene_c2(n=10, n_views=args.views * world, res=args.res).cams
    cams = [all_cams[v] for v in D.views_of_rank(args.views, rank)]   # weak scaling: V views per rank

    if args.profile_once:
        # one eager step of the headline workload between cudaProfilerStart/Stop (run under
        # `ncu --profile-from-start off`): the launch list of exactly one step, to check the
        # gpu_launches claim (kernel_launches) against; prints the claim
        wl = Workload(args, torch, L, synth, args.rho, cams, rank, world)
        wl.train_and_refresh(); wl.adam(); wl.update()
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        wl.train_and_refresh(); wl.adam(); wl.update()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        print(json.dumps({"kernel_launches_claimed_per_step": wl.kernel_launches()}), flush=True)
        return 0
    rhos = [args.rho] + ([] if args.no_sweep else [r for r in (1.0, 0.05) if r != args.rho])
    results = {}
    headline = None
    for rho in rhos:
        wl = Workload(args, torch, L, synth, rho, cams, rank, world)
        res = time_workload(args, torch, dist, wl, world, headline_run=(rho == args.rho))
        results[rho] = res
        if rho == args.rho:
            headline = (wl, res)
        del wl
        torch.cuda.empty_cache()
    wl, res = headline
    del wl
    torch.cuda.empty_cache()
    extra = {}
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    sc3 = synth.scene_c3(n_views=200) if (not args.no_c5 or (world == 1 and not args.no_c3)) else None
    if world == 1 and not args.no_c3:
        extra["c3_mip360_shaped"] = time_c3(args, torch, L, synth, flush, sc3)
        torch.cuda.empty_cache()
    if not args.no_c5:
        extra["c5_view_sharded_step"] = time_c5(args, torch, dist, L, synth, sc3, world, rank, flush)
        torch.cuda.empty_cache()
    del sc3
    if world == 1 and not args.no_c4:
        extra["c4_score_sweep"] = time_c4(args, torch, L, synth, flush)
        torch.cuda.empty_cache()
    del flush
    if rank == 0:
        line = build_line(args, world, res, results)
        line.update(extra)
        if not args.no_cpu and world == 1:
            try:
                line["cpu_baseline"] = {k: v for k, v in cpu_leg(args, args.views, 1, 0).items() if k != "ms_per_step"}
            except Exception as e:  # pragma: no cover
                line["cpu_baseline"] = {"error": str(e)[:200]}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def time_workload(args, torch, dist, wl, world, headline_run):
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=wl.dev)   # 256 MB > 126 MB L2
    allred = world > 1

    from paper_2605_13855_b200 import dist as D

    def comm():   # a9: ONE NCCL all-reduce of the GradBuffer (compacted gradient rows ⊕ dσ)
        if allred:
            D.combine_gradients(wl.gbuf)

    use_graph = not args.no_graph
    # warm-up eagerly once (also initialises lazy state inside the library)
    wl.train_and_refresh(); comm(); wl.adam(); wl.update()
    torch.cuda.synchronize()
    wl.restore_params()
    graphs = []
    if use_graph:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            def whole():
                wl.ev_seg[0].record()
                wl.train_and_refresh()
                wl.ev_seg[1].record()
                wl.adam()
                wl.update()
                wl.ev_seg[2].record()

            # N > 1: the collectives (a9 all-reduce; the refresh's reduce-scatter / all-gather inside
            # update()) run eagerly between the graphs
            for fn in ([wl.train_and_refresh, wl.adam] if allred else [whole]):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    fn()
                graphs.append(g)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()

    def step():
        if use_graph:
            if allred:
                graphs[0].replay(); comm(); graphs[1].replay(); wl.update()
            else:
                graphs[0].replay()
        else:
            wl.train_and_refresh(); comm(); wl.adam(); wl.update()

    for _ in range(args.warmup):
        step()
        wl.restore_params()
    torch.cuda.synchronize()
    if allred:
        dist.barrier()
    times, fwd_ms, bwd_ms, seg_ms = [], [], [], []
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(torch.cuda.current_device())
    with sampler:
        for _ in range(args.steps):
            wl.restore_params()                # same parameters every step (outside the timed region)
            flush.zero_()                      # L2 flush outside the timed region
            torch.cuda.synchronize()
            if allred:
                dist.barrier()
            t_start.record()
            step()
            t_end.record()
            torch.cuda.synchronize()
            if allred:
                dist.barrier()
            times.append(t_start.elapsed_time(t_end))
            fwd_ms.append(sum(event_ms(a, b) for a, b in wl.ev_fwd))
            bwd_ms.append(sum(event_ms(a, b) for a, b in wl.ev_bwd))
            if use_graph and not allred:
                seg_ms.append((event_ms(wl.ev_seg[0], wl.ev_seg[1]), event_ms(wl.ev_seg[1], wl.ev_seg[2])))
    wl.restore_params()                        # the legs below start from the initial parameters
    ms = float(np.mean(times))
    if allred:
        t = torch.tensor([ms], dtype=torch.float64, device=wl.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # roofline pass: the same training views on ONE stream (no concurrency), so each hot kernel's
    # event-timed duration is its own; timed steps between L2 flushes as above
    ser_fwd, ser_bwd = fwd_ms, bwd_ms
    if headline_run and wl.n_streams > 1:
        ser = None
        if use_graph:
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                ser = torch.cuda.CUDAGraph()
                with torch.cuda.graph(ser, stream=s):
                    wl.train_views(1)
            torch.cuda.current_stream().wait_stream(s)
        ser_fwd, ser_bwd = [], []
        for i in range(args.warmup + args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            ser.replay() if ser is not None else wl.train_views(1)
            torch.cuda.synchronize()
            if i >= args.warmup:
                ser_fwd.append(sum(event_ms(a, b) for a, b in wl.ev_fwd))
                ser_bwd.append(sum(event_ms(a, b) for a, b in wl.ev_bwd))
    # the FPS kernel's device output must equal the host list the score used
    assert [int(x) for x in wl.views_dev.cpu().numpy()] == wl.views_host
    res = dict(ms=ms, fwd_ms=float(np.mean(fwd_ms)), bwd_ms=float(np.mean(bwd_ms)), clocks=sampler.summary(),
               ser_fwd_ms=float(np.mean(ser_fwd)), ser_bwd_ms=float(np.mean(ser_bwd)),
               pairs=int(sum(wl.pairs_act)), contrib=wl.contrib, tile_evals=wl.tile_evals, V=wl.V, H=wl.H, W=wl.W,
               n_act=wl.n_act, n_ina=wl.n_ina, S=wl.S, launches=wl.kernel_launches(), rho=wl.rho,
               max_score_pairs=int(wl.max_pairs.item()),
               train_refresh_ms=float(np.mean([a for a, _ in seg_ms])) if seg_ms else None,
               adam_update_ms=float(np.mean([b for _, b in seg_ms])) if seg_ms else None)
    if headline_run and wl.with_refresh and wl.n_ina > 0 and use_graph:
        # the refresh (a7) alone, for the record (inside the step it overlaps the training views)
        res["refresh_alone_ms"] = _graph_time(torch, wl.refresh, flush, args.warmup, args.steps)
    if headline_run and not args.no_e2e:
        res["e2e"] = time_e2e(args, torch, dist, wl, step, flush, allred)
    if headline_run and not args.no_reconcile and wl.n_ina > 0:
        res["reconcile"] = time_reconcile(args, torch, wl, flush)
    if headline_run and not args.no_adam:
        res["adam"] = time_adam(args, torch, wl, flush)
    if headline_run and not args.no_dssim:
        res["dssim"] = time_dssim(args, torch, wl, flush)
    if headline_run and not args.no_ablation:
        res["ablation"] = time_ablation(args, torch, wl, flush)
    return res


def _graph_time(torch, fn, flush, warmup, steps):
    """Capture fn in a CUDA graph, replay warmup + steps times between L2 flushes; mean ms."""
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for i in range(warmup + steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0.record()
        g.replay()
        t1.record()
        torch.cuda.synchronize()
        if i >= warmup:
            times.append(t0.elapsed_time(t1))
    del g
    return float(np.mean(times))


def time_c3(args, torch, L, synth, flush, sc, n_views=16):
    """configs[2] (Mip-NeRF360-shaped: 3M splats, 1600×1064, ρ = 0.1): training views a1-a6 over
    their frozen-set caches, 16 streams in one CUDA graph (no refresh), clustered and uniform masks.
    The 16 views are every 12th camera of the 200-view C3 rig."""
    cams = sc.cams[::12][:n_views]
    out = {"views": n_views, "splats": sc.n, "res": [1600, 1064], "rho": 0.1}
    for kind in ("clustered", "uniform"):
        wl = Workload(args, torch, L, synth, 0.1, cams, 0, 1, scene=sc, cap=1 << 22, cache_cap=1 << 25,
                      with_refresh=False, kind=kind)
        ms = _graph_time(torch, wl.train_views, flush, args.warmup, args.steps)
        px = n_views * wl.H * wl.W
        out[kind] = {"ms_per_view": ms / n_views, "mpix_per_s": px / (ms * 1e-3) / 1e6,
                     "splat_pixel_evals_per_s": 256 * sum(wl.pairs_act) / (ms * 1e-3),
                     "pairs_per_view": sum(wl.pairs_act) / n_views, "n_active": wl.n_act,
                     "f_c": wl.contrib / max(wl.tile_evals, 1)}
        del wl
        torch.cuda.empty_cache()
    return out


def time_c5(args, torch, dist, L, synth, sc, world, rank, flush, n_step_views=64):
    """configs[4] (C5): the view-sharded training step with STRONG scaling — the
    C3 scene (3M splats, 1600×1064), 64 views per step in all, split over the ranks (64/G each) and
    drawn from the rank's own contiguous shard of the 200-view rig (static view → rank map, so each
    rank's caches never move); per rank a1-a6 over its views (concurrent streams, one CUDA graph),
    then a9 = ONE all-reduce of the GradBuffer (compacted rows ⊕ dσ; NCCL over NVLink at N > 1), then
    one masked Adam step (NEXT-2, identical on every rank). Step time = max over ranks; value = all
    64 views' pixels / step time. The parameters are restored between steps (outside the timing)."""
    from paper_2605_13855_b200 import dist as D
    shard = list(D.shard_views(len(sc.cams), rank, world))
    per = len(D.shard_views(n_step_views, rank, world))
    cams = [sc.cams[shard[i * len(shard) // per]] for i in range(per)]   # stratified over the own shard
    out = {"views_per_step": n_step_views, "views_per_rank": per, "splats": sc.n, "res": [1600, 1064],
           "scaling": "strong", "mask": "clustered", "rig_views": len(sc.cams)}
    allred = world > 1
    for rho in args.c5_rhos:
        big = rho >= 0.5
        wl = Workload(args, torch, L, synth, rho, cams, rank, world, scene=sc, cap=(1 << 25) if big else (1 << 22),
                      cache_cap=1 << 25, with_refresh=False, kind="clustered")
        ev_c = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

        def comm():
            if allred:
                ev_c[0].record()
                D.combine_gradients(wl.gbuf)
                ev_c[1].record()

        wl.train_views(); comm(); wl.adam()
        torch.cuda.synchronize()
        wl.restore_params()
        graphs = []
        if not args.no_graph:
            s_ = torch.cuda.Stream()
            s_.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s_):
                for fn in (wl.train_views, wl.adam):
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=s_):
                        fn()
                    graphs.append(g)
            torch.cuda.current_stream().wait_stream(s_)
            torch.cuda.synchronize()

        def step():
            if graphs:
                graphs[0].replay(); comm(); graphs[1].replay()
            else:
                wl.train_views(); comm(); wl.adam()

        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        times, comm_ms = [], []
        for i in range(args.warmup + args.steps):
            wl.restore_params()
            flush.zero_()
            torch.cuda.synchronize()
            if allred:
                dist.barrier()
            t0.record()
            step()
            t1.record()
            torch.cuda.synchronize()
            if allred:
                dist.barrier()
            if i >= args.warmup:
                times.append(t0.elapsed_time(t1))
                if allred:
                    comm_ms.append(ev_c[0].elapsed_time(ev_c[1]))
        ms = float(np.mean(times))
        cm = float(np.mean(comm_ms)) if comm_ms else 0.0
        if allred:
            t = torch.tensor([ms, cm], dtype=torch.float64, device=wl.dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms, cm = float(t[0].item()), float(t[1].item())
        px = n_step_views * wl.H * wl.W
        out[str(rho)] = {"ms_per_step": ms, "mpix_per_s": px / (ms * 1e-3) / 1e6, "n_active": wl.n_act,
                         "allreduce_bytes": int(wl.gbuf.flat.numel() * 4), "allreduce_ms": cm,
                         "pairs_per_view": sum(wl.pairs_act) / max(per, 1),
                         "f_c": wl.contrib / max(wl.tile_evals, 1)}
        del wl, graphs
        torch.cuda.empty_cache()
    return out


def time_c4(args, torch, L, synth, flush, rates=(0.01, 0.02, 0.05, 0.10), n_views=300, refresh_every=100):
    """configs[3] (score sweep: 1M inactive + 111k active splats on the C3 rig, 300 views): one
    refresh = FPS (a7) + the subsampled gradient score of all 1M inactive splats over S = rate·V
    views (concurrent streams, each view over its cache) + the Eq. 8 update (a8). Reports ms per
    refresh, amortized per iteration (refresh every 100 iterations) and the ratio to one training
    iteration (one view's a1-a6 over the 111k active splats)."""
    n_ina, n_act = 1_000_000, 111_000
    sc = synth.scene_c3(n=n_ina + n_act, n_views=n_views)
    dev = torch.device("cuda", torch.cuda.current_device())
    mask = synth.active_mask(sc, n_act / sc.n, "clustered")
    act = torch.from_numpy(np.flatnonzero(mask).astype(np.int32)).to(dev)
    ina = torch.from_numpy(np.flatnonzero(~mask).astype(np.int32)).to(dev)
    rows = torch.from_numpy(sc.rows).to(dev)
    sigma = torch.tensor([sc.sigma], dtype=torch.float32, device=dev)
    centers = torch.from_numpy(synth.camera_centers(sc.cams)).to(dev)
    S_max = max(1, int(round(max(rates) * n_views)))
    vd = torch.empty(S_max, dtype=torch.int32, device=dev)
    L.oit_select_views(centers, S_max, 2605, 1, vd)
    picked = [int(x) for x in vd.cpu().numpy()]          # FPS is greedy: the first S picks are FPS(S)
    from paper_2605_13855_b200.pipeline import ViewPipeline
    cam0 = sc.cams[0]
    big = ViewPipeline(cam0, max(n_ina, n_act), 1 << 24, device=dev)
    caches, targets = [None] * n_views, [None] * n_views
    gen = torch.Generator(device=dev)
    gen.manual_seed(4321)
    for j in picked:
        big.set_camera(sc.cams[j])
        _, st = big.forward(rows, sigma, ina, sc.bg, image=False)
        assert big.pairs_used() <= big.capacity
        caches[j] = st.clone()
        targets[j] = torch.randint(0, 256, (3, cam0["height"], cam0["width"]), generator=gen, device=dev,
                                   dtype=torch.uint8)
    # one training iteration of this scene: a view's a1-a6 over the active set (single stream)
    grad = torch.zeros((n_act, 80), dtype=torch.float32, device=dev)
    dsig = torch.zeros(1, dtype=torch.float32, device=dev)

    def one_iter():
        for j in picked[:4]:
            big.set_camera(sc.cams[j])
            _, st = big.forward(rows, sigma, act, sc.bg, base=caches[j], image=False)
            big.backward(rows, sigma, act, sc.bg, st, None, grad, dsig, target=targets[j], loss="l1")
    iter_ms = _graph_time(torch, one_iter, flush, args.warmup, args.steps) / 4
    del big
    torch.cuda.empty_cache()
    cap = 1 << 24
    n_str = 8
    streams = [torch.cuda.Stream() for _ in range(n_str)]
    ws = [torch.empty(L.oit_score_workspace_bytes(cam0, n_act, n_ina, cap), dtype=torch.uint8, device=dev)
          for _ in range(n_str)]
    sg = torch.zeros((n_ina, 80), dtype=torch.float32, device=dev)
    sds = torch.zeros(1, dtype=torch.float32, device=dev)
    mp = torch.zeros(1, dtype=torch.int64, device=dev)
    bits0 = torch.from_numpy(synth.bits_from_mask(mask).view(np.int32)).to(dev)
    bits = bits0.clone()
    n = sc.n
    act_out, fro, new = (torch.empty(n, dtype=torch.int32, device=dev) for _ in range(3))
    cnt = torch.zeros(3, dtype=torch.int32, device=dev)
    uws = torch.empty(L.oit_update_workspace_bytes(n), dtype=torch.uint8, device=dev)
    out = {"splats": sc.n, "n_inactive_scored": n_ina, "n_active": n_act, "views": n_views,
           "refresh_every": refresh_every, "iteration_ms": iter_ms, "sweep": {}}
    for rate in rates:
        S = max(1, int(round(rate * n_views)))
        views = picked[:S]

        def refresh():
            L.oit_select_views(centers, S, 2605, 1, vd)
            sg.zero_()
            sds.zero_()
            main = torch.cuda.current_stream()
            k_used = min(S, n_str)
            for k in range(k_used):
                part = views[k::k_used]
                streams[k].wait_stream(main)
                with torch.cuda.stream(streams[k]):
                    L.oit_score_subsample(rows, sigma, sc.cams, targets, caches, act, ina, part, "l1", sc.bg, sg, sds,
                                          cap, mp, ws[k], scale=1.0 / S, concurrency=k_used)
            for k in range(k_used):
                main.wait_stream(streams[k])
            bits.copy_(bits0)
            L.oit_update_active_set(sg, ina, [1e-7] * 6, "fresh", n, bits, act_out, cnt[0:1], fro, cnt[1:2], new,
                                    cnt[2:3], uws)
        ms = _graph_time(torch, refresh, flush, args.warmup, args.steps)
        assert int(mp.item()) <= cap, "score pair capacity overflow"
        out["sweep"][f"{rate:g}"] = {"S": S, "ms_per_refresh": ms, "amortized_ms_per_iteration": ms / refresh_every,
                                     "ratio_to_iteration": ms / refresh_every / iter_ms,
                                     "ms_per_scored_view": ms / S}
    return out


def time_ablation(args, torch, wl, flush, n_views=10):
    """NEXT-4 (Table 2 analogue): the a5 moment kernel of our lane = splat backward vs
    the 3DGS-style per-pixel backward (oit_composite_bwd_perpixel), same views, same dL/dC, one
    stream, event-timed around the moment kernel; L2 flushed before each view's backward."""
    L, dev = wl.L, wl.dev
    p = wl.pipe
    grad = torch.zeros_like(wl.grad)
    ds = torch.zeros(1, dtype=torch.float32, device=dev)
    g = torch.empty((3, wl.H, wl.W), dtype=torch.float32, device=dev)
    ev = [(torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))
          for _ in range(2)]
    for e in ev:
        e[0].record(); e[1].record()
    ms = {False: [], True: []}
    for rep in range(2):
        for v in range(min(n_views, wl.V)):
            p.set_camera(wl.cams[v])
            img, st = p.forward(wl.rows, wl.sigma, wl.act, wl.bg, base=wl.caches[v])
            L.oit_loss_grad(wl.cams[v], img, wl.target_f32(v), "l1", g)
            for k, per_pixel in enumerate((False, True)):
                flush.zero_()
                flush.sum()
                torch.cuda.synchronize()
                p.backward(wl.rows, wl.sigma, wl.act, wl.bg, st, g, grad, ds, events=ev[k], per_pixel=per_pixel)
                torch.cuda.synchronize()
                if rep > 0:
                    ms[per_pixel].append(event_ms(*ev[k]))
    ours, pix = float(np.mean(ms[False])), float(np.mean(ms[True]))
    return {"views": min(n_views, wl.V), "moments_ms_per_view_ours": ours, "moments_ms_per_view_per_pixel": pix,
            "speedup": pix / ours}


DSSIM_BYTES_PER_PX = 3 * (8 + 12 + 12 + 8 + 4)   # per pixel (3 channels): stats pass in/out, grad pass in/out


def time_dssim(args, torch, wl, flush):
    """NEXT-3: oit_loss_dssim (the 3DGS (1−λ)L1 + λ·D-SSIM loss and dL/dC) on one 800×800 view,
    event-timed after an L2 flush; HBM roofline on the stencil passes' algorithmic bytes."""
    L, dev = wl.L, wl.dev
    cam = wl.cams[0]
    img = wl.target_f32(1 % wl.V)
    tgt = wl.target_f32(0)
    g = torch.empty_like(tgt)
    loss = torch.zeros(1, dtype=torch.float32, device=dev)
    ws = torch.empty(L.oit_dssim_workspace_bytes(cam), dtype=torch.uint8, device=dev)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for rep in range(args.warmup + max(args.steps, 5)):
        flush.zero_()
        flush.sum()
        torch.cuda.synchronize()
        t0.record()
        L.oit_loss_dssim(cam, img, tgt, g, ws, 0.2, loss)
        t1.record()
        torch.cuda.synchronize()
        if rep >= args.warmup:
            times.append(t0.elapsed_time(t1))
    ms = float(np.mean(times))
    nbytes = wl.H * wl.W * DSSIM_BYTES_PER_PX
    gbs = nbytes / (ms * 1e-3) / 1e9
    return {"ms_per_view": ms, "res": [wl.W, wl.H], "bytes": nbytes, "loss": float(loss.item()),
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": HBM_PEAK_GBS, "unit": "GB/s",
                         "frac": gbs / HBM_PEAK_GBS, "peak_source": HBM_PEAK_SOURCE}}


ADAM_BYTES_PER_ROW = 4 * 320 + 4 * 320 + 4 + 4 + 4   # read g, ℓ, m, v; write ℓ, m, v, row; idx, step r/w


def time_adam(args, torch, wl, flush):
    """NEXT-2: one oit_adam_step over the step's compacted active gradient rows (n_A rows, state
    for all N splats), event-timed on its stream after an L2 flush; HBM roofline against the
    measured copy bandwidth (algorithmic bytes: grad/latent/m/v read, latent/m/v/rows written,
    index and step count)."""
    L, dev = wl.L, wl.dev
    g = torch.Generator(device=dev)
    g.manual_seed(77)
    lat = torch.randn((wl.n, 80), generator=g, device=dev) * 0.5
    m = torch.zeros_like(lat)
    v = torch.zeros_like(lat)
    step = torch.zeros(wl.n, dtype=torch.int32, device=dev)
    rows = torch.empty_like(lat)
    sig = torch.tensor([np.log(4.8), 0.0, 0.0, 0.0], dtype=torch.float32, device=dev)
    sig_out = torch.zeros(1, dtype=torch.float32, device=dev)
    cfg = L.adam_cfg()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for rep in range(args.warmup + max(args.steps, 5)):
        flush.zero_()
        flush.sum()          # read back: the flush's dirty lines are written back before timing
        torch.cuda.synchronize()
        t0.record()
        L.oit_adam_step(wl.grad, wl.act, lat, m, v, step, rows, cfg, dsigma=wl.dsig, sigma_state=sig, sigma=sig_out)
        t1.record()
        torch.cuda.synchronize()
        if rep >= args.warmup:
            times.append(t0.elapsed_time(t1))
    ms = float(np.mean(times))
    nbytes = wl.n_act * ADAM_BYTES_PER_ROW
    gbs = nbytes / (ms * 1e-3) / 1e9
    return {"ms": ms, "rows": wl.n_act, "bytes": nbytes,
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": HBM_PEAK_GBS, "unit": "GB/s",
                         "frac": gbs / HBM_PEAK_GBS, "peak_source": HBM_PEAK_SOURCE}}


def time_reconcile(args, torch, wl, flush):
    """NEXT-1 (§4.1 P:147 lazy pre-render): cost of bringing one view's cache to a new active set
    by the delta (oit_active_set_delta + oit_reconcile_cache: FOLD the newly frozen, UNFOLD the
    re-activated splats) versus re-rendering the new frozen set from scratch (a1-a3, no image).
    The synthetic change: 10 % of the active set frozen, 2 % of the frozen set re-activated
    (seeded). Summed over the V views on one stream; L2 flushed before each repetition."""
    from paper_2605_13855_b200 import synth
    from paper_2605_13855_b200.pipeline import ViewPipeline
    L, dev = wl.L, wl.dev
    mask0 = synth.mask_from_bits(wl.bits0.cpu().numpy().view(np.uint32), wl.n)
    g = np.random.default_rng(4242)
    m = mask0.copy()
    a, i = np.flatnonzero(mask0), np.flatnonzero(~mask0)
    m[a[g.random(len(a)) < 0.10]] = False
    m[i[g.random(len(i)) < 0.02]] = True
    bits_new = torch.from_numpy(synth.bits_from_mask(m).view(np.int32)).to(dev)
    ina_new = torch.from_numpy(np.flatnonzero(~m).astype(np.int32)).to(dev)
    fold = torch.empty(wl.n, dtype=torch.int32, device=dev)
    unfold = torch.empty(wl.n, dtype=torch.int32, device=dev)
    cnt = torch.zeros(2, dtype=torch.int32, device=dev)
    dws = torch.empty(L.oit_delta_workspace_bytes(wl.n), dtype=torch.uint8, device=dev)
    L.oit_active_set_delta(wl.bits0, bits_new, wl.n, fold, cnt[0:1], unfold, cnt[1:2], dws)
    nf, nu = (int(x) for x in cnt.cpu().numpy())
    cap = wl.score_cap
    rws = torch.empty(L.oit_reconcile_workspace_bytes(wl.cams[0], nf + nu, cap), dtype=torch.uint8, device=dev)
    npairs = torch.zeros(1, dtype=torch.int64, device=dev)
    scratch = torch.empty_like(wl.caches[0])
    pipe = ViewPipeline(wl.cams[0], wl.n, cap, device=dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(2 * wl.V)]
    rec_ms, rr_ms = [], []
    max_diff = 0.0
    for rep in range(args.warmup + args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        for v, cam in enumerate(wl.cams):
            scratch.copy_(wl.caches[v])
            ev[2 * v][0].record()
            L.oit_active_set_delta(wl.bits0, bits_new, wl.n, fold, cnt[0:1], unfold, cnt[1:2], dws)
            L.oit_reconcile_cache(wl.rows, wl.sigma, cam, fold[:nf], unfold[:nu], scratch, cap, npairs, rws)
            ev[2 * v][1].record()
            pipe.set_camera(cam)
            ev[2 * v + 1][0].record()
            _, st = pipe.forward(wl.rows, wl.sigma, ina_new, wl.bg, image=False)
            ev[2 * v + 1][1].record()
            if rep == 0 and v < 4:   # sanity (GPU vs GPU; parity is tests/test_gpu_parity.py)
                d = (scratch - st).abs() / (st.abs() + 1e-3)
                max_diff = max(max_diff, float(d.max()))
        torch.cuda.synchronize()
        if rep >= args.warmup:
            rec_ms.append(sum(event_ms(*ev[2 * v]) for v in range(wl.V)))
            rr_ms.append(sum(event_ms(*ev[2 * v + 1]) for v in range(wl.V)))
    assert npairs.item() <= cap and pipe.pairs_used() <= cap
    return dict(ms_per_view=float(np.mean(rec_ms)) / wl.V, rerender_ms_per_view=float(np.mean(rr_ms)) / wl.V,
                n_fold=nf, n_unfold=nu, n_frozen_new=int(ina_new.numel()), max_rel_diff_vs_rerender=max_diff,
                change="10% of the active set frozen, 2% of the frozen set re-activated (seeded)")


def time_e2e(args, torch, dist, wl, step, flush, allred):
    """Same step through the public API with HOST inputs: per step, pinned-host → device copies of
    every training image of the step (the step's input data; on a copy stream, in view order; each
    view waits only for its own image, so the copies overlap the compute of the earlier views), and
    device → host reads of the step's results, the combined gradient rows and the refreshed bitmask —
    all inside the timed region (one CUDA graph per step, copies included). The parameter rows are
    training state, resident on the device and updated there by the step's Adam (copying them in
    each step would overwrite that update); they, σ and the optimizer state are restored between
    steps outside the timed region, as in the device-timed step."""
    targets_h = wl.targets.cpu().pin_memory()
    grad_h = torch.empty_like(wl.grad, device="cpu").pin_memory()
    bits_h = torch.empty_like(wl.bits, device="cpu").pin_memory()
    h2d = targets_h.numel() * targets_h.element_size()
    d2h = grad_h.numel() * 4 + bits_h.numel() * 4
    host_views = [targets_h[v] for v in range(wl.V)]

    def e2e_step():
        wl.train_and_refresh(host_targets=host_views)
        if allred:
            return
        # the combined gradient rows are final here: read them back on the copy stream while the
        # Adam step and the update run (both only read them)
        main = torch.cuda.current_stream()
        wl.copy_stream.wait_stream(main)
        with torch.cuda.stream(wl.copy_stream):
            grad_h.copy_(wl.grad, non_blocking=True)
        wl.adam()
        wl.update()
        bits_h.copy_(wl.bits, non_blocking=True)
        main.wait_stream(wl.copy_stream)

    graph = None
    if not args.no_graph and not allred:
        e2e_step()
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=s):
                e2e_step()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for i in range(args.warmup + args.steps):
        wl.restore_params()
        flush.zero_()
        torch.cuda.synchronize()
        if allred:
            dist.barrier()
        t0.record()
        if graph is not None:
            graph.replay()
        elif allred:
            wl.targets.copy_(targets_h, non_blocking=True)
            step()
            grad_h.copy_(wl.grad, non_blocking=True)
            bits_h.copy_(wl.bits, non_blocking=True)
        else:
            e2e_step()
        t1.record()
        torch.cuda.synchronize()
        if i >= args.warmup:
            times.append(t0.elapsed_time(t1))
    wl.restore_params()
    ms = float(np.mean(times))
    if allred:
        t = torch.tensor([ms], dtype=torch.float64, device=wl.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return dict(ms=ms, h2d=h2d, d2h=d2h)


def _ncu_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from the newest committed
    ncu --set full capture summary (profiles/<round>_traffic.json, tools/traffic_json.py), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json")))
    if not files:
        return None, None
    try:
        d = json.load(open(files[-1]))[kernel]
        return d["dram_bytes_per_launch"], f"profiles/{os.path.basename(files[-1])} ({d['report']}, one C2 view)"
    except Exception:
        return None, None


def mpix_per_s(res, world):
    return world * res["V"] * res["H"] * res["W"] / (res["ms"] * 1e-3) / 1e6


def build_line(args, world, res, results):
    value = mpix_per_s(res, world)
    evals = world * 256 * res["pairs"]
    f_c = res["contrib"] / max(res["tile_evals"], 1)
    # roofline of the dominant kernel (fwd composite or bwd moments, both FP32-ALU bound), in the
    # FP32-instruction accounting of SURVEY §8(d)
    contrib, skipped = res["contrib"], res["tile_evals"] - res["contrib"]
    fwd_instr = contrib * FWD_I_CONTRIB + skipped * FWD_I_SKIP
    bwd_instr = contrib * BWD_I_CONTRIB + skipped * BWD_I_SKIP
    fwd_flops = res["tile_evals"] * FWD_F_TEST + contrib * FWD_F_CONTRIB
    bwd_flops = res["tile_evals"] * BWD_F_TEST + contrib * BWD_F_CONTRIB
    per_kernel = {}
    for name, instr, flops_, kms_ in (("k_fwd_items", fwd_instr, fwd_flops, res["ser_fwd_ms"]),
                                      ("k_moments", bwd_instr, bwd_flops, res["ser_bwd_ms"])):
        a = instr / (kms_ * 1e-3) / 1e12
        per_kernel[name] = {"algorithmic_instr_per_step": instr, "kernel_ms_per_step": kms_, "achieved": a,
                            "frac": a / FP32_PEAK_TINSTR, "flops_per_step": flops_,
                            "frac_flop_accounting": flops_ / (kms_ * 1e-3) / 1e12 / FP32_PEAK_TFLOPS}
    if res["ser_bwd_ms"] >= res["ser_fwd_ms"]:
        kern, tkey = "k_moments (oit_composite_bwd a5)", "k_moments"
        pk = per_kernel["k_moments"]
    else:
        kern = "k_fwd_items (oit_composite_fwd_loss a3+a4)"
        tkey = "k_fwd_items<1, 0, 2>" if args.targets == "u8" else "k_fwd_items<1, 0, 1>"
        pk = per_kernel["k_fwd_items"]
    traffic, traffic_src = _ncu_traffic(tkey)
    achieved = pk["achieved"]
    # step level: the whole timed step's tile-granular evaluations against the fwd+bwd FP32 ceiling
    # at the measured f_c (37.2e12 / (54·f_c + 19·(1 − f_c)) evaluations/s)
    fc = contrib / max(res["tile_evals"], 1)
    ceiling = FP32_PEAK_TINSTR * 1e12 / ((FWD_I_CONTRIB + BWD_I_CONTRIB) * fc + (FWD_I_SKIP + BWD_I_SKIP) * (1 - fc))
    step_evals_per_s = world * res["tile_evals"] / (res["ms"] * 1e-3)
    sweep = {}
    for rho, r in sorted(results.items(), reverse=True):
        sweep[str(rho)] = {"mpix_per_s": mpix_per_s(r, world), "ms_per_step": r["ms"],
                           "evals_per_s": world * 256 * r["pairs"] / (r["ms"] * 1e-3),
                           "fwd_kernel_ms": r["fwd_ms"], "bwd_moments_ms": r["bwd_ms"], "n_active": r["n_act"],
                           "train_and_refresh_ms": r["train_refresh_ms"], "adam_and_update_ms": r["adam_update_ms"],
                           "pairs_per_view": r["pairs"] / r["V"],
                           "f_c": r["contrib"] / max(r["tile_evals"], 1),
                           "f_c_tile_granular": r["contrib"] / max(256 * r["pairs"], 1)}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": res["ms"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded; paper_2605_13855_b200.synth)",
        "config": {"workload": WORKLOAD, "splats": args.splats, "views_per_gpu": res["V"], "res": [res["W"], res["H"]],
                   "rho": res["rho"], "mask": args.kind, "n_active": res["n_act"], "refresh_views_S": res["S"],
                   "step": "one batch of the rank's 100 training views against one parameter state (R28: "
                           "fwd+bwd each, gradients summed; a9 all-reduce at N>1) and, concurrently, the "
                           "period's refresh on the same parameters (R35: a7 FPS + score of the inactive set on "
                           "S views), then one masked Adam step and a8 (Eq. 8 update into a scratch bitmask); "
                           "parameters restored between timed steps",
                   "l2": "flushed between timed steps (256 MB write)", "graph": not args.no_graph,
                   "streams": args.streams, "loss": args.loss,
                   "targets": ("uint8 [3][H][W] 8-bit training images (OIT_TARGET_U8)" if args.targets == "u8"
                               else "fp32 [3][H][W]")},
        "splat_pixel_evals_per_s": evals / (res["ms"] * 1e-3),
        "contributing_fraction_f_c": f_c,
        "evaluated_splat_pixels_per_view": res["tile_evals"] / res["V"],
        "kernel_ms_per_step": {"fwd_composite": res["ser_fwd_ms"], "bwd_moments": res["ser_bwd_ms"],
                               "note": "sum over the step's training views, single-stream roofline pass; the timed "
                                       "step runs views on several streams concurrently",
                               "concurrent_fwd_composite": res["fwd_ms"], "concurrent_bwd_moments": res["bwd_ms"]},
        "segments_ms": {"train_views_and_refresh_overlapped": res["train_refresh_ms"],
                        "adam_and_update": res["adam_update_ms"], "refresh_alone": res.get("refresh_alone_ms")},
        "roofline": {"kernel": kern, "bound": "alu", "achieved": achieved, "peak": FP32_PEAK_TINSTR,
                     "unit": "T FP32 instr/s", "frac": achieved / FP32_PEAK_TINSTR, "traffic": traffic,
                     "algorithmic_instr_per_step": pk["algorithmic_instr_per_step"],
                     "kernel_ms_per_step": pk["kernel_ms_per_step"],
                     "instr_per_eval": {"fwd": [FWD_I_CONTRIB, FWD_I_SKIP], "bwd": [BWD_I_CONTRIB, BWD_I_SKIP],
                                        "note": "[contributing, skipped] FP32 instructions per tile-granular "
                                                "evaluation, SURVEY §8(d); evaluations and contributing pairs are "
                                                "counted on the GPU (oit_composite_fwd_ex counters)"},
                     "per_kernel": per_kernel,
                     "step": {"evals_per_s": step_evals_per_s, "ceiling_evals_per_s": ceiling,
                              "frac": step_evals_per_s / ceiling, "f_c": fc},
                     "timing": "the step's training views replayed on ONE stream (between L2 flushes), the kernel "
                               "with its full-GPU persistent grid (concurrency 1), CUDA events on the launching "
                               f"stream; the timed step launches it with concurrency = {args.streams} (smaller "
                               "grids, views sharing the SMs)",
                     "traffic_source": traffic_src,
                     "peak_source": "148 SMs x 128 FP32 lanes x 1965 MHz = 37.2 T instr/s (B200_PROFILING.md unit "
                                    "counts; MEASURED_PEAKS.json has no FP32 entry)"},
        "clocks": res["clocks"], "gpu_launches": res["launches"] * args.steps,
        "sweep": sweep,
    }
    if "ablation" in res:
        line["next4_bwd_ablation"] = res["ablation"]
    if "dssim" in res:
        line["next3_dssim"] = res["dssim"]
    if "adam" in res:
        line["next2_adam"] = res["adam"]
    if "reconcile" in res:
        line["next1_reconcile"] = res["reconcile"]
    if "e2e" in res:
        e = res["e2e"]
        line["e2e"] = {"value": world * res["V"] * res["H"] * res["W"] / (e["ms"] * 1e-3) / 1e6, "unit": UNIT,
                       "h2d_bytes_per_step": e["h2d"], "d2h_bytes_per_step": e["d2h"], "ms_per_step": e["ms"]}
    return line


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

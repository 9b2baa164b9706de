"""bench.py's JSON line keeps the driver contract (keys, units, derived values) — checked on CPU with
a synthetic measurement record (no GPU, no timing)."""
import sys

import pytest

import bench


def _res(ms=16.0, V=100, W=800, H=800):
    return dict(ms=ms, fwd_ms=20.0, bwd_ms=15.0, clocks={"sm_mhz": 1965.0, "sm_max_mhz": 1965, "reasons": []},
                ser_fwd_ms=7.7, ser_bwd_ms=7.0, pairs=28_500_000, contrib=2_110_000_000, tile_evals=7_300_000_000,
                V=V, H=H, W=W, n_act=60_000, n_ina=240_000, S=5, launches=1600, rho=0.2, max_score_pairs=1,
                train_refresh_ms=13.5, adam_update_ms=0.1,
                e2e=dict(ms=19.0, h2d=288_000_000, d2h=19_237_500))


def test_json_line_has_the_contract_keys(monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    args = bench.parse()
    assert args.gpus == 1 and args.warmup >= 3 and args.steps >= 1 and args.impl == "ours"
    res = _res()
    line = bench.build_line(args, 1, res, {0.2: res})
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "gpu_launches", "e2e"):
        assert k in line, k
    assert line["metric"] == bench.METRIC and line["unit"] == "Mpix/s" and line["higher_is_better"] is True
    assert line["value"] == pytest.approx(100 * 800 * 800 / 16e-3 / 1e6)
    assert line["config"]["workload"] == bench.WORKLOAD
    r = line["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert r["bound"] == "alu" and r["unit"] == "T FP32 instr/s"
    # the §8(d) accounting, recomputable from the line: instructions = contributing·18 + skipped·9
    # (fwd), contributing·36 + skipped·10 (bwd); the dominant kernel is the slower one
    c, sk = res["contrib"], res["tile_evals"] - res["contrib"]
    fwd = r["per_kernel"]["k_fwd_items"]
    assert fwd["algorithmic_instr_per_step"] == c * 18 + sk * 9
    assert fwd["frac"] == pytest.approx((c * 18 + sk * 9) / (res["ser_fwd_ms"] * 1e-3) / 37.2e12, rel=1e-3)
    assert r["per_kernel"]["k_moments"]["algorithmic_instr_per_step"] == c * 36 + sk * 10
    assert r["achieved"] == pytest.approx(fwd["achieved"])     # ser_fwd_ms > ser_bwd_ms here
    fc = c / res["tile_evals"]
    assert r["step"]["ceiling_evals_per_s"] == pytest.approx(37.2e12 / (54 * fc + 19 * (1 - fc)), rel=1e-3)
    assert r["step"]["frac"] == pytest.approx(res["tile_evals"] / 16e-3 / r["step"]["ceiling_evals_per_s"])
    e = line["e2e"]
    assert e["unit"] == "Mpix/s" and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["value"] == pytest.approx(100 * 800 * 800 / 19e-3 / 1e6)
    # whole-job aggregate: N ranks of weak-scaled work report N× the per-rank throughput
    line2 = bench.build_line(args, 2, res, {0.2: res})
    assert line2["value"] == pytest.approx(2 * line["value"]) and line2["n_gpus"] == 2


def test_scan_kernel_count_matches_the_launcher():
    assert bench.scan_kernels(0) == 0
    assert bench.scan_kernels(2500) == 1        # one block: k_scan_blocks writes the total
    assert bench.scan_kernels(4096) == 1
    assert bench.scan_kernels(4097) == 3        # blocks + sums + add

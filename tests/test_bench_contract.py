"""CPU checks of bench.py's pure helpers: the roofline arithmetic the BENCH line reports follows
SURVEY.md §8(d) (K5: 8 FP32 instr per examined pair + 11 per composited pair, against the FP32 lane
peak 148 SMs x 128 lanes x clock), and the per-stage HBM byte counts."""
import json
import os

import pytest

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# per-view device counters of a C3 view (profiles/r02f_bench.json, counts_per_view)
C3 = {"N": 1 << 20, "views": 64, "HW": 1920 * 1080, "ntiles": 120 * 68, "n_vis": 836424.9375,
      "K": 37017915.15625, "examined": 317678856.984375, "composited": 151112789.921875}
PEAKS = {"hbm_gbs": 6528.0, "source": "test", "sm_max_mhz": 1965.0}


def test_k5_work_is_the_survey_count():
    kind, work = bench.stage_work("raster_fwd", C3, 59)
    assert kind == "alu_fp32"
    assert work == 8 * C3["examined"] + 11 * C3["composited"]
    assert abs(work - 4.20e9) / 4.20e9 < 0.01          # 4.20e9 per C3 view


def test_roofline_frac_reproduces_by_hand():
    # one 64-view step whose K5 launches took 47.0 ms in total (one launch per view)
    r = bench.roofline("raster_fwd", C3, 59, 64, 47.0, 64, PEAKS, 148)
    t = 47.0e-3 / 64
    peak = 148 * 128 * 1965e6
    by_hand = (8 * C3["examined"] + 11 * C3["composited"]) / t / peak
    assert r["bound"] == "alu" and r["kernel"] == "raster_fwd"
    assert r["frac"] == pytest.approx(by_hand, rel=1e-12)
    assert r["peak"] == pytest.approx(peak / 1e12, rel=1e-12)
    assert r["avg_launch_ms"] == pytest.approx(47.0 / 64)
    # the same step as one launch of 64 views: the per-launch work scales, the rate does not
    r1 = bench.roofline("raster_fwd", C3, 59, 64, 47.0, 1, PEAKS, 148)
    assert r1["frac"] == pytest.approx(by_hand, rel=1e-12)


def test_hbm_stage_bytes():
    # K1: 44 B of geometry per texel once per call + SH (4 x 48 B) and a 56 B record per visible pair
    kind, b = bench.stage_work("project", C3, 59)
    assert kind == "hbm"
    assert b == pytest.approx(44 * C3["N"] / 64 + (4 * 48 + 56) * C3["n_vis"])
    # K10: image, target, dL (3 channels fp32) per pixel
    assert bench.stage_work("loss", C3, 59) == ("hbm", 12 * 3 * C3["HW"])
    r = bench.roofline("loss", C3, 59, 64, 1.0, 64, PEAKS, 148)
    assert r["frac"] == pytest.approx(12 * 3 * C3["HW"] * 64 / 1e-3 / 1e9 / PEAKS["hbm_gbs"])


def test_committed_bench_line_is_consistent():
    """The committed bench line's roofline is the §8(d) quantity of its own counters and timing."""
    p = os.path.join(ROOT, "profiles", "r02f_bench.json")
    d = json.loads(open(p).read().strip().splitlines()[-1])
    c = dict(C3, **d["counts_per_view"])
    r = d["roofline"]
    work = 8 * c["examined"] + 11 * c["composited"]
    assert r["frac"] == pytest.approx(work / (r["avg_launch_ms"] * 1e-3) / (r["peak"] * 1e12), rel=1e-9)
    assert d["value"] == pytest.approx(64 / (d["ms_per_step"] / 1e3), rel=1e-9)
    assert d["warmup"] >= 3 and d["n_gpus"] == 1 and d["clocks"]["reasons"] == []
    assert d["cpu_baseline"]["cores"] == d["cpu_baseline"]["nproc"]
    assert d["e2e"]["d2h_bytes_per_step"] >= 4 * (1 << 20) * 59   # the gradient planes come back

"""bench.py end to end on the GPU at a small size: the JSON line carries every key of the contract
(value / e2e / roofline / cpu_baseline / clocks / gpu_launches) with self-consistent numbers."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_json_line_c2():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "2", "--views", "4",
                          "--steps", "3", "--warmup", "3", "--cpu-sample-views", "1"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "clocks", "e2e", "gpu_launches", "roofline",
              "cpu_baseline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] == pytest.approx(4 / (d["ms_per_step"] / 1e3), rel=1e-6)
    assert d["gpu_launches"] > 0 and d["overflow"] is False
    r = d["roofline"]
    assert r["bound"] == "alu" and 0 < r["frac"] < 1 and r["kernel"] in ("raster_fwd", "raster_bwd")
    e = d["e2e"]
    assert 0 < e["value"] <= d["value"] * 1.05
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0
    assert set(d["counts_per_view"]) >= {"n_vis", "K", "examined", "composited"}

"""bench.py's one-JSON-line contract (the driver parses it): the reference arm on CPU,
our arm on a B200 at the small config."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.timeout(600)
def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "2", "--warmup", "0", "--cpu-scale", "16"], 560)
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "GTEPS" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["sample_scale"] == 16 and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
@pytest.mark.timeout(900)
def test_our_arm_line_k16():
    d = _run(["--config", "k16", "--steps", "1", "--warmup", "0"], 850)
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 0
    assert d["config"]["workload"].startswith("Graph500 Kronecker scale 16")
    rl = d["roofline"]
    assert rl["bound"] == "hbm" and rl["peak"] > 0 and abs(rl["frac"] - rl["achieved"] / rl["peak"]) < 1e-3
    assert d["gpu_launches"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert "sm_mhz" in d["clocks"]
    v = d["validation"]
    assert v["searches"] == 64 and v["failed_searches"] == 0 and v["rules"] == {}


def test_rank_memory_model_fits_the_multi_gpu_targets():
    """K29 fits one B200 (178 GB usable), K30 needs >= 2 ranks, and
    the 8-rank targets (K29, K30) fit with room for the construction peak."""
    import bench
    gb = 178.0
    assert bench.rank_memory(29, 16, 1, True)["build_peak_gb"] < gb
    assert bench.rank_memory(30, 16, 1, True)["steady_gb"] > gb
    for scale in (29, 30):
        m = bench.rank_memory(scale, 16, 8, True)
        assert m["build_peak_gb"] < gb / 3
    # per-rank bytes shrink with p
    ms = [bench.rank_memory(30, 16, p, True)["steady_gb"] for p in (2, 4, 8)]
    assert ms == sorted(ms, reverse=True)

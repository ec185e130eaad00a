"""bench.py contract pieces that run without a GPU: the reference arm (the reference CPU
executor from oracle/_ref timed on host cores) prints one well-formed JSON line, and the CPU
sample is valid for any host thread count (whole 16-row blocks per chunk)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.mark.parametrize("devices", [1, 3, 8, 16, 24, 64, 128, 192])
@pytest.mark.parametrize("want", [128, 512, 1000])
def test_sample_rows_are_whole_blocks_per_chunk(devices, want):
    import bench
    rows = bench.sample_rows(want, devices)
    assert rows % (16 * devices) == 0 and rows >= 16 * devices


def test_reference_arm_prints_one_json_line():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libmanta_ref.so")):
        pytest.skip("reference build (oracle/_ref) not present")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2", "--warmup", "1", "--cols", "2048"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "cell-updates/s"
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
def test_bench_line_schema_on_gpu():
    """a short N=1 bench run prints one JSON line with every key the driver reads"""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "10", "--warmup", "3", "--rows", "8192", "--cols", "8192",
                        "--matmul-n", "0", "--no-c4", "--no-c1", "--ooc-gib", "0", "--e2e-runs", "1", "--e2e-pipeline", "2", "--e2e-iters", "5",
                        "--cpu-rows", "128", "--cpu-iters", "2"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling", "vs_baseline", "dtype", "data",
              "config", "roofline", "cpu_baseline", "clocks", "e2e", "gpu_launches", "repeats"]:
        assert k in d, k
    assert d["steps"] == 10 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(d["roofline"])
    assert {"value", "unit", "cores", "kind", "sample"} <= set(d["cpu_baseline"])
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(d["e2e"])
    assert d["e2e"]["h2d_bytes_per_step"] == 8192 * 8192 * 4 and d["gpu_launches"] == 10
    assert "workload" in d["config"]

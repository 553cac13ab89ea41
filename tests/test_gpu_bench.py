"""bench.py's JSON contract (the driver parses this line): a small run on one GPU
prints one JSON line with every key the contract names, the HBM roofline object,
the CPU baseline, the e2e object and a positive launch count."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_line_has_the_contract_keys():
    d = _run("--steps", "3", "--warmup", "3", "--members", "64")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["dtype"] == "f64" and d["scaling"] == "weak" and "workload" in d["config"]
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    # dt_commit, then 2 stages + dt_commit per step; small ensembles (64 x 8 tiles,
    # <= 2 waves) fuse the dt into stage 1: 2 stages per step + one dt_commit
    assert d["gpu_launches"] in (1 + 3 * 3, 2 * 3 + 1)
    assert "sm_mhz" in d["clocks"]


@pytest.mark.parametrize("scheme", ["explicit", "sgn"])
def test_bench_scheme_variants_run(scheme):
    d = _run("--steps", "2", "--warmup", "3", "--members", "32", "--no-cpu", "--scheme", scheme)
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and 0 < d["roofline"]["frac"] < 1


def test_reference_arm_line():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "1", "--cells", "256")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["value"] == d["value"]

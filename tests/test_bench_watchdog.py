"""bench.py host logic (no GPU): the watchdog of the multi-rank sub-records.  If
the sub-records do not finish in time (a rank stuck in a collective of the cfg5
NCCL slab leg), rank 0 prints the headline line as it stands -- exactly one
JSON line -- and every rank exits 0; if they do finish, the watchdog stays
silent."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(code):
    return subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=120)


def test_watchdog_fires_and_prints_one_line():
    r = _run("import time, bench\n"
             "bench.SUB_TIMEOUT_S = 0.05\n"
             "bench._watchdog({'metric': 'm', 'value': 1.0}, {'done_leg': {'v': 2}}, 0)\n"
             "time.sleep(30)\nprint('NOT REACHED')\n")
    assert r.returncode == 0, r.stderr
    lines = [x for x in r.stdout.splitlines() if x.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["metric"] == "m" and d["value"] == 1.0
    assert d["sub_records"]["done_leg"] == {"v": 2}
    assert "timed out" in d["sub_records"]["cfg5"]["error"]


def test_watchdog_other_ranks_exit_silently():
    r = _run("import time, bench\n"
             "bench.SUB_TIMEOUT_S = 0.05\n"
             "bench._watchdog({'metric': 'm'}, {}, 1)\n"
             "time.sleep(30)\nprint('NOT REACHED')\n")
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_watchdog_silent_when_done():
    r = _run("import time, bench\n"
             "bench.SUB_TIMEOUT_S = 0.2\n"
             "d = bench._watchdog({'metric': 'm'}, {}, 0)\n"
             "d.set()\ntime.sleep(0.6)\nprint('reached')\n")
    assert r.returncode == 0 and r.stdout.strip() == "reached"


def test_profile_summary_feeds_roofline_traffic():
    """bench.py takes roofline.traffic from the committed ncu launch lists
    (profiles/ncu_summary.json): cfg3's stage 2 and cfg5's bathymetry stage 2,
    both at their algorithmic bytes (96 / 104 B per cell) to within 5 %."""
    sys.path.insert(0, ROOT)
    import bench
    t3 = bench.profile_traffic(1 << 24)
    t5 = bench.profile_traffic(1 << 28, bathy=True)
    assert t3 is not None and t5 is not None
    assert 0.95 * 96 <= t3 / (1 << 24) <= 1.05 * 96
    assert 0.95 * 104 <= t5 / (1 << 28) <= 1.05 * 104
    f = bench.profile_fp64()
    assert f is not None and 0.0 < f["frac"] < 1.0

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

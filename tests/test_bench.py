"""CPU tests of bench.py's host logic: the --gpus N self-launch (N ranks over
gloo, whole-job aggregation, n_gpus = N) and the reference arm's isolation
(it times the oracle only and never maps the product library)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _last_json(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


@pytest.mark.parametrize("n", [1, 2, 3])
def test_gpus_flag_spawns_ranks(n):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", str(n), "--dry-run", "--steps", "2", "--rows", "10"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert d["dry_run"] and d["n_gpus"] == n
    assert d["ms_per_step"] == float(n)            # max over ranks of (1 + rank)
    assert d["value"] == pytest.approx(10 * n * 2 / (n * 2 / 1e3))  # whole-job rows / max time


def test_reference_arm_is_oracle_only():
    code = ("import runpy, sys\n"
            "sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0', '--rows', '8']\n"
            "runpy.run_path('bench.py', run_name='__main__')\n"
            "maps = open('/proc/self/maps').read()\n"
            "print('LIBPAM', 'libpam' in maps, 'PKG', any(m.startswith('paper_2509_08383_b200') for m in sys.modules),"
            " 'ORACLE', 'liboracle' in maps)\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert d["impl"] == "reference" and d["config"]["n"] == 151936 and d["cpu_baseline"]["kind"] == "port"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["value"] > 0
    assert "LIBPAM False PKG False ORACLE True" in r.stdout

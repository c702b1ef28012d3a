"""CPU checks of bench.py's plumbing: the --gpus N self-launch (torchrun
ranks over gloo, one JSON line, max over ranks) and the reference arm (the
unmodified reference from baseline/_ref on the host; libmcf never loaded)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import REPO

BENCH = os.path.join(REPO, "bench.py")


def _json_lines(out: str):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def test_gpus_2_launches_two_ranks():
    res = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--dry-run"], cwd=REPO,
                         capture_output=True, text=True, timeout=300,
                         env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    assert res.returncode == 0, res.stderr[-2000:]
    lines = _json_lines(res.stdout)
    assert len(lines) == 1, res.stdout
    assert lines[0]["n_gpus"] == 2 and lines[0]["ranks_seen"] == 2 and lines[0]["max_rank"] == 1


PROBE = r"""
import runpy, sys
sys.argv = ["bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3",
            "--ref-scale", "0.002"]
runpy.run_path("bench.py", run_name="__main__")
maps = open("/proc/self/maps").read()
print("LIBMCF_LOADED" if "libmcf.so" in maps else "LIBMCF_ABSENT")
"""


def test_reference_arm_runs_the_reference_without_libmcf():
    if not os.path.isdir(os.path.join(REPO, "baseline", "_ref", "multicf")):
        pytest.skip("baseline/_ref (the reference install) absent")
    res = subprocess.run([sys.executable, "-c", PROBE], cwd=REPO, capture_output=True,
                         text=True, timeout=600, env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    assert res.returncode == 0, res.stderr[-2000:]
    assert "LIBMCF_ABSENT" in res.stdout
    (line,) = _json_lines(res.stdout)
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "reference"
    assert line["config"]["workload"] == "cfg1-als-full" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["gpu_launches"] == 0
    assert line["solve_only"]["value"] > 0

"""CPU: bench.py's reference arm (the contract's `--impl reference`) times the
reference's own CPU path (oracle/_ref, the unmodified reference sources) and
prints the contract's JSON line, without ever mapping the product library
(the arm must not load libqapb200.so)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT
from oracle.pyoracle import available

WRAP = r"""
import atexit, runpy, sys
def maps():
    with open("/proc/self/maps") as fh:
        hit = any("libqapb200" in line for line in fh)
    sys.stderr.write("LIBQAPB200_MAPPED=%d\n" % hit)
atexit.register(maps)
sys.argv = ["bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1", "--size", "12"]
runpy.run_path("bench.py", run_name="__main__")
"""


@pytest.mark.skipif(not available("ref"), reason="oracle/_ref not built")
def test_reference_arm_contract_and_isolation():
    r = subprocess.run([sys.executable, "-c", WRAP], cwd=ROOT, capture_output=True, text=True,
                       timeout=600, env=dict(os.environ, CUDA_VISIBLE_DEVICES=""))
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    assert d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "iterations/s" and d["higher_is_better"] is True
    for k in ("metric", "n_gpus", "steps", "warmup", "ms_per_step", "config", "dtype"):
        assert k in d, k
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["sample"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "LIBQAPB200_MAPPED=0" in r.stderr

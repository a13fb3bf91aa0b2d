"""CPU: the reference's OWN instance tests (proj/tests/test_instance.cpp: QAPLIB parse
round trips, swap order, manifest + solution cross-checks, generator determinism),
compiled unmodified against the facade (include/qap/instance.hpp + libqapb200.so) by
`make -C oracle reftests`.  Host code only, so it runs without a GPU."""
import os
import subprocess

import pytest

from conftest import ROOT
from test_gpu_reference_suite import _write_fixtures

EXE = os.path.join(ROOT, "build", "reftests", "test_instance_b200")


def test_reference_instance_tests_pass(tmp_path):
    if not os.path.exists(EXE):
        pytest.skip(f"{EXE} not built (needs /root/reference at build time)")
    _write_fixtures(str(tmp_path))
    env = dict(os.environ, QAPB_FIXTURE_DIR=str(tmp_path))
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=600, env=env,
                         cwd=str(tmp_path))
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-4000:]
    assert "| 0 failed" in out.stdout

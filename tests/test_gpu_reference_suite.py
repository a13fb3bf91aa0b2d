"""GPU: the reference's OWN unit tests (proj/tests/test_lap.cpp, test_rlt2.cpp,
and test_bnb.cpp with the reference's branch-and-bound proj/src/bnb.cpp bounding
its nodes through the facade), compiled unmodified against the B200 facade
headers (include/qap/*.hpp) + libqapb200.so by `make -C oracle reftests`, must pass.
The binaries are built where /root/reference exists and travel in-tree
(build/reftests); fixtures are regenerated from tests/golden/golden.json."""
import json
import os
import subprocess

import pytest

from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu
BIN = os.path.join(ROOT, "build", "reftests")


def _write_fixtures(dirpath):
    """proj/fixtures/* as captured by tests/golden/make_fixtures.py."""
    with open(os.path.join(GOLDEN, "fixtures.json")) as fh:
        files = json.load(fh)
    for name, text in files.items():
        with open(os.path.join(dirpath, name), "w") as fh:
            fh.write(text)


@pytest.mark.parametrize("name", ["test_lap_b200", "test_rlt2_b200", "test_bnb_b200"])
def test_reference_unit_tests_pass_on_b200(name, tmp_path):
    exe = os.path.join(BIN, name)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    _write_fixtures(str(tmp_path))
    env = dict(os.environ, QAPB_FIXTURE_DIR=str(tmp_path))
    out = subprocess.run([exe], capture_output=True, text=True, timeout=1200, env=env)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-4000:]
    assert "| 0 failed" in out.stdout


def test_reference_bnb_banks_spread_over_gpus(tmp_path):
    """Bank-per-GPU placement (QAPB_BANK_GPUS, facade.cpp bank_device): the
    reference's own branch-and-bound tests, unmodified, with its bank threads
    spread over two GPUs, still pass, and engines land on both devices."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    exe = os.path.join(BIN, "test_bnb_b200")
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    _write_fixtures(str(tmp_path))
    env = dict(os.environ, QAPB_FIXTURE_DIR=str(tmp_path), QAPB_BANK_GPUS="2",
               QAPB_BANK_GPUS_VERBOSE="1")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=1200, env=env)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-4000:]
    assert "| 0 failed" in out.stdout
    assert "placed on device 0 of 2" in out.stderr
    assert "placed on device 1 of 2" in out.stderr

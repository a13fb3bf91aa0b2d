"""Shared test fixtures.  `-m gpu` tests need a B200; everything else runs on CPU."""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def lap_cases():
    z = np.load(os.path.join(GOLDEN, "lap_cases.npz"))
    out, oc, on = [], 0, 0
    for k, m in enumerate(z["m"]):
        m = int(m)
        out.append(dict(m=m, cost=z["costs"][oc:oc + m * m].reshape(m, m), value=z["values"][k],
                        r2c=z["r2c"][on:on + m], u=z["u"][on:on + m], v=z["v"][on:on + m]))
        oc += m * m
        on += m
    return out


def hexs(xs):
    return [float.fromhex(x) for x in xs]


def golden_instance(golden, name):
    from paper_1710_03732_b200.instance import QapInstance
    g = golden[name]
    return QapInstance(g["n"], np.array(g["flow"], float), np.array(g["dist"], float), None, name)


def digest(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()[:32]

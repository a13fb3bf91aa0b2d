"""GPU parity over long horizons for the BASELINE.json configs (VERDICT r01
"parity horizons"): every per-iteration bound bitwise against the compiled
reference's trace (tests/golden/long_traces.json, made by
tests/golden/make_long_traces.py from oracle/_ref), and sha256 digests of
every engine array at the last iteration.

  grid20_*  nug20-shaped (4x5 Manhattan grid, flows U{0..10} seed 1; config 5's
            instance): F1/S1 x 100 (SURVEY §8c pins 4306.229804554644 and
            4305.930423138996), F2/S2 x 30
  rand20_*  tai20a-shaped generate_instance(20,1,99) (config 2): all variants x 30
  grid30_*, rand30_*  nug30-shaped (config 3, the bench workload) and tai30-shaped:
            F1/S1 x 20, F2/S2 x 8
  grid42_*  sko42-shaped 6x7 grid (config 4): S1 and F1 x 3 (iteration 1 = 26996)
"""
import json
import os

import pytest

from conftest import digest, hexs

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "long_traces.json")) as fh:
    LONG = json.load(fh)["traces"]


@pytest.fixture(scope="module")
def q():
    import paper_1710_03732_b200 as q
    return q


def _instance(q, key):
    shape = key.split("_")[0]
    grids = {"grid20": (4, 5), "grid30": (5, 6), "grid42": (6, 7)}
    if shape in grids:
        return q.instance.grid_instance(*grids[shape])
    return q.generate_instance(int(shape[4:]), 1, 99)


@pytest.mark.parametrize("key", sorted(LONG))
def test_long_trace_bitwise(q, key):
    tr = LONG[key]
    inst = _instance(q, key)
    eng = q.AscentEngine.from_instance(
        inst, q.AscentConfig(variant=tr["variant"], iter_limit=tr["iters"], record_history=False))
    want = hexs(tr["bounds"])
    for it in range(1, tr["iters"] + 1):
        got = eng.iterate()
        assert got == want[it - 1], (key, it, got, want[it - 1])
    assert eng.best_bound() == float.fromhex(tr["best"])
    for it, snap in tr.get("digests", {}).items():
        assert int(it) == tr["iters"]
        for a in ("pi_z", "pi_y", "pi_x", "b", "c", "d", "theta", "delta"):
            assert digest(eng.array(a)) == snap[a], (key, a)
        if "incz" in snap:
            assert digest(eng.incz()) == snap["incz"], (key, "incz")
        assert eng.x_assignment() == snap["x_assignment"], key
    eng.close()


def test_sko42_shaped_iteration1(q):
    """the sko42-shaped instance's Gilmore-Lawler bound is 26996."""
    eng = q.AscentEngine.from_instance(q.instance.grid_instance(6, 7),
                                       q.AscentConfig(variant="S1", iter_limit=1))
    assert eng.iterate() == 26996.0
    eng.close()

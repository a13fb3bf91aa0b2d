"""GPU parity: the warp-per-LAP Hungarian vs the reference LapSolver (lap.cpp:24-84).
Bit-exact: optimum, assignment and both dual vectors."""
import numpy as np
import pytest

from conftest import golden_instance
from oracle.pyoracle import Oracle, available, best_oracle
from paper_1710_03732_b200.abi import default_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    import paper_1710_03732_b200 as q
    return q


def test_golden_lap_cases_bitwise(q, lap_cases):
    by_m = {}
    for k, c in enumerate(lap_cases):
        by_m.setdefault(c["m"], []).append(k)
    for m, ks in by_m.items():
        b = q.solve_batch(q.LapBatch.from_costs(np.stack([lap_cases[k]["cost"] for k in ks])))
        for s, k in enumerate(ks):
            c = lap_cases[k]
            assert b.values[s] == c["value"], (m, k)
            assert (b.row_to_col[s] == c["r2c"]).all(), (m, k)
            assert (b.u[s] == c["u"]).all() and (b.v[s] == c["v"]).all(), (m, k)
            assert (b.col_to_row[s][b.row_to_col[s]] == np.arange(m)).all()


def test_trivial_and_ties(q):
    """test_lap.cpp:52-67."""
    assert q.solve_lap([5.0], 1).value == 5.0
    r = q.solve_lap(np.array([1.0, 2, 3, 0]), 2)
    assert r.value == 1.0 and list(r.row_to_col) == [0, 1]
    r = q.solve_lap(np.full(16, 3.0), 4)
    assert list(r.row_to_col) == [0, 1, 2, 3]
    with pytest.raises(ValueError):
        q.solve_lap(np.zeros(5), 2)


def test_shift_invariance_and_slots(q):
    """test_lap.cpp:82-98, 135-145."""
    rng = np.random.default_rng(7)
    m = 6
    cost = rng.integers(0, 50, (m, m)).astype(float)
    base = q.solve_lap(cost)
    sh = cost + (np.arange(m)[:, None] * 1.5 + np.arange(m)[None, :] * 0.25)
    r = q.solve_lap(sh)
    assert abs(r.value - (base.value + sum(i * 1.75 for i in range(m)))) < 1e-9
    assert (r.row_to_col == base.row_to_col).all()
    b = q.LapBatch().resize(2, 2)
    b.costs[0] = [[1, 2], [3, 0]]
    b.costs[1] = [[0, 9], [9, 0]]
    q.solve_batch(b, 2)
    assert list(b.values) == [1.0, 0.0]


def test_dual_feasibility_random(q):
    """Invariants of test_lap.cpp:27-49 on larger sizes (all CPL variants)."""
    rng = np.random.default_rng(3)
    for m in (5, 28, 31, 40, 64, 96, 127):
        costs = rng.integers(-20, 80, (16, m, m)).astype(float)
        b = q.solve_batch(q.LapBatch.from_costs(costs))
        for s in range(16):
            c, r, u, v = costs[s], b.row_to_col[s], b.u[s], b.v[s]
            assert sorted(r) == list(range(m))
            red = c - u[:, None] - v[None, :]
            assert red.min() >= -1e-9
            assert abs(red[np.arange(m), r]).max() <= 1e-9
            assert abs(c[np.arange(m), r].sum() - b.values[s]) < 1e-6


def test_z_tiles_of_an_ascent_bitwise(q, golden):
    """Every Z tile of nug12 S1 after 20 iterations (the costs the engine solves)
    and every F1 incz tile after 7 iterations, against the reference solver."""
    orc = best_oracle()
    inst = golden_instance(golden, "nug12")
    for variant, iters, arr in (("S1", 20, "d"), ("F1", 7, "incz")):
        eng = orc.engine_from_instance(inst.flow, inst.dist,
                                       cfg=default_config(variant=variant, iter_limit=iters))
        for _ in range(iters):
            eng.iterate()
        # the costs iteration `iters` solved: S -> the store's D', F -> incz
        tiles = eng.array(arr).reshape(-1, 10, 10)
        want = orc.lap_solve_batch(tiles)
        got = q.solve_batch(q.LapBatch.from_costs(tiles))
        assert (got.values == want[0]).all()
        assert (got.row_to_col == want[1]).all()
        assert (got.u == want[3]).all() and (got.v == want[4]).all()


def test_device_pointer_api(q):
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(9)
    costs = rng.normal(size=(1000, 28, 28))
    dc = torch.tensor(costs, device="cuda")
    vals = torch.empty(1000, dtype=torch.float64, device="cuda")
    q.solve_batch_device(dc.data_ptr(), 28, 1000, vals.data_ptr(),
                         stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = q.solve_batch(q.LapBatch.from_costs(costs)).values
    assert (vals.cpu().numpy() == ref).all()


def test_special_costs_and_large_m_bitwise(q):
    """+inf, huge (|c| > 1e300), NaN and -0.0 costs (the exact safe path) and
    m > 127 (the CTA-per-LAP path) against the reference LapSolver
    (tests/golden/make_lap_special.py): optimum, assignment, both duals."""
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "lap_special.npz"))
    oc = on = 0
    for k, m in enumerate(z["m"]):
        m = int(m)
        cost = z["costs"][oc:oc + m * m].reshape(m, m)
        r2c, u, v = z["r2c"][on:on + m], z["u"][on:on + m], z["v"][on:on + m]
        oc += m * m
        on += m
        for count in (1, 3):  # a lone slot and a batch of identical slots
            b = q.solve_batch(q.LapBatch.from_costs(np.stack([cost] * count)))
            for s in range(count):
                assert b.values[s].tobytes() == np.float64(z["values"][k]).tobytes(), (k, m)
                assert (b.row_to_col[s] == r2c).all(), (k, m)
                assert b.u[s].tobytes() == u.tobytes() and b.v[s].tobytes() == v.tobytes(), (k, m)


def test_undefined_lap_raises(q):
    """A row with no finite cost: LapSolver::solve reads p[-1] (lap.cpp:53,
    undefined behaviour); the drop-in reports it instead of inventing a result."""
    inf = np.inf
    with pytest.raises(ValueError):
        q.solve_lap(np.array([[inf, inf], [1.0, 2.0]]))
    with pytest.raises(ValueError):  # the CTA-per-LAP path too
        c = np.ones((130, 130))
        c[5, :] = inf
        q.solve_lap(c)
    # the solver stays usable afterwards
    assert q.solve_lap(np.array([[1.0, 2.0], [3.0, 0.0]])).value == 1.0

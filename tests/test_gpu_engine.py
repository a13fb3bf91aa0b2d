"""GPU parity: the device-resident AscentEngine vs the reference (golden traces
from the compiled reference, and the oracle library itself when present).
The bar is bitwise: every per-iteration bound and every engine array."""
import math

import numpy as np
import pytest

from conftest import digest, golden_instance, hexs
from oracle.pyoracle import Oracle, available, best_oracle
from paper_1710_03732_b200 import abi
from paper_1710_03732_b200.abi import default_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    import paper_1710_03732_b200 as q
    return q


def _inst(q, golden, key):
    tr = golden["traces"][key]
    if key.startswith("nug12"):
        return golden_instance(golden, "nug12")
    if key.startswith("rand20"):
        return q.generate_instance(20, 1, 99)
    if key.startswith("grid20"):
        return q.instance.grid_instance(4, 5)
    n = int(key[4:key.index("_")])
    return q.generate_instance(n, 100 + (n - 5) // 2, 99)


@pytest.mark.parametrize("key", ["nug12_F1", "nug12_S1", "nug12_F2", "nug12_S2",
                                 "nug12_F1_SA", "nug12_F2_SA", "nug12_S1_SA", "rand20_F1",
                                 "rand20_S1", "rand20_F2", "grid20_F1", "rand7_S2",
                                 "rand7_F1_SA", "rand9_S2", "rand9_F1_SA", "rand11_S2",
                                 "rand11_F1_SA"])
def test_trace_bitwise(q, golden, key):
    tr = golden["traces"][key]
    inst = _inst(q, golden, key)
    cfg = q.AscentConfig(variant=tr["variant"], iter_limit=tr["iters"], sa_enabled=tr["sa"],
                         upper_bound=tr["upper_bound"], seed=tr["seed"])
    eng = q.AscentEngine.from_instance(inst, cfg)
    want = hexs(tr["bounds"])
    for it in range(1, tr["iters"] + 1):
        got = eng.iterate()
        assert got == want[it - 1], (key, it, got, want[it - 1])
        snap = tr["digests"].get(str(it))
        if snap:
            for a in ("pi_z", "pi_y", "pi_x", "b", "c", "d", "theta", "delta"):
                assert digest(eng.array(a)) == snap[a], (key, it, a)
            if "incz" in snap:
                assert digest(eng.incz()) == snap["incz"], (key, it, "incz")
            assert eng.x_assignment() == snap["x_assignment"]
    assert eng.best_bound() == max(want)
    eng.close()


# Fold kernel variants (kernels.cu launch_zfold): chunk 2 at n even selects the
# warp-specialised fold; the environment switches select the others.
FOLD_VARIANTS = {
    "ws": {},
    "ws_stages2": {"QAPB_FOLD_WS_STAGES": "2"},
    "ws_chunk1": {"QAPB_FOLD_CHUNK": "1"},
    "pipe": {"QAPB_FOLD_WS": "0"},
    "pipe_chunk1": {"QAPB_FOLD_CHUNK": "1", "QAPB_FOLD_WS": "0"},
    "pipe_k1": {"QAPB_FOLD_PIPE_K": "1"},
    "pipe_blocked_order": {"QAPB_FOLD_ORDER_BLOCK": "3"},
    "bulk": {"QAPB_FOLD_PIPE": "0"},
    "lean": {"QAPB_FOLD_PIPE": "0", "QAPB_FOLD_BULK": "0"},
    "family": {"QAPB_FOLD_PIPE": "0", "QAPB_FOLD_BULK": "0", "QAPB_FOLD_LEAN": "0"},
}


@pytest.mark.parametrize("fold", sorted(FOLD_VARIANTS))
@pytest.mark.parametrize("key", ["nug12_F1", "nug12_S1", "rand20_F1", "nug12_F1_SA", "nug12_F2",
                                 "nug12_S2", "nug12_F2_SA"])
def test_fold_variants_bitwise(q, golden, key, fold, monkeypatch):
    monkeypatch.setenv("QAPB_FOLD_CHUNK", "2")  # n even, chunk 2: the pipelined fold
    for k, v in FOLD_VARIANTS[fold].items():
        monkeypatch.setenv(k, v)
    tr = golden["traces"][key]
    inst = _inst(q, golden, key)
    cfg = q.AscentConfig(variant=tr["variant"], iter_limit=tr["iters"], sa_enabled=tr["sa"],
                         upper_bound=tr["upper_bound"], seed=tr["seed"])
    eng = q.AscentEngine.from_instance(inst, cfg)
    want = hexs(tr["bounds"])
    for it in range(1, tr["iters"] + 1):
        assert eng.iterate() == want[it - 1], (key, fold, it)
        snap = tr["digests"].get(str(it))
        if snap:
            for a in ("pi_z", "d"):
                assert digest(eng.array(a)) == snap[a], (key, fold, it, a)
            if "incz" in snap:
                assert digest(eng.incz()) == snap["incz"], (key, fold, it, "incz")
    eng.close()


@pytest.mark.parametrize("variant", ["F1", "S1", "F2", "S2"])
def test_run_report_matches_oracle(q, golden, variant):
    orc = best_oracle()
    inst = golden_instance(golden, "nug12")
    for kw in (dict(iter_limit=30), dict(iter_limit=200, early_stop_window=5,
                                         early_stop_delta=0.002),
               dict(iter_limit=50, upper_bound=578.0, min_gap=0.05),
               dict(iter_limit=50, fathom_threshold=540.0)):
        cfg = q.AscentConfig(variant=variant, **kw)
        rep = q.run_ascent(inst, cfg)
        orep, orecs, _ = orc.engine_from_instance(inst.flow, inst.dist,
                                                  cfg=default_config(variant=variant, **kw)).run()
        assert rep.iterations == orep.iterations, kw
        assert rep.termination == q.abi.TERM_NAMES[orep.termination], kw
        assert rep.best_bound == orep.best_bound
        assert [r.bound for r in rep.records] == [r.bound for r in orecs]
        g = [r.gap for r in rep.records]
        og = [r.gap for r in orecs]
        assert all((a == b) or (math.isinf(a) and math.isinf(b)) for a, b in zip(g, og))


def test_zero_instance_feasible(q, golden):
    """test_rlt2.cpp:279-286."""
    rep = q.run_ascent(golden_instance(golden, "zero"), q.AscentConfig(iter_limit=10))
    assert rep.termination == "feasible-found"
    assert rep.best_bound == 0 and rep.certificate_value == 0 and rep.certificate


def test_feasibility_certificate(q):
    """test_rlt2.cpp:288-300: tiny flows, strong linear preference."""
    inst = q.generate_instance(5, 1)
    inst.flow[:] = 0
    inst.linear[:] = 50
    np.fill_diagonal(inst.linear, 0)
    rep = q.run_ascent(inst, q.AscentConfig(variant="S1", iter_limit=20))
    assert rep.termination == "feasible-found"
    assert rep.certificate == [0, 1, 2, 3, 4]
    assert rep.certificate_value == q.evaluate_objective(inst, rep.certificate) == 0.0


def test_snapshot_rules_and_warm_start(q):
    """test_rlt2.cpp:357-376."""
    inst = q.generate_instance(5, 3)
    eng = q.AscentEngine(q.init_coefficients(inst), q.AscentConfig(variant="F1", iter_limit=5))
    eng.iterate()
    with pytest.raises(q.engine.LogicError):
        eng.snapshot()
    inst = q.generate_instance(7, 2718)
    eng = q.AscentEngine(q.init_coefficients(inst), q.AscentConfig(variant="S1", iter_limit=30))
    for _ in range(30):
        eng.iterate()
    parent = eng.best_bound()
    snap = eng.snapshot()
    st = eng.store()
    assert (snap.d == st.d).all() and (snap.b == st.b).all()
    rep = q.run_ascent_warm(snap, q.AscentConfig(variant="S1", iter_limit=30))
    assert rep.records[0].bound >= parent - 1e-7
    assert all(b.bound >= a.bound - 1e-7 for a, b in zip(rep.records, rep.records[1:]))


def test_s_store_is_exact_reformulation(q):
    """test_rlt2.cpp:153-174 on the device store."""
    inst = q.generate_instance(6, 31)
    rng = np.random.default_rng(5)
    perms = [rng.permutation(6) for _ in range(10)]
    for v in ("S1", "S2"):
        eng = q.AscentEngine(q.init_coefficients(inst), q.AscentConfig(variant=v, iter_limit=1))
        for _ in range(25):
            eng.iterate()
            st = eng.store()
            for p in perms:
                assert abs(q.store_evaluate(st, p) - q.evaluate_objective(inst, p)) <= \
                    1e-9 * abs(q.evaluate_objective(inst, p))


def test_store_engine_equals_instance_engine(q):
    inst = q.generate_instance(9, 77)
    inst.linear[:] = np.arange(81).reshape(9, 9) % 7
    st = q.init_coefficients(inst)
    orc = best_oracle()
    b, c, d = orc.init_coefficients(inst.flow, inst.dist, inst.linear)
    assert (st.b == b).all() and (st.c == c).all() and (st.d == d).all()
    e1 = q.AscentEngine(st, q.AscentConfig(variant="S2", iter_limit=10))
    e2 = q.AscentEngine.from_instance(inst, q.AscentConfig(variant="S2", iter_limit=10))
    assert [r.bound for r in e1.run().records] == [r.bound for r in e2.run().records]


def test_iterate_continues_after_run_and_n3(q):
    inst = q.generate_instance(3, 5)
    orc = best_oracle()
    for v in ("F1", "S2"):
        eng = q.AscentEngine.from_instance(inst, q.AscentConfig(variant=v, iter_limit=4))
        oe = orc.engine_from_instance(inst.flow, inst.dist,
                                      cfg=default_config(variant=v, iter_limit=4))
        rep, orep = eng.run(), oe.run()
        assert [r.bound for r in rep.records] == [r.bound for r in orep[1]]
        for _ in range(3):
            assert eng.iterate() == oe.iterate()
        assert eng.iteration() == 7 or rep.termination == "feasible-found"


def test_errors(q):
    with pytest.raises(ValueError):
        q.init_coefficients(q.generate_instance(2, 1))
    with pytest.raises(ValueError):
        q.AscentEngine(q.CoefficientStore(2, np.zeros(4), np.zeros(4), np.zeros(0)))


def test_launch_accounting(q, golden):
    inst = golden_instance(golden, "nug12")
    eng = q.AscentEngine.from_instance(inst, q.AscentConfig(iter_limit=10))
    n0 = eng.launch_count()
    eng.run()
    assert eng.launch_count() - n0 >= 10 * 4


def test_n30_n42_reference_pins(q):
    """Large sizes.  n=30: bitwise against the compiled reference (oracle/_ref) for 4
    iterations of generate_instance(30,1,99) F1 and S1 when it is present.  n=42 (the
    sko42 size: 2.37 G z cells, the CPL=2 LAP path for m=40): generate_instance(42,1,99) S1
    iterations 1-2 against the reference values printed in SURVEY.md §8c (16 significant
    digits, so compared to 1e-15 relative; a reference run there takes ~1 min/iteration)."""
    inst30 = q.generate_instance(30, 1, 99)
    for variant in ("F1", "S1"):
        eng = q.AscentEngine.from_instance(inst30, q.AscentConfig(variant=variant, iter_limit=4))
        got = [eng.iterate() for _ in range(4)]
        eng.close()
        if available("ref"):
            cfg = default_config()
            cfg.variant = abi.VARIANTS[variant]
            cfg.iter_limit = 4
            ref = Oracle("ref").engine_from_instance(inst30.flow, inst30.dist, None, cfg)
            want = [ref.iterate() for _ in range(4)]
            assert got == want, (variant, got, want)
        else:
            want4 = {"F1": 1538557.650137826, "S1": 1538728.316958316}[variant]
            assert got[0] == 1473912.0 and math.isclose(got[3], want4, rel_tol=1e-15)
    eng = q.AscentEngine.from_instance(q.generate_instance(42, 1, 99),
                                       q.AscentConfig(variant="S1", iter_limit=2))
    got = [eng.iterate() for _ in range(2)]
    eng.close()
    assert got[0] == 3146129.0
    assert math.isclose(got[1], 3184361.336432928, rel_tol=1e-15), got

"""Device-resident stores: collapse_store on the B200 against the
reference's collapse_store (oracle/_ref, else the host restatement that
tests/test_abi.py pins to it), and the B&B node flow of bnb.cpp:317-387 run
device-to-device against the same flow through host stores.  Bitwise."""
import ctypes

import numpy as np
import pytest

from oracle.pyoracle import Oracle, available
from paper_1710_03732_b200 import abi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    import paper_1710_03732_b200 as q
    return q


def _random_store(q, m, seed):
    rng = np.random.default_rng(seed)
    nb, nc, nd = abi.store_sizes(m)
    b, c, d = rng.normal(size=nb), rng.normal(size=nc), rng.normal(size=nd)
    d[rng.random(nd) < 0.3] = 0.0
    d[rng.random(nd) < 0.05] = -0.0
    c[rng.random(nc) < 0.05] = -0.0
    return q.CoefficientStore(m, b, c, d, 1.25)


def _ref_collapse(q, st, fac, loc):
    if not available("ref"):
        return q.collapse_store(st, fac, loc)
    ref = Oracle("ref")
    nb, nc, nd = abi.store_sizes(st.m - 1)
    ob, oc, od = np.empty(nb), np.empty(nc), np.empty(max(nd, 0))
    off = ctypes.c_double()
    rc = ref.lib.qref_collapse_store(st.m, abi.dptr(st.b), abi.dptr(st.c), abi.dptr(st.d),
                                     st.offset, fac, loc, abi.dptr(ob), abi.dptr(oc),
                                     abi.dptr(od), ctypes.byref(off))
    assert rc == 0
    return q.CoefficientStore(st.m - 1, ob, oc, od, off.value)


def _same(a, b):
    assert a.m == b.m
    assert a.b.tobytes() == b.b.tobytes()
    assert a.c.tobytes() == b.c.tobytes()
    if a.m >= 3:
        assert a.d.tobytes() == b.d.tobytes()
    assert a.offset == b.offset


@pytest.mark.parametrize("m,fac,loc", [(5, 0, 4), (7, 3, 1), (7, 6, 0), (9, 4, 8), (12, 0, 0),
                                       (12, 11, 5)])
def test_device_collapse_bitwise(q, m, fac, loc):
    st = _random_store(q, m, 100 + m + fac)
    ds = q.DeviceStore.upload(st)
    child = ds.collapse(fac, loc)
    _same(child.download(), _ref_collapse(q, st, fac, loc))
    # a second level (grandchild) from the device-resident child
    g = child.collapse((fac + 1) % (m - 1), loc % (m - 1)).download()
    _same(g, _ref_collapse(q, _ref_collapse(q, st, fac, loc), (fac + 1) % (m - 1), loc % (m - 1)))


def test_device_collapse_after_ascent_n20(q):
    """A real S1 snapshot at n=20 (rlt2 store after 5 iterations) folded on the device."""
    inst = q.generate_instance(20, 1, 99)
    eng = q.AscentEngine.from_instance(inst, q.AscentConfig(variant="S1", iter_limit=5))
    for _ in range(5):
        eng.iterate()
    host = eng.snapshot()
    ds = q.DeviceStore.from_engine(eng)
    _same(ds.download(), host)
    for fac, loc in [(0, 19), (7, 3), (19, 0)]:
        _same(ds.collapse(fac, loc).download(), _ref_collapse(q, host, fac, loc))
    eng.close()


def test_node_flow_device_vs_host(q, golden):
    """bnb.cpp:317-387: parent S1 run -> snapshot -> collapse -> child engine run, all on
    the device, equals the same flow through host stores iteration by iteration."""
    from conftest import golden_instance
    inst = golden_instance(golden, "nug12")
    cfg = q.AscentConfig(variant="S1", iter_limit=15)
    parent = q.AscentEngine.from_instance(inst, cfg)
    for _ in range(15):
        parent.iterate()
    snap_dev = q.DeviceStore.from_engine(parent)
    snap_host = parent.snapshot()
    for fac, loc in [(0, 0), (5, 9), (11, 2)]:
        child_dev = q.AscentEngine.from_device_store(snap_dev.collapse(fac, loc),
                                                     q.AscentConfig(variant="S1", iter_limit=10))
        child_host = q.AscentEngine(q.collapse_store(snap_host, fac, loc),
                                    q.AscentConfig(variant="S1", iter_limit=10))
        for _ in range(10):
            assert child_dev.iterate() == child_host.iterate()
        rd, rh = child_dev.run(), child_host.run()
        assert rd.best_bound == rh.best_bound
        child_dev.close()
        child_host.close()
    parent.close()


def test_snapshot_rules(q, golden):
    from conftest import golden_instance
    inst = golden_instance(golden, "nug12")
    eng = q.AscentEngine.from_instance(inst, q.AscentConfig(variant="F1", iter_limit=3))
    eng.iterate()
    from paper_1710_03732_b200.engine import LogicError
    with pytest.raises(LogicError):  # rlt2.cpp:538-540: F variants do not snapshot
        q.DeviceStore.from_engine(eng)
    eng.close()
    st = _random_store(q, 3, 1)
    with pytest.raises(ValueError):  # rlt2.cpp:111: std::invalid_argument, store too small
        q.DeviceStore.upload(q.CoefficientStore(2, st.b[:4], st.c[:4], None, 0.0)).collapse(0, 0)

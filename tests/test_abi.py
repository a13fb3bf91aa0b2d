"""CPU: the C-ABI library loads, exports every declared entry point, and its
host-side helpers follow the reference (no GPU compute here)."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden_instance
from oracle.pyoracle import Oracle, available
from paper_1710_03732_b200 import abi

HEADER = os.path.join(ROOT, "include", "qapb200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"QAPB_API[^;(]*?\b(qapb_\w+)\s*\(", text, re.S)))


def test_library_exports_every_declared_symbol():
    import paper_1710_03732_b200 as q
    syms = declared_symbols()
    assert len(syms) >= 30
    lib = ctypes.CDLL(q.library_path)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_config_defaults_match_reference():
    """AscentConfig defaults, rlt2.hpp:98-121, through qapb_config_init."""
    import paper_1710_03732_b200 as q
    c = abi.Config()
    q.lib.qapb_config_init(ctypes.byref(c))
    d = abi.default_config()
    for name, _ in abi.Config._fields_:
        assert getattr(c, name) == getattr(d, name), name
    assert c.kappa_z_upper == 2.0 / 3.0 and math.isinf(c.upper_bound)
    assert q.AscentConfig().to_c().iter_limit == 100


def test_variant_names_and_parse():
    import paper_1710_03732_b200 as q
    assert [q.variant_name(v) for v in range(4)] == ["F1", "F2", "S1", "S2"]
    assert q.parse_variant("s2") == abi.S2
    with pytest.raises(ValueError):
        q.parse_variant("X9")


@pytest.mark.gpu
def test_redistribute_family_known_answers():
    """test_rlt2.cpp:207-247 (the device rule of the phase-2 kernel, store.cu)."""
    from paper_1710_03732_b200 import redistribute_family as rf
    ok, add = rf([10.0, 0.0, 0.0])
    assert ok and list(add) == [-10.0, 2.0, 2.0]
    ok, add = rf([0.0, 0.0, 0.0])
    assert ok and list(add) == [0.0, 0.0, 0.0]
    ok, add = rf([3.0, 6.0, 9.0])
    assert ok and list(add) == [-3.0, -6.0, -9.0]
    ok, add = rf([3.0, 6.0, 9.0], 0)
    assert not ok
    ok, add = rf([4.0, 0.0, 8.0])
    assert ok and list(add) == [-4.0, 3.0, -8.0]
    ok, add = rf([5.0, 1e-10, 0.0])
    assert ok and list(add) == [-5.0, 1.0, 1.0]


@pytest.mark.gpu
@pytest.mark.skipif(not available("port"), reason="oracle port not built")
def test_store_helpers_exact():
    """store_evaluate / collapse_store exactness (test_rlt2.cpp:94-107, 313-355), both
    on the device (store.cu)."""
    import itertools
    from paper_1710_03732_b200 import CoefficientStore, collapse_store, store_evaluate
    from paper_1710_03732_b200.instance import evaluate_objective, generate_instance
    port = Oracle("port")
    inst = generate_instance(6, 321)
    inst.linear[:] = np.arange(36).reshape(6, 6) % 5
    b, c, d = port.init_coefficients(inst.flow, inst.dist, inst.linear)
    st = CoefficientStore(6, b, c, d, 0.0)
    for perm in itertools.islice(itertools.permutations(range(6)), 0, 720, 7):
        assert abs(store_evaluate(st, perm) - evaluate_objective(inst, perm)) < 1e-9
    fac, loc = 2, 4
    child = collapse_store(st, fac, loc)
    assert child.m == 5
    ff = [i for i in range(6) if i != fac]
    fl = [p for p in range(6) if p != loc]
    for cp in itertools.permutations(range(5)):
        full = [0] * 6
        full[fac] = loc
        for i in range(5):
            full[ff[i]] = fl[cp[i]]
        assert abs(store_evaluate(child, cp) - evaluate_objective(inst, full)) < 1e-9


@pytest.mark.gpu
@pytest.mark.skipif(not available("ref"), reason="reference build absent")
def test_store_evaluate_bitwise_vs_reference():
    """store_evaluate (rlt2.cpp:91-107) on the device, summed in the reference's order."""
    from paper_1710_03732_b200 import CoefficientStore, store_evaluate
    ref = Oracle("ref")
    rng = np.random.default_rng(11)
    for m in (3, 5, 8):
        nb, nc, nd = abi.store_sizes(m)
        b, c, d = rng.normal(size=nb), rng.normal(size=nc), rng.normal(size=nd)
        st = CoefficientStore(m, b, c, d, 0.25)
        for _ in range(20):
            perm = rng.permutation(m).astype(np.int32)
            want = ctypes.c_double()
            assert ref.lib.qref_store_evaluate(m, abi.dptr(b), abi.dptr(c), abi.dptr(d), 0.25,
                                               abi.iptr(perm), ctypes.byref(want)) == 0
            assert store_evaluate(st, list(perm)) == want.value


@pytest.mark.gpu
@pytest.mark.skipif(not available("ref"), reason="reference build absent")
def test_collapse_store_bitwise_vs_reference():
    from paper_1710_03732_b200 import CoefficientStore, collapse_store
    ref = Oracle("ref")
    rng = np.random.default_rng(5)
    m = 7
    nb, nc, nd = abi.store_sizes(m)
    b, c, d = rng.normal(size=nb), rng.normal(size=nc), rng.normal(size=nd)
    d[rng.random(nd) < 0.3] = 0.0
    st = CoefficientStore(m, b, c, d, 1.5)
    out = collapse_store(st, 3, 1)
    ob, oc, od = np.empty(abi.store_sizes(6)[0]), np.empty(abi.store_sizes(6)[1]), \
        np.empty(abi.store_sizes(6)[2])
    off = ctypes.c_double()
    rc = ref.lib.qref_collapse_store(m, abi.dptr(b), abi.dptr(c), abi.dptr(d), 1.5, 3, 1,
                                     abi.dptr(ob), abi.dptr(oc), abi.dptr(od), ctypes.byref(off))
    assert rc == 0
    assert (out.b == ob).all() and (out.c == oc).all() and (out.d == od).all()
    assert out.offset == off.value


def test_instance_io(golden):
    from paper_1710_03732_b200.instance import parse_qaplib, evaluate_objective
    g = golden["nug12"]
    text = "12\n\n" + "\n".join(" ".join(str(x) for x in r) for r in g["flow"]) + "\n\n" + \
        "\n".join(" ".join(str(x) for x in r) for r in g["dist"])
    inst = parse_qaplib(text)
    assert inst.n == 12 and (inst.flow == np.array(g["flow"])).all()
    two = golden_instance(golden, "two")
    assert evaluate_objective(two, [0, 1]) == 6.0
    with pytest.raises(RuntimeError):
        parse_qaplib("3 1 2")

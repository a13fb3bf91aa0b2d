"""BoundReport::to_json byte-identical to the reference's (rlt2.cpp:604-630, nlohmann
dump(2)) -- SURVEY.md §8f #2.  CPU only: both sides are host formatting code."""
import ctypes as C
import json
import re

import numpy as np
import pytest

from oracle.pyoracle import Oracle, available
from paper_1710_03732_b200 import abi, lib


def _call(fn, instance, variant, sa, best, ub, gap, term, iters, wall, cert, cval, recs):
    buf = C.create_string_buffer(1 << 20)
    ln = C.c_size_t()
    cert_arr = (C.c_int * len(cert))(*cert) if cert else None
    r = np.ascontiguousarray(np.asarray(recs, np.float64).reshape(-1))
    fn.restype = C.c_int
    rc = fn(instance.encode(), variant.encode(), int(sa), C.c_double(best), C.c_double(ub),
            C.c_double(gap), term.encode(), int(iters), C.c_double(wall), cert_arr, len(cert),
            C.c_double(cval), abi.dptr(r) if len(recs) else None, len(recs), buf,
            C.c_size_t(len(buf)), C.byref(ln))
    assert rc == 0
    return buf.value.decode()


def _cases():
    rng = np.random.default_rng(7)
    inf = float("inf")
    yield ("nug12", "F1", False, 567.33680882290673, inf, inf, "iteration-limit", 3, 12.5, [],
           0.0, [[1, 493.0, -1.0, 0.5, 0.1, 0.01], [2, 503.23863636363637, inf, 1e-5, 0.0, 2.5e-7],
                 [3, 514.90710227272723, 0.1234, 123456789012345.0, 1234567890123456.0, -0.0]])
    yield ("two\"q\\\n", "S2", True, 6.0, 6.0, 0.0, "feasible-found", 1, 0.25, [1, 0], 6.0, [])
    vals = np.concatenate([rng.normal(size=40) * 10.0 ** rng.integers(-12, 18, size=40),
                           rng.integers(-10 ** 6, 10 ** 6, size=20).astype(float),
                           [1e-4, 1e-5, 9.999e-5, 1e15, 1e16, 123456789012345678.0, 0.1, 1 / 3,
                            2.0 ** -1074, 1.7976931348623157e308, -2.5e-300, 5e-324]])
    recs = [[k, vals[k % len(vals)], vals[(k * 7) % len(vals)], vals[(k * 3) % len(vals)],
             vals[(k * 5) % len(vals)], vals[(k * 11) % len(vals)]] for k in range(len(vals))]
    many = rng.standard_normal(6 * 3000) * 10.0 ** rng.uniform(-30, 30, size=6 * 3000)
    yield ("many", "S1", False, 1.0, 2.0, 0.5, "gap-closed", 3000, 1.5, [], 0.0,
           [[k] + list(many[6 * k + 1:6 * k + 6]) for k in range(3000)])
    yield ("rand", "F2", True, float(vals[0]), float(vals[1]), float(vals[2]), "early-stop",
           len(recs), float(vals[3]), list(range(12)), float(vals[4]), recs)


def _stock_int_arrays(text):
    """The reference vendors nlohmann/json in proj/vendor/, which is absent here; the oracle
    build takes the container's copy (cudnn_frontend/thirdparty, nlohmann 3.11.3) whose
    serializer was patched to print integer arrays on one line ("Custom from FE" in its
    dump()).  Stock nlohmann dump(2) prints every non-empty array one element per line;
    undo the patch on the oracle's text so the comparison is against stock behaviour."""
    def expand(m):
        ind = m.group(1)
        items = m.group(3).split(",")
        inner = ",\n".join(ind + "  " + x for x in items)
        return f'{ind}{m.group(2)}[\n{inner}\n{ind}]'
    return re.sub(r'(?m)^( *)("[^"]*": )\[(-?\d+(?:,-?\d+)*)\]', expand, text)


@pytest.mark.skipif(not available("ref"), reason="reference build absent")
@pytest.mark.parametrize("case", list(_cases()), ids=["nug12", "tiny", "many", "random"])
def test_report_json_byte_identical(case):
    ref = Oracle("ref")
    ours = _call(lib.qapb_report_json, *case)
    theirs = _stock_int_arrays(_call(ref.lib.qref_report_json, *case))
    assert ours == theirs
    json.loads(ours.replace("-0.0", "0.0"))  # well-formed

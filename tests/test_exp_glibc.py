"""CPU: the SA acceptance test's exp (rlt2.cpp:494 std::exp) restated from
glibc (csrc/glibc_exp.cuh) is bitwise the host libm's, for the build the
host's IFUNC picks and for the other one (GLIBC_TUNABLES masks FMA/AVX2 in a
subprocess).  The device side is tests/test_gpu_exp.py."""
import ctypes as C
import os
import re
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

SPECIAL = [0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, np.nan, 2.0**-54, -2.0**-54, 2.0**-55,
           -2.0**-53, 512.0, -512.0, 511.999, 1024.0, -1024.0, 709.78, 709.79, -708.39,
           -708.4, -744.4, -745.13, -745.14, -746.0, 5e-324, -5e-324, 1e300, -1e300,
           *(float.fromhex(h) for h in ("-0x1.bafef5135235bp+0", "-0x1.6063d1ae7a948p+3",
                                         "-0x1.84fd45030fefdp+4"))]


def arguments(n, seed):
    """The SA domain (-kap/T <= 0, rlt2.cpp:493-494), the full range and raw bits."""
    rng = np.random.default_rng(seed)
    raw = rng.integers(0, 2**63, n, dtype=np.int64).view(np.float64)
    raw = np.where(rng.random(n) < 0.5, raw, -raw)
    return np.concatenate([-rng.random(n) * 40.0, -rng.random(n) * 800.0,
                           (rng.random(n) - 0.5) * 1500.0, -rng.random(n) * 1e-3, raw,
                           np.array(SPECIAL)])


def _lib():
    import paper_1710_03732_b200 as q
    lib = C.CDLL(q.library_path)
    lib.qapb_exp_glibc.argtypes = [C.c_double, C.c_int]
    lib.qapb_exp_glibc.restype = C.c_double
    lib.qapb_exp_variant.restype = C.c_int
    return lib


def _libm_exp(x):
    from oracle.pyoracle import _load
    orc = _load("port")
    orc.orc_exp_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    orc.orc_exp_batch(x.ctypes.data, y.ctypes.data, x.size)
    return y


def same_bits(a, b):
    return (a.view(np.int64) == b.view(np.int64)) | (np.isnan(a) & np.isnan(b))


def check(variant, n, seed):
    lib = _lib()
    x = arguments(n, seed)
    want = _libm_exp(x)
    got = np.array([lib.qapb_exp_glibc(float(v), variant) for v in x])
    bad = ~same_bits(got, want)
    return int(bad.sum()), x[bad][:5]


def test_exp_table_is_the_generated_one():
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import gen_exp_table
    text = open(os.path.join(ROOT, "paper_1710_03732_b200", "csrc", "exp_table.h")).read()
    vals = [int(h, 16) for h in re.findall(r"0x([0-9a-f]{16})ULL", text)]
    assert vals == gen_exp_table.table()


def test_host_libm_build_detected_and_bitwise():
    lib = _lib()
    v = lib.qapb_exp_variant()
    assert v in (0, 1), "host libm is not glibc >= 2.28"
    nbad, ex = check(v, 60000, 1)
    assert nbad == 0, ex


def test_builds_differ_somewhere():
    """Both restatements are needed: they round differently at these x."""
    lib = _lib()
    x = float.fromhex("-0x1.bafef5135235bp+0")
    assert lib.qapb_exp_glibc(x, 1) != lib.qapb_exp_glibc(x, 0)


@pytest.mark.skipif(not os.path.exists("/proc/cpuinfo") or
                    " fma " not in open("/proc/cpuinfo").read(), reason="no FMA on this host")
def test_other_build_via_tunables():
    """Mask FMA/AVX2 so glibc's IFUNC picks the SSE2 build; the restatement of
    that build must then be detected and bitwise too."""
    code = ("import sys; sys.path[:0]=[%r, %r]\n"
            "import test_exp_glibc as t\n"
            "assert t._lib().qapb_exp_variant() == 0\n"
            "nbad, ex = t.check(0, 30000, 2)\n"
            "assert nbad == 0, ex\n") % (ROOT, os.path.join(ROOT, "tests"))
    env = dict(os.environ, GLIBC_TUNABLES="glibc.cpu.hwcaps=-AVX2,-FMA")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]


def test_variant_override(monkeypatch):
    code = ("import sys; sys.path[:0]=[%r, %r]\n"
            "import test_exp_glibc as t\n"
            "print(t._lib().qapb_exp_variant())\n") % (ROOT, os.path.join(ROOT, "tests"))
    for val, want in (("fma", "1"), ("nofma", "0")):
        env = dict(os.environ, QAPB_EXP_VARIANT=val)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                           text=True, timeout=300)
        assert r.stdout.strip().splitlines()[-1] == want, r.stderr[-2000:]

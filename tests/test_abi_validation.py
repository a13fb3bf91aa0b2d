"""CPU: the C-ABI rejects bad arguments with the reference's error class
(QAPB_EINVAL <-> std::invalid_argument) before touching a device, so these run
without a GPU.  References: rlt2.cpp:209 (m >= 3), lap.cpp:26 (m > 0),
rlt2.cpp:34-42 (parse_variant), rlt2.cpp:111 (collapse_store)."""
import ctypes as C

import pytest

EINVAL = 1


@pytest.fixture(scope="module")
def lib():
    import paper_1710_03732_b200 as q
    lib = C.CDLL(q.library_path)
    lib.qapb_last_error.restype = C.c_char_p
    lib.qapb_engine_create.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                                       C.c_void_p, C.c_void_p]
    lib.qapb_store_collapse_offset.argtypes = [C.c_void_p, C.c_double, C.c_int, C.c_int,
                                               C.c_void_p]
    return lib


def test_engine_rejects_small_problems(lib):
    assert lib.qapb_engine_create(2, None, None, None, 0.0, None, None) == EINVAL
    assert b"m >= 3" in lib.qapb_last_error()
    assert lib.qapb_engine_create_instance(2, None, None, None, None, None) == EINVAL
    assert b"n >= 3" in lib.qapb_last_error()


def test_lap_rejects_bad_sizes(lib):
    assert lib.qapb_lap_solve(None, 0, None, None, None, None, None) == EINVAL
    assert lib.qapb_lap_solve_batch(None, 0, 1, None, None, None, None, None) == EINVAL
    assert lib.qapb_lap_solve_batch(None, 3, -1, None, None, None, None, None) == EINVAL


def test_variant_and_store_arguments(lib):
    v = C.c_int()
    assert lib.qapb_parse_variant(b"X9", C.byref(v)) == EINVAL
    assert lib.qapb_store_collapse_offset(None, 0.0, 0, 0, None) == EINVAL

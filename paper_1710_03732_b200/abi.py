"""ctypes mirrors of the C-ABI structs in include/qapb200.h.

Plain data only: no library is loaded here, so both the product bindings
(paper_1710_03732_b200.engine) and the test-only oracle bindings share the
struct layouts without depending on each other.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

F1, F2, S1, S2 = 0, 1, 2, 3
VARIANTS = {"F1": F1, "F2": F2, "S1": S1, "S2": S2}
VARIANT_NAMES = {v: k for k, v in VARIANTS.items()}

TERM_NAMES = {0: "iteration-limit", 1: "gap-closed", 2: "feasible-found", 3: "early-stop"}

ARR = {"pi_z": 0, "pi_y": 1, "pi_x": 2, "b": 3, "c": 4, "d": 5, "theta": 6, "delta": 7,
       "incz": 8}


class Config(C.Structure):
    """qapb_config == qap::AscentConfig (rlt2.hpp:98-121)."""
    _fields_ = [
        ("variant", C.c_int),
        ("sa_enabled", C.c_int),
        ("iter_limit", C.c_int),
        ("min_gap", C.c_double),
        ("kappa_z_upper", C.c_double),
        ("phi_split", C.c_double),
        ("kappa_y", C.c_double),
        ("kappa_x", C.c_double),
        ("varphi", C.c_double),
        ("sa_t0_fraction", C.c_double),
        ("sa_kappa_lb_cap", C.c_double),
        ("sa_cool_factor", C.c_double),
        ("sa_cool_period", C.c_int),
        ("workers", C.c_int),
        ("seed", C.c_uint64),
        ("upper_bound", C.c_double),
        ("fathom_threshold", C.c_double),
        ("early_stop_window", C.c_int),
        ("early_stop_delta", C.c_double),
        ("record_history", C.c_int),
        ("device", C.c_int),
    ]


class Record(C.Structure):
    """qapb_record == qap::IterationRecord (rlt2.hpp:123-128)."""
    _fields_ = [("iteration", C.c_int), ("bound", C.c_double), ("gap", C.c_double),
                ("z_ms", C.c_double), ("y_ms", C.c_double), ("x_ms", C.c_double)]


class Report(C.Structure):
    """qapb_report == scalar part of qap::BoundReport (rlt2.hpp:130-146)."""
    _fields_ = [("best_bound", C.c_double), ("upper_bound", C.c_double), ("gap", C.c_double),
                ("termination", C.c_int), ("iterations", C.c_int),
                ("has_certificate", C.c_int), ("certificate_value", C.c_double),
                ("wall_ms", C.c_double), ("n_records", C.c_int)]


def default_config(**kw) -> Config:
    """AscentConfig defaults, rlt2.hpp:98-121."""
    c = Config(variant=F1, sa_enabled=0, iter_limit=100, min_gap=0.0,
               kappa_z_upper=2.0 / 3.0, phi_split=0.5, kappa_y=1.0, kappa_x=1.0, varphi=0.5,
               sa_t0_fraction=0.04, sa_kappa_lb_cap=0.25, sa_cool_factor=0.99,
               sa_cool_period=100, workers=1, seed=0, upper_bound=math.inf,
               fathom_threshold=math.inf, early_stop_window=0, early_stop_delta=0.0002,
               record_history=1, device=0)
    for k, v in kw.items():
        if k == "variant" and isinstance(v, str):
            v = VARIANTS[v.upper()]
        if isinstance(v, bool):
            v = int(v)
        setattr(c, k, v)
    return c


def store_sizes(m: int):
    """(len b, len c, len d) for a size-m store (StoreIndex, rlt2.hpp:25-69)."""
    tiles = (m * (m - 1) // 2) * (m * (m - 1))
    return m * m, m * m * (m - 1) * (m - 1), tiles * (m - 2) * (m - 2)


def dptr(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


def iptr(a):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)

"""ctypes binding of libqapb200.so with the reference's class/function names.

Every call goes through the C-ABI in include/qapb200.h; the status codes are
turned back into the exception types the reference throws
(std::invalid_argument -> ValueError, std::logic_error -> LogicError,
std::runtime_error -> RuntimeError).  No CPU fallback exists: if the CUDA
library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field, fields
from typing import List, Optional

import numpy as np

from .abi import (ARR, TERM_NAMES, VARIANT_NAMES, VARIANTS, Config, Record, Report,
                  default_config, dptr, iptr, store_sizes)
from .instance import QapInstance, evaluate_objective

HERE = os.path.dirname(os.path.abspath(__file__))
library_path = os.path.join(HERE, "libqapb200.so")

if not os.path.exists(library_path):
    raise ImportError(
        f"{library_path} is not built: run `make -C {HERE}` or "
        "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")

lib = C.CDLL(library_path)
_vp = C.c_void_p
_P = C.POINTER
lib.qapb_last_error.restype = C.c_char_p
lib.qapb_variant_name.restype = C.c_char_p
lib.qapb_lap_solve_batch.argtypes = [_vp, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp]
lib.qapb_lap_solve_batch_device.argtypes = [_vp, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp, _vp]
lib.qapb_init_coefficients.argtypes = [C.c_int, _vp, _vp, _vp, _vp, _vp, _vp]
lib.qapb_store_evaluate.argtypes = [C.c_int, _vp, _vp, _vp, C.c_double, _vp, _P(C.c_double)]
lib.qapb_collapse_store.argtypes = [C.c_int, _vp, _vp, _vp, C.c_double, C.c_int, C.c_int,
                                    _vp, _vp, _vp, _P(C.c_double)]
lib.qapb_redistribute_family.argtypes = [_vp, _vp, C.c_int, C.c_double, _P(C.c_int)]
lib.qapb_engine_create.argtypes = [C.c_int, _vp, _vp, _vp, C.c_double, _P(Config), _P(_vp)]
lib.qapb_engine_create_instance.argtypes = [C.c_int, _vp, _vp, _vp, _P(Config), _P(_vp)]
lib.qapb_engine_destroy.argtypes = [_vp]
lib.qapb_engine_iterate.argtypes = [_vp, _P(C.c_double)]
lib.qapb_engine_run.argtypes = [_vp, _P(Report), _vp, C.c_int, _vp]
lib.qapb_engine_best_bound.argtypes = [_vp, _P(C.c_double)]
lib.qapb_engine_gap.argtypes = [_vp, _P(C.c_double)]
lib.qapb_engine_iteration.argtypes = [_vp, _P(C.c_int)]
lib.qapb_engine_last_record.argtypes = [_vp, _P(Record)]
lib.qapb_engine_certificate.argtypes = [_vp, _P(C.c_int), _vp, _P(C.c_double)]
lib.qapb_engine_x_assignment.argtypes = [_vp, _vp]
lib.qapb_engine_array_size.argtypes = [_vp, C.c_int, _P(C.c_size_t)]
lib.qapb_engine_get_array.argtypes = [_vp, C.c_int, _vp, C.c_size_t]
lib.qapb_engine_store_offset.argtypes = [_vp, _P(C.c_double)]
lib.qapb_engine_snapshot.argtypes = [_vp, _vp, _vp, _vp, _P(C.c_double)]
lib.qapb_engine_launch_count.argtypes = [_vp, _P(C.c_longlong)]
lib.qapb_run_ascent.argtypes = [C.c_int, _vp, _vp, _vp, _P(Config), _P(Report), _vp, C.c_int,
                                _vp]
lib.qapb_store_upload.argtypes = [C.c_int, _vp, _vp, _vp, C.c_double, C.c_int, _P(_vp)]
lib.qapb_store_from_engine.argtypes = [_vp, _P(_vp)]
lib.qapb_store_collapse.argtypes = [_vp, C.c_int, C.c_int, _P(_vp)]
lib.qapb_store_info.argtypes = [_vp, _P(C.c_int), _P(C.c_double)]
lib.qapb_store_download.argtypes = [_vp, _vp, _vp, _vp, _P(C.c_double)]
lib.qapb_store_destroy.argtypes = [_vp]
lib.qapb_engine_create_from_store.argtypes = [_vp, _P(Config), _P(_vp)]
lib.qapb_report_json.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_double, C.c_double,
                                 C.c_double, C.c_char_p, C.c_int, C.c_double, _vp, C.c_int,
                                 C.c_double, _vp, C.c_int, C.c_char_p, C.c_size_t,
                                 _P(C.c_size_t)]
lib.qapb_device_count.argtypes = [_P(C.c_int)]
lib.qapb_engine_enqueue.argtypes = [_vp, C.c_int]
lib.qapb_engine_synchronize.argtypes = [_vp]
lib.qapb_engine_stream.argtypes = [_vp, _P(_vp)]
lib.qapb_engine_set_profiling.argtypes = [_vp, C.c_int]
lib.qapb_engine_kernel_times.argtypes = [_vp, _vp, _vp, C.c_int]
lib.qapb_engine_history.argtypes = [_vp, C.c_int, C.c_int, _vp, _vp]
lib.qapb_engine_time_kernel.argtypes = [_vp, C.c_int, C.c_int, _P(C.c_double)]
lib.qapb_shard_plan.argtypes = [C.c_int, C.c_int, _vp]
lib.qapb_shard_exchange_counts.argtypes = [C.c_int, C.c_int, C.c_int, _vp, _vp]
lib.qapb_nccl_unique_id.argtypes = [_vp]
lib.qapb_engine_create_instance_sharded.argtypes = [C.c_int, _vp, _vp, _vp, _P(Config), C.c_int,
                                                    C.c_int, _vp, _P(_vp)]


def shard_plan(n: int, world: int) -> List[int]:
    """First-location boundaries per rank (world+1 entries), SURVEY.md §8(e)."""
    b = np.zeros(world + 1, np.int32)
    _check(lib.qapb_shard_plan(n, world, iptr(b)))
    return [int(x) for x in b]


def shard_exchange_counts(n: int, world: int, rank: int):
    """Doubles `rank` sends to / receives from each peer in one exchange."""
    s = np.zeros(world, np.int64)
    r = np.zeros(world, np.int64)
    _check(lib.qapb_shard_exchange_counts(n, world, rank, s.ctypes.data_as(C.c_void_p),
                                          r.ctypes.data_as(C.c_void_p)))
    return s, r


def nccl_unique_id() -> bytes:
    import torch  # noqa: F401  (bind to the NCCL torch already loaded, see csrc/nccl_dyn.h)
    buf = (C.c_ubyte * 128)()
    _check(lib.qapb_nccl_unique_id(buf))
    return bytes(buf)

KERNEL_NAMES = ["xyfold", "zfold", "zlap", "phase2", "ystage", "xstage", "xchg"]


class QapbError(RuntimeError):
    """Device failure (QAPB_ECUDA); never raised silently."""


class LogicError(RuntimeError):
    """std::logic_error counterpart (rlt2.cpp:332-335, 538-540)."""


def _check(rc: int):
    if rc == 0:
        return
    msg = lib.qapb_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise LogicError(msg)
    if rc == 4:
        raise QapbError(msg)
    raise RuntimeError(msg)


def variant_name(v: int) -> str:
    return lib.qapb_variant_name(int(v)).decode()


def parse_variant(s: str) -> int:
    v = C.c_int()
    _check(lib.qapb_parse_variant(s.encode(), C.byref(v)))
    return v.value


# ---------------------------------------------------------------- LAP -------
@dataclass
class LapResult:
    """lap.hpp:10-16."""
    value: float
    row_to_col: np.ndarray
    col_to_row: np.ndarray
    u: np.ndarray
    v: np.ndarray


def solve_lap(cost, m: Optional[int] = None) -> LapResult:
    """solve_lap (lap.cpp:86-102): one dense LAP on the device."""
    cost = np.ascontiguousarray(cost, dtype=np.float64)
    if m is None:
        m = int(round(math.sqrt(cost.size)))
    if cost.size != m * m:
        raise ValueError("lap: cost size != m*m")
    r = solve_batch(LapBatch.from_costs(cost.reshape(1, m, m)))
    return LapResult(float(r.values[0]), r.row_to_col[0].copy(), r.col_to_row[0].copy(),
                     r.u[0].copy(), r.v[0].copy())


@dataclass
class LapBatch:
    """lap.hpp:37-48: count slots of one size m."""
    m: int = 0
    count: int = 0
    costs: np.ndarray = None
    values: np.ndarray = None
    row_to_col: np.ndarray = None
    col_to_row: np.ndarray = None
    u: np.ndarray = None
    v: np.ndarray = None

    def resize(self, count: int, m: int):
        self.m, self.count = m, count
        self.costs = np.zeros((count, m, m))
        self.values = np.zeros(count)
        self.row_to_col = np.full((count, m), -1, np.int32)
        self.col_to_row = np.full((count, m), -1, np.int32)
        self.u = np.zeros((count, m))
        self.v = np.zeros((count, m))
        return self

    def cost(self, s: int) -> np.ndarray:
        return self.costs[s]

    @classmethod
    def from_costs(cls, costs) -> "LapBatch":
        costs = np.ascontiguousarray(costs, dtype=np.float64)
        b = cls().resize(costs.shape[0], costs.shape[1])
        b.costs[...] = costs
        return b


def solve_batch(batch: LapBatch, workers: int = 1) -> LapBatch:
    """solve_batch (lap.cpp:127-138): every slot on the device, one warp per LAP.
    `workers` is accepted for API parity; results never depend on it."""
    if batch.m <= 0:
        raise ValueError("lap: m must be positive")
    _check(lib.qapb_lap_solve_batch(dptr(batch.costs), batch.m, batch.count,
                                    dptr(batch.values), iptr(batch.row_to_col),
                                    iptr(batch.col_to_row), dptr(batch.u), dptr(batch.v)))
    return batch


def solve_batch_serial(batch: LapBatch) -> LapBatch:
    """lap.cpp:122-125 — same results as solve_batch (kept for API parity)."""
    return solve_batch(batch, 1)


def solve_batch_device(costs_ptr: int, m: int, count: int, values_ptr=0, r2c_ptr=0, c2r_ptr=0,
                       u_ptr=0, v_ptr=0, stream: int = 0):
    """Device-pointer batch (e.g. torch tensors' data_ptr()), enqueued on `stream`."""
    _check(lib.qapb_lap_solve_batch_device(costs_ptr, m, count, values_ptr or None,
                                           r2c_ptr or None, c2r_ptr or None, u_ptr or None,
                                           v_ptr or None, stream or None))


# ---------------------------------------------------------------- store -----
@dataclass
class CoefficientStore:
    """rlt2.hpp:72-82 (reference layout)."""
    m: int
    b: np.ndarray
    c: np.ndarray
    d: np.ndarray
    offset: float = 0.0

    def copy(self) -> "CoefficientStore":
        return CoefficientStore(self.m, self.b.copy(), self.c.copy(), self.d.copy(), self.offset)


def init_coefficients(inst: QapInstance) -> CoefficientStore:
    """rlt2.cpp:66-89 (computed on the device)."""
    n = inst.n
    if n < 3:
        raise ValueError("init_coefficients: n >= 3 required by RLT2")
    nb, nc, nd = store_sizes(n)
    b, c, d = np.empty(nb), np.empty(nc), np.empty(nd)
    _check(lib.qapb_init_coefficients(n, dptr(inst.flow), dptr(inst.dist), dptr(inst.linear),
                                      dptr(b), dptr(c), dptr(d)))
    return CoefficientStore(n, b, c, d, 0.0)


def store_evaluate(st: CoefficientStore, perm) -> float:
    """rlt2.cpp:91-107."""
    p = np.ascontiguousarray(perm, dtype=np.int32)
    v = C.c_double()
    _check(lib.qapb_store_evaluate(st.m, dptr(st.b), dptr(st.c), dptr(st.d), st.offset, iptr(p),
                                   C.byref(v)))
    return v.value


def collapse_store(st: CoefficientStore, fac: int, loc: int) -> CoefficientStore:
    """rlt2.cpp:109-182."""
    mc = st.m - 1
    if mc < 2:
        raise ValueError("collapse_store: store too small")
    nb, nc, nd = store_sizes(mc)
    ob, oc, od = np.empty(nb), np.empty(nc), np.zeros(max(nd, 0))
    off = C.c_double()
    _check(lib.qapb_collapse_store(st.m, dptr(st.b), dptr(st.c), dptr(st.d), st.offset, fac, loc,
                                   dptr(ob), dptr(oc), dptr(od), C.byref(off)))
    return CoefficientStore(mc, ob, oc, od, off.value)


class DeviceStore:
    """A CoefficientStore held in HBM (include/qapb200.h): the B&B
    node flow of bnb.cpp:317-387 -- parent snapshot, collapse_store per child,
    AscentEngine(child) -- without host round trips."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def upload(cls, st: CoefficientStore, device: int = 0) -> "DeviceStore":
        h = _vp()
        d = None if st.d is None else np.ascontiguousarray(st.d, np.float64)
        _check(lib.qapb_store_upload(st.m, dptr(np.ascontiguousarray(st.b, np.float64)),
                                     dptr(np.ascontiguousarray(st.c, np.float64)), dptr(d),
                                     float(st.offset), device, C.byref(h)))
        return cls(h)

    @classmethod
    def from_engine(cls, eng: "AscentEngine") -> "DeviceStore":
        """AscentEngine::snapshot() (rlt2.cpp:537-542) kept on the device."""
        h = _vp()
        _check(lib.qapb_store_from_engine(eng._h, C.byref(h)))
        return cls(h)

    def collapse(self, fac: int, loc: int) -> "DeviceStore":
        """collapse_store(st, fac, loc), rlt2.cpp:109-182, on the device."""
        h = _vp()
        _check(lib.qapb_store_collapse(self._h, fac, loc, C.byref(h)))
        return DeviceStore(h)

    @property
    def m(self) -> int:
        m = C.c_int()
        _check(lib.qapb_store_info(self._h, C.byref(m), None))
        return m.value

    def download(self) -> CoefficientStore:
        m = self.m
        nb, nc, nd = store_sizes(m)
        b, c, d = np.empty(nb), np.empty(nc), np.empty(max(nd, 0))
        off = C.c_double()
        _check(lib.qapb_store_download(self._h, dptr(b), dptr(c), dptr(d) if nd > 0 else None,
                                       C.byref(off)))
        return CoefficientStore(m, b, c, d, off.value)

    def close(self):
        if getattr(self, "_h", None):
            lib.qapb_store_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


def redistribute_family(pi, virtual_slots: int = 3, tol: float = 1e-9):
    """rlt2.cpp:184-205 -> (ok, add[3])."""
    pi = np.ascontiguousarray(pi, dtype=np.float64)
    add = np.empty(3)
    ok = C.c_int()
    _check(lib.qapb_redistribute_family(dptr(pi), dptr(add), virtual_slots, tol, C.byref(ok)))
    return bool(ok.value), add


# ---------------------------------------------------------------- engine ----
@dataclass
class AscentConfig:
    """rlt2.hpp:98-121 (same fields and defaults) + `device`."""
    variant: int = 0
    sa_enabled: bool = False
    iter_limit: int = 100
    min_gap: float = 0.0
    kappa_z_upper: float = 2.0 / 3.0
    phi_split: float = 0.5
    kappa_y: float = 1.0
    kappa_x: float = 1.0
    varphi: float = 0.5
    sa_t0_fraction: float = 0.04
    sa_kappa_lb_cap: float = 0.25
    sa_cool_factor: float = 0.99
    sa_cool_period: int = 100
    workers: int = 1
    seed: int = 0
    upper_bound: float = math.inf
    fathom_threshold: float = math.inf
    early_stop_window: int = 0
    early_stop_delta: float = 0.0002
    record_history: bool = True
    device: int = 0

    def to_c(self) -> Config:
        kw = {f.name: getattr(self, f.name) for f in fields(self)}
        if isinstance(kw["variant"], str):
            kw["variant"] = VARIANTS[kw["variant"].upper()]
        return default_config(**kw)


@dataclass
class IterationRecord:
    """rlt2.hpp:123-128."""
    iteration: int = 0
    bound: float = 0.0
    gap: float = 0.0
    z_ms: float = 0.0
    y_ms: float = 0.0
    x_ms: float = 0.0


@dataclass
class BoundReport:
    """rlt2.hpp:130-146."""
    instance: str = ""
    variant: str = ""
    sa_enabled: bool = False
    best_bound: float = -math.inf
    upper_bound: float = math.inf
    gap: float = math.inf
    termination: str = ""
    iterations: int = 0
    certificate: List[int] = field(default_factory=list)
    certificate_value: float = 0.0
    wall_ms: float = 0.0
    records: List[IterationRecord] = field(default_factory=list)

    def to_json(self) -> str:
        """rlt2.cpp:604-630, byte-identical to the reference (qapb_report_json)."""
        recs = np.array([[r.iteration, r.bound, r.gap, r.z_ms, r.y_ms, r.x_ms]
                         for r in self.records], np.float64).reshape(-1)
        cert = (C.c_int * len(self.certificate))(*self.certificate) if self.certificate else None
        ln = C.c_size_t()
        lib.qapb_report_json(self.instance.encode(), self.variant.encode(), int(self.sa_enabled),
                             self.best_bound, self.upper_bound, self.gap,
                             self.termination.encode(), self.iterations, self.wall_ms, cert,
                             len(self.certificate), self.certificate_value,
                             dptr(recs) if len(self.records) else None, len(self.records), None,
                             0, C.byref(ln))
        buf = C.create_string_buffer(ln.value + 1)
        _check(lib.qapb_report_json(self.instance.encode(), self.variant.encode(),
                                    int(self.sa_enabled), self.best_bound, self.upper_bound,
                                    self.gap, self.termination.encode(), self.iterations,
                                    self.wall_ms, cert, len(self.certificate),
                                    self.certificate_value,
                                    dptr(recs) if len(self.records) else None,
                                    len(self.records), buf, len(buf), C.byref(ln)))
        return buf.value.decode()

    def to_csv(self) -> str:
        """rlt2.cpp:632-640 (default ostream formatting, precision 6)."""
        def g(x):
            s = "%g" % x
            return "inf" if s == "inf" else ("-inf" if s == "-inf" else s)
        out = ["iteration,bound,gap,z_ms,y_ms,x_ms"]
        for r in self.records:
            gap = r.gap if math.isfinite(r.gap) else -1.0
            out.append(f"{r.iteration},{g(r.bound)},{g(gap)},{g(r.z_ms)},{g(r.y_ms)},{g(r.x_ms)}")
        return "\n".join(out) + "\n"


def _report(rep: Report, recs, cert, cfg: AscentConfig) -> BoundReport:
    r = BoundReport()
    r.variant = VARIANT_NAMES[cfg.to_c().variant]
    r.sa_enabled = bool(cfg.sa_enabled)
    r.best_bound = rep.best_bound
    r.upper_bound = rep.upper_bound
    r.gap = rep.gap
    r.termination = TERM_NAMES[rep.termination]
    r.iterations = rep.iterations
    if rep.has_certificate:
        r.certificate = [int(x) for x in cert]
        r.certificate_value = rep.certificate_value
    r.wall_ms = rep.wall_ms
    r.records = [IterationRecord(x.iteration, x.bound, x.gap, x.z_ms, x.y_ms, x.x_ms)
                 for x in (recs[i] for i in range(rep.n_records))]
    return r


class AscentEngine:
    """rlt2.hpp:151-213, device resident.  `store` is consumed (copied to HBM)."""

    def __init__(self, store: CoefficientStore, cfg: Optional[AscentConfig] = None):
        self.cfg = cfg or AscentConfig()
        self.m = store.m
        h = C.c_void_p()
        c = self.cfg.to_c()
        d = None if store.d is None else np.ascontiguousarray(store.d, np.float64)
        _check(lib.qapb_engine_create(store.m, dptr(np.ascontiguousarray(store.b, np.float64)),
                                      dptr(np.ascontiguousarray(store.c, np.float64)), dptr(d),
                                      float(store.offset), C.byref(c), C.byref(h)))
        self._h = h

    @classmethod
    def from_instance(cls, inst: QapInstance, cfg: Optional[AscentConfig] = None):
        """AscentEngine(init_coefficients(inst), cfg) with the store built on the device."""
        self = cls.__new__(cls)
        self.cfg = cfg or AscentConfig()
        self.m = inst.n
        h = C.c_void_p()
        c = self.cfg.to_c()
        _check(lib.qapb_engine_create_instance(inst.n, dptr(inst.flow), dptr(inst.dist),
                                               dptr(inst.linear), C.byref(c), C.byref(h)))
        self._h = h
        return self

    @classmethod
    def from_device_store(cls, store: "DeviceStore", cfg: Optional[AscentConfig] = None):
        """AscentEngine(CoefficientStore, cfg) from a store already in HBM."""
        self = cls.__new__(cls)
        self.cfg = cfg or AscentConfig()
        self.m = store.m
        h = C.c_void_p()
        c = self.cfg.to_c()
        _check(lib.qapb_engine_create_from_store(store._h, C.byref(c), C.byref(h)))
        self._h = h
        return self

    @classmethod
    def from_instance_sharded(cls, inst: QapInstance, cfg: Optional[AscentConfig], rank: int,
                              world: int, nccl_id: bytes):
        """One rank of a z-sharded engine (one process per GPU).
        Every rank passes the same instance, cfg and NCCL id; cfg.device = its GPU."""
        import torch  # noqa: F401  (bind to the NCCL torch already loaded)
        self = cls.__new__(cls)
        self.cfg = cfg or AscentConfig()
        self.m = inst.n
        h = C.c_void_p()
        c = self.cfg.to_c()
        idbuf = (C.c_ubyte * 128).from_buffer_copy(nccl_id)
        _check(lib.qapb_engine_create_instance_sharded(inst.n, dptr(inst.flow), dptr(inst.dist),
                                                       dptr(inst.linear), C.byref(c), rank, world,
                                                       idbuf, C.byref(h)))
        self._h = h
        return self

    def close(self):
        if getattr(self, "_h", None):
            lib.qapb_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def iterate(self) -> float:
        b = C.c_double()
        _check(lib.qapb_engine_iterate(self._h, C.byref(b)))
        return b.value

    def run(self) -> BoundReport:
        rep = Report()
        n = max(1, self.cfg.iter_limit)
        recs = (Record * n)()
        cert = np.full(self.m, -1, np.int32)
        _check(lib.qapb_engine_run(self._h, C.byref(rep), recs, n, iptr(cert)))
        return _report(rep, recs, cert, self.cfg)

    def best_bound(self) -> float:
        v = C.c_double()
        _check(lib.qapb_engine_best_bound(self._h, C.byref(v)))
        return v.value

    def gap(self) -> float:
        v = C.c_double()
        _check(lib.qapb_engine_gap(self._h, C.byref(v)))
        return v.value

    def iteration(self) -> int:
        v = C.c_int()
        _check(lib.qapb_engine_iteration(self._h, C.byref(v)))
        return v.value

    def _array(self, which: str) -> np.ndarray:
        n = C.c_size_t()
        _check(lib.qapb_engine_array_size(self._h, ARR[which], C.byref(n)))
        out = np.empty(n.value)
        if n.value:
            _check(lib.qapb_engine_get_array(self._h, ARR[which], dptr(out), n.value))
        return out

    def pi_z(self): return self._array("pi_z")
    def pi_y(self): return self._array("pi_y")
    def pi_x(self): return self._array("pi_x")
    def theta(self): return self._array("theta")
    def delta(self): return self._array("delta")
    def incz(self): return self._array("incz")
    def array(self, which: str): return self._array(which)

    def store(self) -> CoefficientStore:
        off = C.c_double()
        _check(lib.qapb_engine_store_offset(self._h, C.byref(off)))
        return CoefficientStore(self.m, self._array("b"), self._array("c"), self._array("d"),
                                off.value)

    def snapshot(self) -> CoefficientStore:
        nb, nc, nd = store_sizes(self.m)
        b, c, d = np.empty(nb), np.empty(nc), np.empty(nd)
        off = C.c_double()
        _check(lib.qapb_engine_snapshot(self._h, dptr(b), dptr(c), dptr(d), C.byref(off)))
        return CoefficientStore(self.m, b, c, d, off.value)

    def has_certificate(self) -> bool:
        return self._cert()[0]

    def certificate(self) -> List[int]:
        return self._cert()[1]

    def certificate_value(self) -> float:
        return self._cert()[2]

    def _cert(self):
        has = C.c_int()
        perm = np.full(self.m, -1, np.int32)
        val = C.c_double()
        _check(lib.qapb_engine_certificate(self._h, C.byref(has), iptr(perm), C.byref(val)))
        return bool(has.value), ([int(x) for x in perm] if has.value else []), val.value

    def x_assignment(self) -> List[int]:
        x = np.empty(self.m, np.int32)
        _check(lib.qapb_engine_x_assignment(self._h, iptr(x)))
        return [int(v) for v in x]

    # ---- device-loop / measurement hooks (B200 extension) ----
    def enqueue(self, iters: int):
        """Enqueue `iters` iterate() steps with no host synchronisation."""
        _check(lib.qapb_engine_enqueue(self._h, iters))

    def synchronize(self):
        _check(lib.qapb_engine_synchronize(self._h))

    def stream(self) -> int:
        s = C.c_void_p()
        _check(lib.qapb_engine_stream(self._h, C.byref(s)))
        return s.value or 0

    def set_profiling(self, on: bool):
        _check(lib.qapb_engine_set_profiling(self._h, int(on)))

    def kernel_times(self, reset: bool = False):
        ms = np.zeros(len(KERNEL_NAMES))
        n = np.zeros(len(KERNEL_NAMES), np.int64)
        _check(lib.qapb_engine_kernel_times(self._h, dptr(ms), n.ctypes.data_as(C.c_void_p),
                                            int(reset)))
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(KERNEL_NAMES)}

    def history(self, start: int = 0, count: Optional[int] = None):
        if count is None:
            count = self.iteration() - start
        b, best = np.empty(count), np.empty(count)
        _check(lib.qapb_engine_history(self._h, start, count, dptr(b), dptr(best)))
        return b, best

    def time_kernel(self, kind: str, reps: int = 5) -> float:
        """Tuning only: mean ms of one kernel kind; destroys the numerical state."""
        ms = C.c_double()
        _check(lib.qapb_engine_time_kernel(self._h, KERNEL_NAMES.index(kind), reps, C.byref(ms)))
        return ms.value

    def launch_count(self) -> int:
        n = C.c_longlong()
        _check(lib.qapb_engine_launch_count(self._h, C.byref(n)))
        return n.value


def run_ascent(inst: QapInstance, cfg: Optional[AscentConfig] = None) -> BoundReport:
    """rlt2.cpp:590-597."""
    cfg = cfg or AscentConfig()
    rep = Report()
    n = max(1, cfg.iter_limit)
    recs = (Record * n)()
    cert = np.full(inst.n, -1, np.int32)
    c = cfg.to_c()
    _check(lib.qapb_run_ascent(inst.n, dptr(inst.flow), dptr(inst.dist), dptr(inst.linear),
                               C.byref(c), C.byref(rep), recs, n, iptr(cert)))
    r = _report(rep, recs, cert, cfg)
    r.instance = inst.name
    return r


def run_ascent_warm(warm: CoefficientStore, cfg: Optional[AscentConfig] = None) -> BoundReport:
    """rlt2.cpp:599-602."""
    eng = AscentEngine(warm, cfg)
    try:
        return eng.run()
    finally:
        eng.close()


__all__ = ["AscentConfig", "AscentEngine", "BoundReport", "CoefficientStore", "IterationRecord",
           "LapBatch", "LapResult", "LogicError", "QapbError", "collapse_store",
           "evaluate_objective", "init_coefficients", "redistribute_family", "run_ascent",
           "run_ascent_warm", "solve_batch", "solve_batch_serial", "solve_lap",
           "store_evaluate"]

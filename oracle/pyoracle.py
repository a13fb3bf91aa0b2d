"""oracle/pyoracle.py — TEST INFRASTRUCTURE ONLY (the checker, never the product).

ctypes bindings for the two CPU oracles of the RLT2 dual-ascent path:

* ``kind="ref"``  — the unmodified reference library compiled from
  /root/reference/proj/src by oracle/Makefile into oracle/_ref/libqapref.so
  (wrapper: oracle/ref_capi.cpp);
* ``kind="port"`` — the plain-C restatement oracle/rlt2_oracle.c
  (oracle/liboracle_port.so).

Both expose the same surface so tests can cross-check them and use whichever
exists.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
reference arm import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def _load_abi():
    """The shared struct layouts (paper_1710_03732_b200/abi.py: plain ctypes,
    loads no library) imported as a standalone module, so that using the
    oracle never runs the product package's __init__ (which maps
    libqapb200.so) -- the reference arm of bench.py must not load it."""
    import importlib.util
    name = "_qapb_abi_layouts"
    if name in sys.modules:
        return sys.modules[name]
    path = os.path.join(os.path.dirname(HERE), "paper_1710_03732_b200", "abi.py")
    spec = importlib.util.spec_from_file_location(name, path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules[name] = mod
    spec.loader.exec_module(mod)
    return mod


_abi = _load_abi()
Config, Record, Report, ARR, TERM_NAMES = _abi.Config, _abi.Record, _abi.Report, _abi.ARR, \
    _abi.TERM_NAMES
default_config, dptr, iptr, store_sizes = _abi.default_config, _abi.dptr, _abi.iptr, \
    _abi.store_sizes

REF_LIB = os.path.join(HERE, "_ref", "libqapref.so")
PORT_LIB = os.path.join(HERE, "liboracle_port.so")

_libs: dict[str, C.CDLL] = {}


def available(kind: str) -> bool:
    return os.path.exists(REF_LIB if kind == "ref" else PORT_LIB)


def _load(kind: str) -> C.CDLL:
    if kind in _libs:
        return _libs[kind]
    path = REF_LIB if kind == "ref" else PORT_LIB
    if not os.path.exists(path):
        raise FileNotFoundError(f"oracle '{kind}' not built: {path}")
    lib = C.CDLL(path)
    pre = "qref_" if kind == "ref" else "orc_"
    vp = C.c_void_p
    P = C.POINTER
    if kind == "ref":
        lib.qref_lap_solve.argtypes = [vp, C.c_int, vp, vp, vp, vp, P(C.c_double)]
        lib.qref_lap_solve.restype = C.c_int
        lib.qref_lap_solve_batch.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, vp]
        lib.qref_generate_instance.argtypes = [C.c_int, C.c_ulonglong, C.c_int, vp, vp]
        lib.qref_init_coefficients.argtypes = [C.c_int, vp, vp, vp, vp, vp, vp]
        lib.qref_engine_create.argtypes = [C.c_int, vp, vp, vp, C.c_double, P(Config), P(vp)]
        lib.qref_store_evaluate.argtypes = [C.c_int, vp, vp, vp, C.c_double, vp, P(C.c_double)]
        lib.qref_collapse_store.argtypes = [C.c_int, vp, vp, vp, C.c_double, C.c_int, C.c_int,
                                            vp, vp, vp, P(C.c_double)]
        lib.qref_evaluate_objective.argtypes = [C.c_int, vp, vp, vp, vp, P(C.c_double)]
        lib.qref_last_error.restype = C.c_char_p
        lib.qref_redistribute_family.argtypes = [vp, vp, C.c_int, C.c_double, P(C.c_int)]
    else:
        lib.orc_lap_solve.argtypes = [vp, C.c_int, vp, vp, vp, vp]
        lib.orc_lap_solve.restype = C.c_double
        lib.orc_generate_instance.argtypes = [C.c_int, C.c_uint64, C.c_int, vp, vp]
        lib.orc_init_coefficients.argtypes = [C.c_int, vp, vp, vp, vp, vp, vp]
        lib.orc_engine_create.argtypes = [C.c_int, vp, vp, vp, C.c_double, P(Config), P(vp)]
        lib.orc_last_error.restype = C.c_char_p
        lib.orc_redistribute_family.argtypes = [vp, vp, C.c_int, C.c_double]
    for name in ("engine_iterate",):
        getattr(lib, pre + name).argtypes = [vp, P(C.c_double)]
    getattr(lib, pre + "engine_run").argtypes = [vp, P(Report), vp, C.c_int, vp]
    getattr(lib, pre + "engine_array_size").argtypes = [vp, C.c_int, P(C.c_size_t)]
    getattr(lib, pre + "engine_get_array").argtypes = [vp, C.c_int, vp, C.c_size_t]
    getattr(lib, pre + "engine_scalars").argtypes = [vp, P(C.c_double), P(C.c_double),
                                                    P(C.c_int), P(C.c_double), P(C.c_double)]
    getattr(lib, pre + "engine_certificate").argtypes = [vp, P(C.c_int), vp, P(C.c_double)]
    getattr(lib, pre + "engine_x_assignment").argtypes = [vp, vp]
    getattr(lib, pre + "engine_destroy").argtypes = [vp]
    _libs[kind] = lib
    return lib


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Oracle:
    """One CPU implementation of the path (reference build or C port)."""

    def __init__(self, kind: str = "ref"):
        self.kind = kind
        self.lib = _load(kind)
        self.pre = "qref_" if kind == "ref" else "orc_"

    def _check(self, rc: int):
        if rc:
            raise OracleError(rc, getattr(self.lib, self.pre + "last_error")().decode())

    # ---- LAP (lap.cpp:24-84) ----
    def lap_solve(self, cost: np.ndarray):
        cost = np.ascontiguousarray(cost, dtype=np.float64)
        m = cost.shape[0]
        r2c = np.empty(m, np.int32)
        c2r = np.empty(m, np.int32)
        u = np.empty(m)
        v = np.empty(m)
        if self.kind == "ref":
            val = C.c_double()
            self._check(self.lib.qref_lap_solve(dptr(cost), m, iptr(r2c), iptr(c2r), dptr(u),
                                                dptr(v), C.byref(val)))
            value = val.value
        else:
            value = self.lib.orc_lap_solve(dptr(cost), m, iptr(r2c), iptr(c2r), dptr(u), dptr(v))
        return value, r2c, c2r, u, v

    def lap_solve_batch(self, costs: np.ndarray, workers: int = 0):
        costs = np.ascontiguousarray(costs, dtype=np.float64)
        count, m, _ = costs.shape
        values = np.empty(count)
        r2c = np.empty((count, m), np.int32)
        c2r = np.empty((count, m), np.int32)
        u = np.empty((count, m))
        v = np.empty((count, m))
        if self.kind == "ref":
            self._check(self.lib.qref_lap_solve_batch(
                dptr(costs), m, count, workers or os.cpu_count(), dptr(values), iptr(r2c),
                iptr(c2r), dptr(u), dptr(v)))
        else:
            for s in range(count):
                values[s], r2c[s], c2r[s], u[s], v[s] = self.lap_solve(costs[s])
        return values, r2c, c2r, u, v

    # ---- instances / store ----
    def generate_instance(self, n: int, seed: int, max_entry: int = 99):
        flow = np.zeros((n, n))
        dist = np.zeros((n, n))
        self._check(getattr(self.lib, self.pre + "generate_instance")(
            n, seed, max_entry, dptr(flow), dptr(dist)))
        return flow, dist

    def init_coefficients(self, flow, dist, linear=None):
        n = flow.shape[0]
        nb, nc, nd = store_sizes(n)
        b, c, d = np.empty(nb), np.empty(nc), np.empty(nd)
        lin = None if linear is None else np.ascontiguousarray(linear, np.float64)
        self._check(getattr(self.lib, self.pre + "init_coefficients")(
            n, dptr(np.ascontiguousarray(flow, np.float64)),
            dptr(np.ascontiguousarray(dist, np.float64)), dptr(lin), dptr(b), dptr(c), dptr(d)))
        return b, c, d

    def redistribute_family(self, pi, virtual_slots=3, tol=1e-9):
        pi = np.ascontiguousarray(pi, np.float64)
        add = np.empty(3)
        if self.kind == "ref":
            ok = C.c_int()
            self._check(self.lib.qref_redistribute_family(dptr(pi), dptr(add), virtual_slots, tol,
                                                          C.byref(ok)))
            return bool(ok.value), add
        ok = self.lib.orc_redistribute_family(dptr(pi), dptr(add), virtual_slots, tol)
        return bool(ok), add

    def engine(self, m, b, c, d, offset=0.0, cfg: Config | None = None) -> "OracleEngine":
        return OracleEngine(self, m, b, c, d, offset, cfg or default_config())

    def engine_from_instance(self, flow, dist, linear=None, cfg=None) -> "OracleEngine":
        b, c, d = self.init_coefficients(flow, dist, linear)
        return self.engine(flow.shape[0], b, c, d, 0.0, cfg)


def _as_cfg(cfg) -> Config:
    """A config struct of this module's Config type (callers may hold the
    product package's identical-layout class)."""
    if isinstance(cfg, Config):
        return cfg
    out = Config()
    for name, _ in Config._fields_:
        setattr(out, name, getattr(cfg, name))
    return out


class OracleEngine:
    def __init__(self, orc: Oracle, m, b, c, d, offset, cfg: Config):
        self.o = orc
        self.m = m
        cfg = _as_cfg(cfg)
        self.cfg = cfg
        h = C.c_void_p()
        self._b, self._c = np.ascontiguousarray(b, np.float64), np.ascontiguousarray(c, np.float64)
        dd = None if d is None else np.ascontiguousarray(d, np.float64)
        orc._check(getattr(orc.lib, orc.pre + "engine_create")(
            m, dptr(self._b), dptr(self._c), dptr(dd), float(offset), C.byref(cfg), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            getattr(self.o.lib, self.o.pre + "engine_destroy")(self.h)
            self.h = None

    def _fn(self, name):
        return getattr(self.o.lib, self.o.pre + name)

    def iterate(self) -> float:
        b = C.c_double()
        self.o._check(self._fn("engine_iterate")(self.h, C.byref(b)))
        return b.value

    def run(self):
        rep = Report()
        recs = (Record * max(1, self.cfg.iter_limit))()
        cert = np.full(self.m, -1, np.int32)
        self.o._check(self._fn("engine_run")(self.h, C.byref(rep), recs, self.cfg.iter_limit,
                                             iptr(cert)))
        return rep, [recs[i] for i in range(rep.n_records)], cert

    def scalars(self):
        best, gap, last, running = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        it = C.c_int()
        self._fn("engine_scalars")(self.h, C.byref(best), C.byref(gap), C.byref(it),
                                   C.byref(last), C.byref(running))
        return dict(best=best.value, gap=gap.value, iteration=it.value, last_bound=last.value,
                    running=running.value)

    def array(self, which) -> np.ndarray:
        w = ARR[which] if isinstance(which, str) else which
        n = C.c_size_t()
        self._fn("engine_array_size")(self.h, w, C.byref(n))
        out = np.empty(n.value)
        if n.value:
            self.o._check(self._fn("engine_get_array")(self.h, w, dptr(out), n.value))
        return out

    def certificate(self):
        has = C.c_int()
        perm = np.full(self.m, -1, np.int32)
        val = C.c_double()
        self._fn("engine_certificate")(self.h, C.byref(has), iptr(perm), C.byref(val))
        return bool(has.value), perm, val.value

    def x_assignment(self):
        x = np.empty(self.m, np.int32)
        self._fn("engine_x_assignment")(self.h, iptr(x))
        return x


def best_oracle() -> Oracle:
    """The compiled reference when present, else the C port."""
    return Oracle("ref" if available("ref") else "port")


__all__ = ["Oracle", "OracleEngine", "OracleError", "available", "best_oracle", "TERM_NAMES"]

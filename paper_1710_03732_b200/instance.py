"""QAP instances: QAPLIB I/O, seeded generator, objective.

Host-side conveniences with the semantics of /root/reference/proj/src/instance.cpp
(out of the hot path); they produce the synthetic inputs of
the benchmark configurations.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

_M64 = (1 << 64) - 1


class _MT19937_64:
    """std::mt19937_64 (the generator behind generate_instance, instance.cpp:139)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & _M64
        for i in range(1, 312):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & _M64
        self.idx = 312

    def __call__(self) -> int:
        if self.idx >= 312:
            mt = self.mt
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _M64


@dataclass
class QapInstance:
    """Lawler-form QAP data (instance.hpp:13-24); matrices are n x n float64."""
    n: int
    flow: np.ndarray
    dist: np.ndarray
    linear: np.ndarray = field(default=None)
    name: str = ""

    def __post_init__(self):
        self.flow = np.ascontiguousarray(self.flow, dtype=np.float64).reshape(self.n, self.n)
        self.dist = np.ascontiguousarray(self.dist, dtype=np.float64).reshape(self.n, self.n)
        if self.linear is None:
            self.linear = np.zeros((self.n, self.n))
        self.linear = np.ascontiguousarray(self.linear, dtype=np.float64).reshape(self.n, self.n)


def evaluate_objective(inst: QapInstance, perm) -> float:
    """instance.cpp:11-26 (same summation order)."""
    n = inst.n
    perm = [int(p) for p in perm]
    if len(perm) != n:
        raise ValueError("perm size != n")
    if sorted(perm) != list(range(n)):
        raise ValueError("not a permutation")
    v = 0.0
    for i in range(n):
        v += float(inst.linear[i, perm[i]])
        for j in range(n):
            v += float(inst.flow[i, j]) * float(inst.dist[perm[i], perm[j]])
    return v


def generate_instance(n: int, seed: int, max_entry: int = 99) -> QapInstance:
    """instance.cpp:131-150: symmetric, zero diagonal, integers in [0, max_entry]."""
    if n < 2:
        raise ValueError("n must be >= 2")
    g = _MT19937_64(seed)
    f = np.zeros((n, n))
    d = np.zeros((n, n))
    for i in range(n):
        for j in range(i + 1, n):
            f[i, j] = f[j, i] = float(g() % (max_entry + 1))
    for p in range(n):
        for q in range(p + 1, n):
            d[p, q] = d[q, p] = float(g() % (max_entry + 1))
    return QapInstance(n, f, d, np.zeros((n, n)), f"rand{n}-{seed}")


def grid_instance(rows: int, cols: int, flow_seed: int = 1, max_flow: int = 10,
                  name: str = "") -> QapInstance:
    """Nugent-shaped instance: Manhattan distances on a rows x cols grid (as
    tests/test_bnb.cpp:35-44 grid_instance) with the flow matrix of
    generate_instance(rows*cols, flow_seed, max_flow)."""
    n = rows * cols
    base = generate_instance(n, flow_seed, max_flow)
    d = np.zeros((n, n))
    for a in range(n):
        for b in range(n):
            d[a, b] = abs(a // cols - b // cols) + abs(a % cols - b % cols)
    return QapInstance(n, base.flow, d, np.zeros((n, n)), name or f"grid{rows}x{cols}")


def parse_qaplib(text: str, swap_order: bool = False, name: str = "") -> QapInstance:
    """instance.cpp:37-61."""
    toks = text.split()
    try:
        n = int(toks[0])
    except (IndexError, ValueError):
        raise RuntimeError("bad instance size")
    if n <= 0:
        raise RuntimeError("bad instance size")
    nn = n * n
    vals = [float(t) for t in toks[1:]]
    if len(vals) < 2 * nn:
        raise RuntimeError("truncated input")
    a = np.array(vals[:nn]).reshape(n, n)
    b = np.array(vals[nn:2 * nn]).reshape(n, n)
    rest = vals[2 * nn:]
    if rest:
        if len(rest) < nn:
            raise RuntimeError("truncated linear-cost matrix")
        lin = np.array(rest[:nn]).reshape(n, n)
    else:
        lin = np.zeros((n, n))
    flow, dist = (b, a) if swap_order else (a, b)
    return QapInstance(n, flow, dist, lin, name)


def load_qaplib_file(path: str, swap_order: bool = False) -> QapInstance:
    with open(path) as fh:
        text = fh.read()
    return parse_qaplib(text, swap_order, os.path.splitext(os.path.basename(path))[0])


def parse_solution(text: str, expect_n: int):
    """instance.cpp:82-102: returns (perm 0-based, value)."""
    toks = text.split()
    n, v = int(toks[0]), float(toks[1])
    if n != expect_n:
        raise RuntimeError("solution size mismatch")
    perm = [int(t) - 1 for t in toks[2:2 + n]]
    if sorted(perm) != list(range(n)):
        raise RuntimeError("solution is not a permutation")
    return perm, v

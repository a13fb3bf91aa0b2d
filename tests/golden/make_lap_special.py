"""Generate tests/golden/lap_special.npz from the COMPILED REFERENCE
(oracle/_ref/libqapref.so, LapSolver::solve, lap.cpp:24-84): LAP inputs the
fast warp solvers do not take — +inf and huge (|c| > 1e300) costs, NaN, -0.0
— and sizes above the warp solvers' limit (m > 127, the CTA-per-LAP path).

    python tests/golden/make_lap_special.py

Every case is one where the reference is well defined (its scan always finds
a column).  Test infrastructure only; the GPU tests read the .npz.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Oracle  # noqa: E402


def cases():
    inf = np.inf
    rng = np.random.default_rng(1701)
    out = []
    out.append(np.array([[inf, 1, 5], [2, inf, 3], [4, 6, inf]]))   # ADVICE r01 example
    out.append(np.array([[1e301, 2, 3, 4], [5, 1e301, 7, 8], [9, 10, 1e301, 12],
                         [13, 14, 15, 1e301]]))
    for m in (5, 10, 28, 31, 40, 64):
        for kind in range(4):
            c = rng.integers(0, 100, (m, m)).astype(float)
            if kind == 0:    # sparse +inf (a finite perfect matching survives: diagonal)
                mask = rng.random((m, m)) < 0.3
                np.fill_diagonal(mask, False)
                c[mask] = inf
            elif kind == 1:  # huge finite costs mixed with small ones
                mask = rng.random((m, m)) < 0.2
                c[mask] = rng.choice([1e301, 1e305, -1e302], mask.sum())
            elif kind == 2:  # NaN entries off a finite diagonal
                mask = rng.random((m, m)) < 0.1
                np.fill_diagonal(mask, False)
                c[mask] = np.nan
            else:            # signed zeros (the argmin key's +-0 tie rule)
                c = np.floor(rng.random((m, m)) * 3.0) - 1.0
                c[c == 0] = rng.choice([0.0, -0.0], (c == 0).sum())
            out.append(c)
    for m in (128, 150, 203):  # the CTA-per-LAP path
        out.append(rng.integers(0, 1000, (m, m)).astype(float))
        out.append(np.floor(rng.random((m, m)) * 4.0))
    return out


def main():
    orc = Oracle("ref")
    ms, costs, vals, r2cs, us, vs = [], [], [], [], [], []
    for c in cases():
        m = c.shape[0]
        val, r2c, _, u, v = orc.lap_solve(c)
        ms.append(m)
        costs.append(c.ravel())
        vals.append(val)
        r2cs.append(r2c)
        us.append(u)
        vs.append(v)
    np.savez_compressed(os.path.join(HERE, "lap_special.npz"), m=np.array(ms),
                        costs=np.concatenate(costs), values=np.array(vals),
                        r2c=np.concatenate(r2cs), u=np.concatenate(us), v=np.concatenate(vs))
    print("wrote", len(ms), "cases")


if __name__ == "__main__":
    main()

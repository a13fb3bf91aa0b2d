"""Generate tests/golden/* from the COMPILED REFERENCE (oracle/_ref/libqapref.so).

Run here (where /root/reference exists) after `make -C oracle ref`:

    python tests/golden/make_golden.py

Outputs (committed, small):
  golden.json     per-iteration bound traces (hex floats, bitwise) and
                  sha256 digests of the engine arrays at chosen iterations,
                  iteration-1 Gilmore-Lawler values, instance data
  lap_cases.npz   LAP inputs + reference outputs (values, r2c, u, v)

Nothing on the GPU box regenerates these; the tests only read them.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle.pyoracle import Oracle  # noqa: E402
from paper_1710_03732_b200.abi import default_config  # noqa: E402

REF_FIX = "/root/reference/proj/fixtures"


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()[:32]


def load_dat(path):
    toks = open(path).read().split()
    n = int(toks[0])
    v = np.array(toks[1:], dtype=float)
    return n, v[:n * n].reshape(n, n), v[n * n:2 * n * n].reshape(n, n)


def grid(rows, cols, orc, seed=1, mx=10):
    n = rows * cols
    f, _ = orc.generate_instance(n, seed, mx)
    d = np.zeros((n, n))
    for a in range(n):
        for b in range(n):
            d[a, b] = abs(a // cols - b // cols) + abs(a % cols - b % cols)
    return f, d


ARRAYS = ["pi_z", "pi_y", "pi_x", "b", "c", "d", "theta", "delta"]


def trace(orc, f, d, variant, iters, sa=False, ub=float("inf"), seed=0, snap_at=(),
          workers=8):
    cfg = default_config(variant=variant, iter_limit=iters, sa_enabled=sa, upper_bound=ub,
                         seed=seed, workers=workers)
    eng = orc.engine_from_instance(f, d, cfg=cfg)
    bounds, best, snaps = [], [], {}
    for it in range(1, iters + 1):
        bounds.append(float(eng.iterate()).hex())
        best.append(float(eng.scalars()["best"]).hex())
        if it in snap_at:
            snaps[str(it)] = {a: digest(eng.array(a)) for a in ARRAYS}
            if variant in ("F1", "F2"):
                snaps[str(it)]["incz"] = digest(eng.array("incz"))
            snaps[str(it)]["x_assignment"] = [int(x) for x in eng.x_assignment()]
    has, perm, val = eng.certificate()
    return {"variant": variant, "iters": iters, "sa": sa, "upper_bound": ub, "seed": seed,
            "bounds": bounds, "best": best, "digests": snaps,
            "certificate": [int(x) for x in perm] if has else [], "certificate_value": val}


def main():
    orc = Oracle("ref")
    out = {"generator": "oracle/_ref/libqapref.so (reference proj/src compiled unmodified)"}
    n, F, D = load_dat(os.path.join(REF_FIX, "nug12.dat"))
    out["nug12"] = {"n": n, "flow": F.astype(int).tolist(), "dist": D.astype(int).tolist()}
    for name in ("nug5", "zero", "two"):
        nn, f, d = load_dat(os.path.join(REF_FIX, f"{name}.dat"))
        out[name] = {"n": nn, "flow": f.astype(int).tolist(), "dist": d.astype(int).tolist()}
    tr = {}
    for v in ("F1", "S1", "F2", "S2"):
        tr[f"nug12_{v}"] = trace(orc, F, D, v, 100, snap_at=(1, 2, 5, 100))
    tr["nug12_F1_SA"] = trace(orc, F, D, "F1", 100, sa=True, ub=578.0, snap_at=(100,))
    tr["nug12_F2_SA"] = trace(orc, F, D, "F2", 60, sa=True, ub=578.0, snap_at=(60,))
    tr["nug12_S1_SA"] = trace(orc, F, D, "S1", 60, sa=True, ub=578.0, seed=7, snap_at=(60,))
    f20, d20 = orc.generate_instance(20, 1, 99)
    tr["rand20_F1"] = trace(orc, f20, d20, "F1", 3, snap_at=(1, 2, 3))
    tr["rand20_S1"] = trace(orc, f20, d20, "S1", 3, snap_at=(3,))
    tr["rand20_F2"] = trace(orc, f20, d20, "F2", 2, snap_at=(2,))
    gf, gd = grid(4, 5, orc)
    tr["grid20_F1"] = trace(orc, gf, gd, "F1", 4, snap_at=(4,))
    for seed in (1, 2, 3):  # odd and small sizes exercise the non-bulk tile path
        nn = 5 + seed * 2
        f, d = orc.generate_instance(nn, 100 + seed, 99)
        tr[f"rand{nn}_S2"] = trace(orc, f, d, "S2", 40, snap_at=(40,))
        tr[f"rand{nn}_F1_SA"] = trace(orc, f, d, "F1", 40, sa=True, ub=float("inf"), seed=seed,
                                      snap_at=(40,))
    # n=30 pins: the bench workload and the tai-a-shaped case
    g30f, g30d = grid(5, 6, orc)
    tr["grid30_F1"] = trace(orc, g30f, g30d, "F1", 6, snap_at=(2,))
    f30, d30 = orc.generate_instance(30, 1, 99)
    tr["rand30_S1"] = trace(orc, f30, d30, "S1", 3)
    out["traces"] = tr
    # iteration-1 (Gilmore-Lawler) values of the reference test instances
    gl = {}
    for seed in range(6):
        nn = 5 + seed % 3
        f, d = orc.generate_instance(nn, seed * 31 + 1, 99)
        gl[f"{nn}_{seed * 31 + 1}"] = float(orc.engine_from_instance(
            f, d, cfg=default_config(iter_limit=1)).iterate()).hex()
    out["gl"] = gl
    # pinned instances: iteration-1 values
    out["instances"] = {
        "gen20_1_99_sha": digest(f20) + digest(d20),
        "gen30_1_99_sha": "".join(digest(x) for x in orc.generate_instance(30, 1, 99)),
        "gen42_1_10_sha": "".join(digest(x) for x in orc.generate_instance(42, 1, 10)),
    }
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)

    # LAP cases
    rng = np.random.default_rng(2024)
    costs, ms = [], []
    for _ in range(300):  # test_lap.cpp:69-80 shape: m<=8, negatives
        m = int(rng.integers(1, 9))
        costs.append((rng.integers(0, 100, (m, m)) - 20.0).ravel())
        ms.append(m)
    for m in (1, 2, 3, 4, 9, 10, 16, 17, 28, 29, 30, 31, 32, 33, 40, 41, 42, 47, 63, 64, 65,
              90, 100, 127):
        for kind in range(3):
            if kind == 0:
                c = rng.integers(0, 100, (m, m)).astype(float)
            elif kind == 1:
                c = rng.normal(size=(m, m)) * 10.0
            else:
                c = np.floor(rng.random((m, m)) * 3.0)  # heavy ties
            costs.append(c.ravel())
            ms.append(m)
    for m in (4, 7):
        costs.append(np.full(m * m, 3.0))  # all-equal -> identity
        ms.append(m)
        costs.append(np.zeros(m * m))
        ms.append(m)
    vals, r2cs, us, vs = [], [], [], []
    for c, m in zip(costs, ms):
        val, r2c, c2r, u, v = orc.lap_solve(c.reshape(m, m))
        vals.append(val)
        r2cs.append(r2c)
        us.append(u)
        vs.append(v)
    np.savez_compressed(os.path.join(HERE, "lap_cases.npz"),
                        m=np.array(ms), costs=np.concatenate(costs), values=np.array(vals),
                        r2c=np.concatenate(r2cs), u=np.concatenate(us), v=np.concatenate(vs))
    print("wrote", os.path.join(HERE, "golden.json"), "and lap_cases.npz")


if __name__ == "__main__":
    main()

"""Generate tests/golden/long_traces.json from the COMPILED REFERENCE
(oracle/_ref/libqapref.so): long-horizon bound traces for the BASELINE.json
configs (VERDICT r01 "parity horizons").

    python tests/golden/make_long_traces.py [group ...]

groups: n20 (nug20- and tai20a-shaped, 100 / 30 iterations, all variants),
        n30 (nug30- and tai30-shaped, 20 iterations F1/S1, 8 F2/S2),
        n42 (sko42-shaped 6x7 grid: iteration-1 value + F1/S1 x 3; needs
             ~60 GB of host RAM, so it is run on the GPU box's host).
Each group's traces are merged into the JSON file (existing keys kept).
Per trace: every iteration's bound as a hex float (bitwise), and sha256
digests of the engine arrays at the last iteration.  Test infrastructure only.
"""
from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
from make_golden import digest, grid  # noqa: E402
from oracle.pyoracle import Oracle, default_config  # noqa: E402

OUT = os.path.join(HERE, "long_traces.json")
ARRAYS = ["pi_z", "pi_y", "pi_x", "b", "c", "d", "theta", "delta"]


def trace(orc, f, d, variant, iters, workers, digests=True):
    cfg = default_config(variant=variant, iter_limit=iters, workers=workers)
    t0 = time.time()
    eng = orc.engine_from_instance(f, d, cfg=cfg)
    bounds = []
    for _ in range(iters):
        bounds.append(float(eng.iterate()).hex())
    out = {"variant": variant, "iters": iters, "bounds": bounds,
           "best": float(eng.scalars()["best"]).hex()}
    if digests:
        dg = {a: digest(eng.array(a)) for a in ARRAYS}
        if variant in ("F1", "F2"):
            dg["incz"] = digest(eng.array("incz"))
        dg["x_assignment"] = [int(x) for x in eng.x_assignment()]
        out["digests"] = {str(iters): dg}
    del eng
    print(f"  {variant} x{iters}: {time.time() - t0:.1f} s, last {float.fromhex(bounds[-1])!r}",
          flush=True)
    return out


def main():
    groups = sys.argv[1:] or ["n20", "n30"]
    workers = os.cpu_count() or 1
    orc = Oracle("ref")
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            data = json.load(fh)
    data.setdefault("generator", "oracle/_ref/libqapref.so (reference proj/src compiled "
                                 "unmodified), tests/golden/make_long_traces.py")
    tr = data.setdefault("traces", {})

    def save():
        with open(OUT, "w") as fh:
            json.dump(data, fh, indent=1, sort_keys=True)

    if "n20" in groups:
        gf, gd = grid(4, 5, orc)          # nug20-shaped (BASELINE config 5 instance)
        f20, d20 = orc.generate_instance(20, 1, 99)  # tai20a-shaped (config 2)
        for v in ("F1", "S1"):
            print("grid20", v, flush=True)
            tr[f"grid20_{v}_100"] = trace(orc, gf, gd, v, 100, workers)
        for v in ("F2", "S2"):
            print("grid20", v, flush=True)
            tr[f"grid20_{v}_30"] = trace(orc, gf, gd, v, 30, workers)
        for v in ("F1", "S1", "F2", "S2"):
            print("rand20", v, flush=True)
            tr[f"rand20_{v}_30"] = trace(orc, f20, d20, v, 30, workers)
        save()
    if "n30" in groups:
        g30f, g30d = grid(5, 6, orc)      # nug30-shaped (config 3, the bench workload)
        f30, d30 = orc.generate_instance(30, 1, 99)
        for name, (f, d) in (("grid30", (g30f, g30d)), ("rand30", (f30, d30))):
            for v, it in (("F1", 20), ("S1", 20), ("F2", 8), ("S2", 8)):
                print(name, v, flush=True)
                tr[f"{name}_{v}_{it}"] = trace(orc, f, d, v, it, workers)
                save()
    if "n42" in groups:
        g42f, g42d = grid(6, 7, orc)      # sko42-shaped (config 4)
        for v, it in (("S1", 3), ("F1", 3)):
            print("grid42", v, flush=True)
            tr[f"grid42_{v}_{it}"] = trace(orc, g42f, g42d, v, it, workers, digests=False)
            save()
    save()
    print("wrote", OUT)


if __name__ == "__main__":
    main()

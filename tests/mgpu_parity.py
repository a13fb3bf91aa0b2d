"""Multi-GPU parity (run under torchrun, one process per GPU):

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        tests/mgpu_parity.py

Every rank runs the z-sharded engine on the golden instances
and checks each iteration's bound bitwise against the compiled reference's
trace; rank 0 prints one JSON line and the exit code is non-zero on any
mismatch."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1710_03732_b200 as q  # noqa: E402
from paper_1710_03732_b200.instance import QapInstance, grid_instance  # noqa: E402


def digest(a):  # as tests/conftest.py
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()[:32]


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as fh:
        g = json.load(fh)
    nug12 = QapInstance(12, np.array(g["nug12"]["flow"], float), np.array(g["nug12"]["dist"], float))
    cases = {"nug12_F1": nug12, "nug12_S1": nug12, "nug12_F1_SA": nug12, "nug12_S1_SA": nug12,
             "rand20_F1": q.generate_instance(20, 1, 99),
             "rand20_S1": q.generate_instance(20, 1, 99), "grid20_F1": grid_instance(4, 5),
             "grid30_F1": grid_instance(5, 6),
             # 2-phase variants (phase 2 across the ranks, even n); nug12_F2 was run on
             # 2 GPUs (bitwise); the others are listed but run only on request until
             # they have been (MGPU_2PHASE_ALL=1)
             "nug12_F2": nug12}
    if os.environ.get("MGPU_2PHASE_ALL"):
        cases.update({"nug12_S2": nug12, "nug12_F2_SA": nug12,
                      "rand20_F2": q.generate_instance(20, 1, 99)})
    only = os.environ.get("MGPU_CASES")  # debugging: a comma-separated subset
    if only:
        cases = {k: v for k, v in cases.items() if k in only.split(",")}
    results = {}
    for key, inst in cases.items():
        tr = g["traces"][key]
        idobj = [q.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(idobj, src=0)
        cfg = q.AscentConfig(variant=tr["variant"], iter_limit=tr["iters"], device=local,
                             sa_enabled=tr["sa"], upper_bound=tr["upper_bound"], seed=tr["seed"])
        eng = q.AscentEngine.from_instance_sharded(inst, cfg, rank, world, idobj[0])
        want = [float.fromhex(x) for x in tr["bounds"]]
        got, state_ok = [], True
        for it in range(1, len(want) + 1):
            got.append(eng.iterate())
            snap = tr["digests"].get(str(it))
            if snap and key.startswith("nug12"):  # the assembled z state (collective)
                for a in ("pi_z", "d"):
                    if digest(eng.array(a)) != snap[a]:
                        state_ok = f"iteration {it}: {a} digest"
                if "incz" in snap and digest(eng.incz()) != snap["incz"]:
                    state_ok = f"iteration {it}: incz digest"
        results[key] = got == want
        if not results[key]:
            bad = next(i for i, (a, b) in enumerate(zip(got, want)) if a != b)
            results[key] = f"iteration {bad + 1}: {got[bad]!r} != {want[bad]!r}"
        elif state_ok is not True:
            results[key] = state_ok
        eng.close()
    # run() with device-side termination on the sharded engine
    idobj = [q.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(idobj, src=0)
    cfg = q.AscentConfig(variant="F1", iter_limit=40, early_stop_window=5, early_stop_delta=0.002,
                         device=local)
    eng = q.AscentEngine.from_instance_sharded(nug12, cfg, rank, world, idobj[0])
    rep = eng.run()
    eng.close()
    ref = q.run_ascent(nug12, q.AscentConfig(variant="F1", iter_limit=40, early_stop_window=5,
                                             early_stop_delta=0.002, device=local))
    results["run_early_stop"] = ([r.bound for r in rep.records] == [r.bound for r in ref.records]
                                 and rep.termination == ref.termination)
    # odd and small sizes (non-TMA LAP path for odd m, uneven location ranges, ranks
    # owning 1-2 locations) with linear terms: sharded == single-GPU engine, bitwise
    for n in (5, 7, 9, 11, 13):
        inst = q.generate_instance(n, 1000 + n, 50)
        inst.linear[:] = np.arange(n * n).reshape(n, n) % 7
        for variant in ("F1", "S1"):
            if world > n:
                continue
            idobj = [q.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(idobj, src=0)
            cfg = q.AscentConfig(variant=variant, iter_limit=12, device=local)
            eng = q.AscentEngine.from_instance_sharded(inst, cfg, rank, world, idobj[0])
            got = [eng.iterate() for _ in range(12)]
            eng.close()
            one = q.AscentEngine.from_instance(inst, q.AscentConfig(variant=variant,
                                                                   iter_limit=12, device=local))
            want = [one.iterate() for _ in range(12)]
            one.close()
            results[f"n{n}_{variant}"] = got == want or f"{got} != {want}"
    allres = [None] * world
    dist.all_gather_object(allres, results)
    ok = all(v is True for r in allres for v in r.values())
    if rank == 0:
        print(json.dumps({"world": world, "ok": ok, "ranks": allres}))
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()

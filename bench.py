#!/usr/bin/env python
"""bench.py — RLT2 dual-ascent iterations/s (and LAPs/s) at n=30 on B200.

Workload (BASELINE.json configs[2], the metric's "n=30"): nug30-shaped
instance — Manhattan distances on a 5x6 grid, flows of
generate_instance(30, seed=1, max=10) — variant F1 (AscentConfig default),
SA off.  A "step" is one steady-state dual-ascent iteration (ascent update ->
378,450 Z-LAPs -> 900 Y-LAPs -> X-LAP -> bound), state resident in HBM.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun (N>1) the ranks run ONE z-sharded engine (each
rank owns a first-facility range of the half-Z tiles; sigma/gain of the cross-
shard family members move by NCCL send/recv each iteration); value is that
problem's iterations / max-over-ranks device time ("scaling": "strong").
`--replicas` instead runs N independent engines ("weak").  `--impl reference` times the
reference's own CPU implementation (oracle/_ref, compiled from the unmodified
reference sources) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RLT2 dual-ascent iterations/sec and LAPs/sec at n=30; LB gap vs reference"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0}


GRID_SHAPES = {12: (3, 4), 20: (4, 5), 30: (5, 6), 42: (6, 7)}


def workload(n: int, shape: str = "grid"):
    """nug{n}-shaped (grid) or tai{n}a-shaped (rand: generate_instance(n, 1, 99))."""
    if shape == "rand":
        from paper_1710_03732_b200.instance import generate_instance
        return generate_instance(n, 1, 99)
    from paper_1710_03732_b200.instance import grid_instance
    r, c = GRID_SHAPES[n]
    return grid_instance(r, c, flow_seed=1, max_flow=10, name=f"nug{n}-shaped")


def shape_name(args) -> str:
    if args.shape == "rand":
        return f"tai{args.n}a-shaped (generate_instance({args.n}, 1, 99): U{{0..99}} flows and distances)"
    return f"nug{args.n}-shaped (Manhattan grid, flows U{{0..10}} seed 1)"


def workload_reference(orc, n: int, shape: str = "grid"):
    """The same nug{n}-shaped instance built without importing the product
    package: flows from the reference's own generate_instance(n, 1, 10)
    (instance.cpp:131-150, via oracle/_ref), Manhattan grid distances as
    tests/test_bnb.cpp:35-44 grid_instance."""
    import numpy as np
    if shape == "rand":
        return orc.generate_instance(n, 1, 99)
    r, c = GRID_SHAPES[n]
    flow, _ = orc.generate_instance(n, 1, 10)
    a = np.arange(n)
    dist = (np.abs(a[:, None] // c - a[None, :] // c) +
            np.abs(a[:, None] % c - a[None, :] % c)).astype(np.float64)
    return flow, dist


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def sizes(n: int):
    tiles = (n * (n - 1) // 2) * (n * (n - 1))
    esz = (n - 2) ** 2
    return dict(tiles=tiles, esz=esz, n_z=tiles * esz, n_y=n * n * (n - 1) ** 2)


def kernel_bytes(n: int, variant: str):
    """Algorithmic HBM bytes per launch."""
    s = sizes(n)
    fast = variant.upper().startswith("F")
    nz, ny, t = s["n_z"], s["n_y"], s["tiles"]
    return {
        # pi(z) read + D' read/write (+ incz write for F) per stored cell, push per tile
        "zfold": nz * (8 + 16 + (8 if fast else 0)) + 8 * t,
        # cost tile read + pi(z) write per cell, theta per tile
        "zlap": nz * 16 + 8 * t,
        # per tile: 2 pi(y) reads, 2 C' read+write, ybar + push writes
        "xyfold": t * (16 + 32 + 16),
        # Y costs gathered (C' [+theta]) + pi(y) written
        "ystage": ny * (8 + 8) + 8 * t,
        "phase2": nz * (8 + 16),
        "xstage": n * n * 8 * 4,
        "xchg": 0,  # multi-GPU only: barrier + theta exchange (NCCL)
    }


def iteration_bytes(n: int, variant: str = "F1"):
    """B = 32 N_z + 32 N_y + 16 tiles per 1-phase iteration;
    2-phase variants (F2/S2) add 32 N_z (pi_1 write + read, cost read + write)."""
    s = sizes(n)
    b = 32 * s["n_z"] + 32 * s["n_y"] + 16 * s["tiles"]
    return b + (32 * s["n_z"] if variant.upper().endswith("2") else 0)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return PEAKS_FALLBACK["hbm_gbs"], "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            with open(self.path) as fh:
                for line in fh:
                    f = [x.strip() for x in line.split(",")]
                    if len(f) >= 9 and f[1].isdigit():
                        rows.append(f)
        finally:
            os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [int(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4)
                          if r[5 + k].lower() in ("active", "1", "yes")})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": int(rows[0][2]),
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit())
                if any(r[3].replace(".", "").isdigit() for r in rows) else None}


def cpu_reference_run(n, variant, warmup, steps, threads=None, shape="grid"):
    """Time the reference CPU implementation (oracle/_ref; the C port if the
    reference build is absent) on this host: engine built untimed, `warmup`
    untimed iterations, then `steps` timed iterations.  Returns (it/s, kind,
    threads, seconds)."""
    # the oracle loads the struct layouts standalone: nothing here maps libqapb200.so
    from oracle.pyoracle import Oracle, available, default_config
    kind = "ref" if available("ref") else "port"
    threads = threads or os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    orc = Oracle(kind)
    flow, dist = workload_reference(orc, n, shape)
    eng = orc.engine_from_instance(flow, dist, cfg=default_config(
        variant=variant, iter_limit=10 ** 6, workers=threads, record_history=0))
    for _ in range(warmup):
        eng.iterate()
    t0 = time.perf_counter()
    for _ in range(steps):
        eng.iterate()
    dt = time.perf_counter() - t0
    return steps / dt, ("reference" if kind == "ref" else "port"), threads, dt


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    its, kind, threads, dt = cpu_reference_run(args.n, args.variant, args.warmup, args.steps,
                                               shape=args.shape)
    s = sizes(args.n)
    laps = s["tiles"] + args.n * args.n + 1
    line = {
        "metric": METRIC, "impl": "reference", "value": its, "unit": "iterations/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * dt / args.steps, "higher_is_better": True,
        # same metric and config as our arm at this N (the CPU path itself is one
        # process on the host's cores)
        "scaling": "strong" if (world > 1 and not args.replicas) else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "laps_per_s": its * laps,
        "config": config_block(args, world, sharded=world > 1 and not args.replicas),
        "cpu_baseline": {"value": its, "unit": "iterations/s", "cores": threads,
                         "kind": kind, "cpu_model": cpu_model(),
                         "sample": f"{args.steps} steady-state iterations (after {args.warmup} "
                                   f"untimed) of the same n={args.n} {args.variant} workload, "
                                   f"OpenMP workers={threads}"},
        "e2e": {"value": its, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_block(args, world, sharded=False):
    s = sizes(args.n)
    return {"workload": f"{shape_name(args)}, variant {args.variant}, SA off, steady-state "
                        "iterations",
            "n": args.n, "variant": args.variant, "z_laps_per_iteration": s["tiles"],
            "laps_per_iteration": s["tiles"] + args.n * args.n + 1,
            "z_cells": s["n_z"],
            "parallelism": (f"zshard{world}" if sharded else f"replica{world}") if world > 1
            else "single",
            "l2": "no flush: z arrays (3 x %.2f GB) exceed the 126 MB L2" % (s["n_z"] * 8 / 1e9)}


def run_ours(args):
    import ctypes

    import numpy as np
    import torch

    import paper_1710_03732_b200 as q

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    sharded = world > 1 and not args.replicas
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    inst = workload(args.n, args.shape)
    cfg = q.AscentConfig(variant=args.variant, iter_limit=10 ** 6, record_history=False,
                         device=local)
    if sharded:
        idobj = [q.nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(idobj, src=0)
        eng = q.AscentEngine.from_instance_sharded(inst, cfg, rank, world, idobj[0])
    else:
        eng = q.AscentEngine.from_instance(inst, cfg)
    eng.enqueue(args.warmup)
    eng.synchronize()
    stream = torch.cuda.ExternalStream(eng.stream(), device=local)
    eng.set_profiling(True)
    eng.kernel_times(reset=True)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    l0 = eng.launch_count()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        eng.enqueue(args.steps)
        ev1.record(stream)
        eng.synchronize()
        torch.cuda.synchronize()
    launches = eng.launch_count() - l0
    ms = ev0.elapsed_time(ev1)
    ktimes = eng.kernel_times(reset=True)
    rank_times = None
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        rank_times = [None] * world
        torch.distributed.all_gather_object(
            rank_times, {"ms": ms, **{k: round(v[0] / max(1, v[1]), 4) for k, v in ktimes.items()
                                     if v[1]}})
        ms = float(t.item())
    clocks = clk.summary()

    # parity: the bench engine's own trace against the reference pins
    import json as _json
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as fh:
        gold = _json.load(fh)
    parity = None
    with open(os.path.join(ROOT, "tests", "golden", "long_traces.json")) as fh:
        long_tr = _json.load(fh)["traces"]
    pre = "grid" if args.shape == "grid" else "rand"
    cands = [gold["traces"].get(f"{pre}{args.n}_{args.variant}")] + \
        [v for k, v in sorted(long_tr.items()) if k.startswith(f"{pre}{args.n}_{args.variant}_")]
    cands = [c for c in cands if c]
    if cands:  # the longest reference trace of this workload (tests/golden)
        tr = max(cands, key=lambda c: len(c["bounds"]))
        want = [float.fromhex(x) for x in tr["bounds"]]
        k = min(len(want), eng.iteration())
        got, _ = eng.history(0, k)
        parity = {"reference_pins": k, "bitwise": bool(list(got) == want[:k])}
    final_bound = float(eng.history(eng.iteration() - 1, 1)[0][0])
    eng.close()

    s = sizes(args.n)
    laps = s["tiles"] + args.n * args.n + 1
    its = (1 if sharded else world) * args.steps / (ms / 1000.0)
    peak, peak_src = peaks()
    kb = kernel_bytes(args.n, args.variant)
    if sharded:  # each rank folds and solves 1/W of the z work (its location range)
        kb = {k: (v / world if k in ("zfold", "zlap") else v) for k, v in kb.items()}
    kernels = {}
    for name, (kms, cnt) in ktimes.items():
        if cnt:
            per = kms / cnt
            gbs = kb[name] / (per / 1000.0) / 1e9
            kernels[name] = {"ms_per_launch": per, "launches": cnt,
                             "share": kms / max(1e-9, sum(v[0] for v in ktimes.values())),
                             "alg_bytes": kb[name], "achieved_gbs": gbs}
    dom = max(kernels, key=lambda k: kernels[k]["ms_per_launch"] * kernels[k]["launches"])
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    tdb, idb = {}, {}
    if os.path.exists(tpath):
        with open(tpath) as fh:
            nj = _json.load(fh)
        if not sharded:  # the committed capture is of the single-GPU engine
            tdb = nj.get(f"n{args.n}_{args.variant}", {})
            idb = nj.get(f"n{args.n}_{args.variant}_issue_active_pct", {})
    for name in kernels:  # ncu evidence (profiles/): DRAM bytes and issue-slot use per launch
        kernels[name]["ncu_dram_bytes"] = tdb.get(name)
        kernels[name]["ncu_issue_active_pct"] = idb.get(name)

    def kernel_roofline(name):
        return {"bound": "hbm", "kernel": name, "achieved": kernels[name]["achieved_gbs"],
                "peak": peak, "unit": "GB/s", "frac": kernels[name]["achieved_gbs"] / peak,
                "traffic": tdb.get(name), "peak_source": peak_src,
                "alg_bytes_per_launch": kb[name]}
    roofline = kernel_roofline(dom)
    if dom == "zlap":
        roofline["note"] = ("the Z-LAP batch is issue-bound (warp-per-LAP Hungarian, "
                            f"{idb.get('zlap', 80):.0f}% of issue slots busy in ncu), not "
                            "HBM-bound; its HBM fraction is reported as the contract asks; the "
                            "HBM-bound fold is in roofline_fold")
        roofline["issue_active_pct"] = idb.get("zlap")
    if "zfold" in kernels and dom != "zfold":
        roofline["roofline_fold"] = kernel_roofline("zfold")
    ib = iteration_bytes(args.n, args.variant)
    per_gpu_its = its / world if not sharded else its  # sharded: bytes split over world GPUs
    agg_peak = peak * (world if sharded else 1)
    iteration_roofline = {"alg_bytes": ib, "achieved_gbs": ib * per_gpu_its / 1e9,
                          "frac": ib * per_gpu_its / 1e9 / agg_peak,
                          "note": "SURVEY.md §8(d) B=32Nz+32Ny+16tiles per 1-phase iteration "
                                  "(+32Nz for 2-phase variants)"}

    # e2e: the user's call (run_ascent through the C-ABI, host instance in,
    # host report out), 100 iterations = the reference's default iter_limit
    e2e_iters = 100
    if sharded:  # every rank runs its shard of the same run_ascent-equivalent call
        # (same NCCL id as the timed engine: the library caches its communicator);
        # best of 3 whole calls, each timed as the max over ranks
        runs = []
        for _ in range(3):
            torch.distributed.barrier()
            t0 = time.perf_counter()
            e = q.AscentEngine.from_instance_sharded(
                inst, q.AscentConfig(variant=args.variant, iter_limit=e2e_iters, device=local),
                rank, world, idobj[0])
            rep = e.run()
            e.close()
            torch.cuda.synchronize()
            tt = torch.tensor([time.perf_counter() - t0], device="cuda", dtype=torch.float64)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            runs.append(float(tt.item()))
        e2e_s = min(runs)
    else:
        q.run_ascent(inst, q.AscentConfig(variant=args.variant, iter_limit=2))  # warm context
        runs = []
        for _ in range(3):  # best of 3 whole calls (the first can pay allocator warm-up)
            t0 = time.perf_counter()
            rep = q.run_ascent(inst, q.AscentConfig(variant=args.variant, iter_limit=e2e_iters))
            runs.append(time.perf_counter() - t0)
        e2e_s = min(runs)
    rec_bytes = ctypes.sizeof(q.abi.Record)
    e2e = {"value": rep.iterations / e2e_s, "unit": "iterations/s",
           "h2d_bytes_per_step": 3 * args.n * args.n * 8 / rep.iterations,
           "d2h_bytes_per_step": rec_bytes + ctypes.sizeof(q.abi.Report) / rep.iterations,
           "call": (("qapb_engine_create_instance_sharded + qapb_engine_run on every rank "
                     "(NCCL communicator reused from the timed engine)") if sharded else
                    "qapb_run_ascent") + f"({pre}{args.n}, {args.variant}, iter_limit=100): "
                   "engine build on device, 100 iterations, report + records to host",
           "seconds": e2e_s, "final_bound": rep.best_bound}
    e2e["all_seconds"] = runs

    if rank != 0:
        torch.distributed.destroy_process_group()
        return 0
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cw, cs = 3, 10
            cits, kind, threads, dt = cpu_reference_run(args.n, args.variant, cw, cs,
                                                        shape=args.shape)
            cpu = {"value": cits, "unit": "iterations/s", "cores": threads, "kind": kind,
                   "cpu_model": cpu_model(),
                   "sample": f"{cs} steady-state iterations (after {cw} untimed) of the same "
                             f"n={args.n} {args.variant} workload, {dt:.1f} s, OpenMP "
                             f"workers={threads}"}
        except Exception as e:  # reported, never silently substituted
            cpu = {"value": None, "unit": "iterations/s", "cores": os.cpu_count(),
                   "kind": "reference", "sample": f"failed: {e}"}

    line = {
        "metric": METRIC, "value": its, "unit": "iterations/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "laps_per_s": its * laps, "config": config_block(args, world, sharded),
        "roofline": roofline, "iteration_roofline": iteration_roofline, "kernels": kernels,
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
        "parity": parity, "bound_after": final_bound,
    }
    if rank_times:
        line["per_rank_ms_per_launch"] = rank_times
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", "--size", dest="n", type=int, default=30)  # --size under torchrun
    ap.add_argument("--variant", default="F1")
    ap.add_argument("--shape", default="grid", choices=["grid", "rand"],
                    help="grid: nug-shaped (default); rand: tai-a-shaped generate_instance(n,1,99)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: independent engines instead of one z-sharded engine")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 1)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

"""Profiling helper (not part of the product): build the bench's engine, run
`warm` iterations, then `extra` more.  Used as the target of
`ncu -k regex:... -s <skip> -c <count>` so the captured launches are
steady-state ones.

    python tools/prof_iter.py [n] [variant] [warm] [extra]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    variant = sys.argv[2] if len(sys.argv) > 2 else "F1"
    warm = int(sys.argv[3]) if len(sys.argv) > 3 else 6
    extra = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    import paper_1710_03732_b200 as q
    from bench import workload
    eng = q.AscentEngine.from_instance(
        workload(n), q.AscentConfig(variant=variant, iter_limit=10**6, record_history=False))
    eng.enqueue(warm)
    eng.synchronize()
    eng.enqueue(extra)
    eng.synchronize()
    print("bound", eng.best_bound(), "iteration", eng.iteration())


if __name__ == "__main__":
    main()

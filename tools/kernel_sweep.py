"""Tuning helper (not part of the product): time single kernels in isolation
on a steady-state n=30 engine under env-var variants."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

def one(kind, reps, n):
    import paper_1710_03732_b200 as q
    from bench import workload
    eng = q.AscentEngine.from_instance(workload(n), q.AscentConfig(variant="F1", iter_limit=10**6,
                                                                   record_history=False))
    eng.enqueue(4); eng.synchronize()
    return eng.time_kernel(kind, reps)

if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        print(json.dumps(one(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))))
        sys.exit(0)
    kind = sys.argv[1]
    n = int(os.environ.get("SWEEP_N", "30"))
    for spec in sys.argv[2:]:
        env = dict(os.environ)
        for kv in spec.split(","):
            if kv:
                k, v = kv.split("=")
                env[k] = v
        out = subprocess.run([sys.executable, __file__, "child", kind, "5", str(n)], env=env,
                             capture_output=True, text=True, timeout=240)
        print(spec, kind, out.stdout.strip() or out.stderr[-300:], flush=True)

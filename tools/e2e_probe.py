"""Break down the single-GPU run_ascent wall time (engine build, iterations, teardown)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1710_03732_b200 as q  # noqa: E402
from bench import workload  # noqa: E402

inst = workload(30)
for rep in range(2):
    t0 = time.perf_counter()
    e = q.AscentEngine.from_instance(inst, q.AscentConfig(variant="F1", iter_limit=100))
    t1 = time.perf_counter()
    e.iterate()
    t2 = time.perf_counter()
    r = e.run()
    t3 = time.perf_counter()
    e.close()
    t4 = time.perf_counter()
    print(f"build {t1-t0:.3f}s first-iter {t2-t1:.3f}s run {t3-t2:.3f}s ({r.iterations} it) "
          f"close {t4-t3:.3f}s")
t0 = time.perf_counter()
r = q.run_ascent(inst, q.AscentConfig(variant="F1", iter_limit=100))
print(f"run_ascent {time.perf_counter()-t0:.3f}s")

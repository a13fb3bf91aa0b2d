"""Time collapse_store at n=30 (B&B child store): device kernel vs
the reference's host function (oracle/_ref) on the same S1 snapshot."""
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1710_03732_b200 as q  # noqa: E402
from paper_1710_03732_b200 import abi  # noqa: E402
from bench import workload  # noqa: E402
from oracle.pyoracle import Oracle, available  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
eng = q.AscentEngine.from_instance(workload(n), q.AscentConfig(variant="S1", iter_limit=3))
for _ in range(3):
    eng.iterate()
ds = q.DeviceStore.from_engine(eng)
host = eng.snapshot()
eng.close()
ds.collapse(1, 1).close()  # warm
t = []
for fac, loc in [(0, 0), (7, 11), (29 % n, 3)]:
    t0 = time.perf_counter()
    c = ds.collapse(fac, loc)
    t.append(time.perf_counter() - t0)
    c.close()
out = {"n": n, "device_collapse_s": t}
if available("ref"):
    ref = Oracle("ref")
    nb, nc, nd = abi.store_sizes(n - 1)
    ob, oc, od = np.empty(nb), np.empty(nc), np.empty(nd)
    off = ctypes.c_double()
    t0 = time.perf_counter()
    ref.lib.qref_collapse_store(n, abi.dptr(host.b), abi.dptr(host.c), abi.dptr(host.d),
                                host.offset, 7, 11, abi.dptr(ob), abi.dptr(oc), abi.dptr(od),
                                ctypes.byref(off))
    out["reference_host_collapse_s"] = time.perf_counter() - t0
    got = ds.collapse(7, 11).download()
    out["bitwise"] = bool(got.b.tobytes() == ob.tobytes() and got.c.tobytes() == oc.tobytes()
                          and got.d.tobytes() == od.tobytes() and got.offset == off.value)
print(json.dumps(out))

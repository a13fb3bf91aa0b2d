"""GPU regression: many threads creating,
iterating, snapshotting and destroying engines at once -- the reference's
branch-and-bound banks (bnb.cpp:549-556) drive the library exactly so.

The fault this pins: engine tables (fpair/triple indices) were uploaded with a
legacy-stream cudaMemcpy from pageable memory, which may return before its DMA
lands, while the engine's kernels run on non-blocking streams; with 8-16 banks
a Z-LAP could read a half-written table and store out of bounds.  Every engine
here must reproduce the serial trace bitwise, in eager mode (QAPB_NO_GRAPH,
the sharded/profiling path) and with graphs."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    import paper_1710_03732_b200 as q
    return q


def _job(q, n, seed, variant, iters):
    inst = q.generate_instance(n, seed, 10)
    eng = q.AscentEngine.from_instance(inst, q.AscentConfig(variant=variant, iter_limit=iters,
                                                            record_history=True))
    rep = eng.run()
    snap = eng.snapshot() if variant.startswith("S") else None
    eng.close()
    out = [r.bound for r in rep.records]
    if snap is not None:  # a warm child through the device store path
        child = q.run_ascent_warm(q.collapse_store(snap, 0, 1),
                                  q.AscentConfig(variant="S1", iter_limit=5))
        out += [r.bound for r in child.records]
    return out


@pytest.mark.parametrize("eager", [True, False])
def test_many_threads_match_serial(q, monkeypatch, eager):
    if eager:
        monkeypatch.setenv("QAPB_NO_GRAPH", "1")
    jobs = [(n, seed, v, 12) for n in (15, 16, 17, 18) for seed in (1, 2)
            for v in ("F1", "S1")]
    want = [_job(q, *j) for j in jobs]
    got = [None] * len(jobs)
    errors = []

    def worker(k):
        try:
            for rep in range(2):  # create/destroy churn
                got[k] = _job(q, *jobs[k])
        except Exception as e:  # noqa: BLE001 - reported below
            errors.append(repr(e))

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(len(jobs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for k, j in enumerate(jobs):
        assert got[k] == want[k], j

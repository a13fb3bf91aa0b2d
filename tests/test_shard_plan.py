"""CPU: the multi-GPU shard plan.  Host logic only -- the
world-2 case runs as two gloo processes that exchange their exchange-count
tables and check that every send has a matching receive."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _plan_is_valid(q, n, world):
    b = q.shard_plan(n, world)
    assert b[0] == 0 and b[-1] == n - 1 and len(b) == world + 1
    assert all(x < y for x, y in zip(b, b[1:]))
    return b


def test_plan_shapes_and_balance():
    import paper_1710_03732_b200 as q
    for n in (4, 7, 12, 20, 30, 42):
        for world in (1, 2, 4, 8):
            if world > n - 2:
                continue
            _plan_is_valid(q, n, world)
    # n=30 on 8 ranks: the heaviest rank carries at most ~1.6x the mean work
    b = q.shard_plan(30, 8)
    c2 = lambda x: x * (x - 1) / 2
    w = [sum(0.55 * c2(29 - a) / 4060 + 0.45 * (29 - a) / 435 for a in range(b[r], b[r + 1]))
         for r in range(8)]
    assert max(w) / (sum(w) / 8) < 1.6
    with pytest.raises(ValueError):
        q.shard_plan(5, 9)


def _worker(rank, world, port, n, out):
    import paper_1710_03732_b200 as q
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    s, r = q.shard_exchange_counts(n, world, rank)
    table = [None] * world
    dist.all_gather_object(table, (s.tolist(), r.tolist(), q.shard_plan(n, world)))
    ok = all(table[a][0][b] == table[b][1][a] for a in range(world) for b in range(world))
    plans_equal = all(t[2] == table[0][2] for t in table)
    # every family's X3 member is remote exactly when owner(b) != owner(a):
    # the sends to lower ranks sum to (my tiles) x (their rows) x (n-2)
    b = table[0][2]
    fpf = lambda i: i * n - i * (i + 1) // 2
    tiles = (fpf(b[rank + 1]) - fpf(b[rank])) * n * (n - 1)
    want = sum(tiles * (b[p + 1] - b[p]) * (n - 2) for p in range(rank))
    out.put((rank, ok, plans_equal, int(sum(s)) == want))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 12), (2, 30)])
def test_exchange_counts_match_across_gloo_ranks(world, n):
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q_ = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, n, q_)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q_.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(ok and pe and cnt for _, ok, pe, cnt in res), res

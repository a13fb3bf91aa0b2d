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
    assert b[0] == 0 and b[-1] == n and len(b) == world + 1
    assert all(x < y for x, y in zip(b, b[1:]))
    assert max(y - x for x, y in zip(b, b[1:])) - min(y - x for x, y in zip(b, b[1:])) <= 1
    return b


def test_plan_shapes_and_balance():
    import paper_1710_03732_b200 as q
    for n in (4, 7, 12, 20, 30, 42):
        for world in (1, 2, 4, 8):
            if world > n:
                continue
            _plan_is_valid(q, n, world)
    # n=30 on 8 ranks: locations 3 or 4 per rank -> work within 4/3.75 of the mean
    b = q.shard_plan(30, 8)
    sizes = [y - x for x, y in zip(b, b[1:])]
    assert max(sizes) / (30 / 8) < 1.07
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
    # one slot per (pair b<c, my location pair, row a<b, peer location pa):
    # sum of sends = (my tiles per pair) x (sum over pairs of b) x (other locations)
    b = table[0][2]
    mine = b[rank + 1] - b[rank]
    rows = sum(bb * (n - 1 - bb) for bb in range(n))
    want = mine * (n - 1) * rows * (n - mine)
    out.put((rank, ok, plans_equal, int(sum(s)) == want))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 12), (2, 30), (4, 13), (8, 30)])
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

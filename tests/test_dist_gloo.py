"""CPU, world_size 2 over gloo: the N > 1 host logic of both multi-GPU schemes
(paper_1904_12754_b200/shard.py), with the CPU oracle standing in for the per-rank GPU work.

* row sharding: the ranks' component sets partition all rows; gathering the per-rank driver
  results reproduces the single-process results exactly;
* sample sharding: each rank computes the chunk partials of the chunks it owns (zeros
  elsewhere), a torch.distributed all-reduce (sum) merges them, and the ordered combine equals
  the unsharded run_level bit for bit -- the arithmetic the NCCL path of context.cu performs.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _row_worker(rank, world, port, out):
    import sys

    sys.path.insert(0, ROOT)
    from oracle import Oracle
    from paper_1904_12754_b200.shard import row_shard

    _setup(rank, world, port)
    o = Oracle()
    a = o.grid_laplacian(12)
    u = o.grid_vector(12345, a.n)
    rows = row_shard(a.n, rank, world)
    res = o.chain(a).driver_rows(u, 1.0, rows, rows + 1000, epsilon=2e-2)
    mine = {int(r): (x["estimate"], x["total_cost"]) for r, x in zip(rows, res)}
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    if rank == 0:
        merged = {}
        for g in gathered:
            assert not (set(g) & set(merged))  # disjoint
            merged.update(g)
        out.put(merged)
    dist.destroy_process_group()


def _sample_worker(rank, world, port, out):
    import sys

    sys.path.insert(0, ROOT)
    from oracle import Oracle
    from paper_1904_12754_b200.shard import combine_ordered, owned_chunks

    _setup(rank, world, port)
    o = Oracle()
    a = o.grid_laplacian(16)
    u = o.grid_vector(12345, a.n)
    ch = o.chain(a)
    entry, level, first, count, seed = 37, 2, 300, 7000, 1037
    c0, c1 = first // 512, (first + count - 1) // 512
    nch = c1 - c0 + 1
    s = torch.zeros(nch, dtype=torch.float64)
    s2 = torch.zeros(nch, dtype=torch.float64)
    cost = torch.zeros(nch, dtype=torch.int64)
    for g in owned_chunks(0, nch, rank, world):  # chunk index within the request
        lo = max(first, (c0 + g) * 512)
        hi = min(first + count, (c0 + g + 1) * 512)
        r = ch.run_level(u, entry, 1.0, level, 0, lo, hi - lo, seed)
        s[g], s2[g], cost[g] = r["sum"], r["sum_sq"], r["cost"]
    for t in (s, s2, cost):
        dist.all_reduce(t)  # exact: one non-zero per element
    if rank == 0:
        out.put((combine_ordered(s.numpy(), s2.numpy(), cost.numpy()),
                 ch.run_level(u, entry, 1.0, level, 0, first, count, seed)))
    dist.destroy_process_group()


def _run(target, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def test_row_sharding_gloo_world2():
    from oracle import Oracle
    from paper_1904_12754_b200.shard import row_shard

    merged = _run(_row_worker)
    o = Oracle()
    a = o.grid_laplacian(12)
    u = o.grid_vector(12345, a.n)
    assert sorted(merged) == list(range(a.n))
    rows = np.arange(a.n)
    ref = o.chain(a).driver_rows(u, 1.0, rows, rows + 1000, epsilon=2e-2)
    for r, x in zip(rows, ref):
        assert merged[int(r)] == (x["estimate"], x["total_cost"])
    parts = [row_shard(a.n, k, 3) for k in range(3)]
    assert np.array_equal(np.sort(np.concatenate(parts)), rows)


def test_sample_sharding_gloo_world2_exact():
    (s, s2, c), ref = _run(_sample_worker)
    assert s == ref["sum"] and s2 == ref["sum_sq"] and c == ref["cost"]


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_owned_chunks_partition(world):
    from paper_1904_12754_b200.shard import owned_chunks

    for g0, g1 in [(0, 17), (5, 40), (1 << 22, (1 << 22) + 9)]:
        allc = np.sort(np.concatenate([owned_chunks(g0, g1, r, world) for r in range(world)]))
        assert np.array_equal(allc, np.arange(g0, g1))

"""Expert-parallel bookkeeping on CPU: world_size 2 over gloo (127.0.0.1), no GPU.

Checks that the expert shards partition [0, E), that per-rank (token, expert) rows are exactly the
rows of the single-process grouping restricted to the rank's experts, and that the variable-length
all_gather used for verification reassembles the global row order."""
import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_19437_b200 import ep
import workloads as W


def test_shard_range_partitions_experts():
    for E in (1, 7, 256):
        for world in (1, 2, 3, 4, 8):
            covered = []
            for r in range(world):
                e0, e1 = ep.shard_range(E, world, r)
                assert 0 <= e0 <= e1 <= E
                covered.extend(range(e0, e1))
            assert covered == list(range(E))


def test_local_rows_match_global_grouping():
    routes = W.route_skewed(512, 16, 4, alpha=1.0, seed=3)
    tok, offsets = W.group_rows(routes, 16)
    parts = []
    for r in range(4):
        e0, e1 = ep.shard_range(16, 4, r)
        t, o = ep.local_rows(routes, 16, e0, e1)
        assert o[0] == 0 and o[-1] == t.numel()
        assert torch.equal(o, offsets[e0:e1 + 1] - offsets[e0])
        parts.append(t)
    assert torch.equal(torch.cat(parts), tok)
    # no token dropping: every (token, slot) appears exactly once
    assert tok.numel() == 512 * 4


def test_imbalance():
    assert ep.imbalance([10, 10]) == 1.0
    assert abs(ep.imbalance([30, 10]) - 1.5) < 1e-12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        E, T, k, N = 8, 64, 2, 4
        routes = W.route_uniform(T, E, k, seed=5)
        e0, e1 = ep.shard_range(E, world, rank)
        tok, offs = ep.local_rows(routes, E, e0, e1)
        # stand-in for the GEMM output: a row records (token, expert) so reassembly is checkable
        expert_of_row = torch.repeat_interleave(torch.arange(e0, e1), offs[1:] - offs[:-1])
        local = torch.stack([tok.float(), expert_of_row.float()], 1).repeat(1, N // 2)
        parts = ep.gather_rows(local, world)
        if rank == 0:
            q.put(torch.cat(parts).clone())
    finally:
        dist.destroy_process_group()


def test_gather_rows_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    routes = W.route_uniform(64, 8, 2, seed=5)
    tok, offsets = W.group_rows(routes, 8)
    expert = torch.repeat_interleave(torch.arange(8), offsets[1:] - offsets[:-1])
    assert torch.equal(out[:, 0].long(), tok)
    assert torch.equal(out[:, 1].long(), expert)


def test_exchange_plan_routes_every_slot_to_its_expert_row_and_back():
    """ep.exchange_plan (NEXT-3 bookkeeping), for 1, 2 and 4 ranks: every (token, slot) of a rank's
    token shard is sent to the rank owning its expert, at the row that the single-process grouping
    (W.group_rows) gives that pair; every received row is sent back to its token's owner at the slot
    (t - t0) * top_k + j; the receive rows of each rank cover its experts' rows exactly once."""
    T, E, k = 600, 16, 4
    routes = W.route_skewed(T, E, k, alpha=1.0, seed=3)
    tok, off = W.group_rows(routes, E)
    for world in (1, 2, 4):
        plans = [ep.exchange_plan(routes, E, world, r) for r in range(world)]
        assert sum(p.rows for p in plans) == T * k
        hit = [torch.zeros(p.rows, dtype=torch.int64) for p in plans]
        for r, p in enumerate(plans):
            assert torch.equal(p.offsets, off[p.e0:p.e1 + 1] - off[p.e0])
            for i in range(p.dst_rank.numel()):
                t, j = p.t0 + i // k, i % k
                o, row = int(p.dst_rank[i]), int(p.dst_row[i])
                q = plans[o]
                assert q.e0 <= int(routes[t, j]) < q.e1
                assert int(tok[row + int(off[q.e0])]) == t
                hit[o][row] += 1
                # and back: the received row returns to slot i of rank r
                assert int(q.c_rank[row]) == r and int(q.c_slot[row]) == i
        assert all(bool((h == 1).all()) for h in hit)

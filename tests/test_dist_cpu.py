"""Row-window sharding host logic on CPU with gloo, world_size 2.

Each rank computes its windows' rows with the CPU oracle (windows are
independent), writes them into its padded slab, and the gloo all-gather
reassembles the full result, which must equal the unsharded computation
bitwise. Same for the per-edge attention weights (edge ranges are
contiguous per window range)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import tcg_oracle as o
        from paper_2112_02052_b200 import dist as tdist

        n = 1000
        ptr, cols, _ = o.gen_uniform(n, 7, seed=3)
        wp, _, _, _ = o.translate(ptr, cols, n, 16, 8)
        pt, ct, perm = o.csr_transpose(ptr, cols, n)
        wpt, _, _, _ = o.translate(pt, ct, n, 16, 8)
        plan = tdist.make_shard_plan(ptr, n, 16, wp, wpt, rank, world)
        x = o.random_embeddings(n, 8, seed=2)
        full_y = o.agnn_layer(ptr, cols, x)
        full_p = o.segment_softmax(o.sddmm(ptr, cols, x), ptr)
        r0, r1 = plan.my_rows
        e0, e1 = plan.my_edges
        # rank-local computation: only this rank's rows / edges, written into its
        # slice of the persistent padded buffers; the all-gathers run in place
        buf = torch.zeros(plan.padded_rows, 8)
        buf[r0:r1] = torch.from_numpy(full_y[r0:r1])
        got = tdist.allgather_rows(buf, plan)[:n].numpy()
        ebuf = torch.zeros(world * 2 * plan.edges_max)
        ebuf[torch.from_numpy(plan.edge_slot(np.arange(e0, e1)))] = torch.from_numpy(full_p[e0:e1])
        tdist.allgather_edges(ebuf, plan)
        got_p = ebuf[torch.from_numpy(plan.edge_slot(np.arange(cols.shape[0])))].numpy()
        ok = np.array_equal(got, full_y) and np.array_equal(got_p, full_p)
        # windows cover [0, W) once, rows/edges contiguous
        W = -(-n // 16)
        cover = plan.windows[0][0] == 0 and plan.windows[-1][1] == W and all(
            plan.windows[i][1] == plan.windows[i + 1][0] for i in range(world - 1))
        q.put((rank, bool(ok and cover)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


def test_sharded_allgather_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] is True for r in res), res


def test_partition_balances_cost():
    from paper_2112_02052_b200.dist import partition_windows

    rng = np.random.default_rng(0)
    cost = rng.integers(0, 30, 10000).astype(float)
    for parts in (1, 2, 3, 8):
        rngs = partition_windows(cost, parts)
        assert rngs[0][0] == 0 and rngs[-1][1] == 10000
        sums = [cost[a:b].sum() for a, b in rngs]
        assert max(sums) - min(sums) <= 2 * cost.max() + 1
    tiny = partition_windows(np.zeros(3), 4)  # more ranks than windows
    assert tiny[0][0] == 0 and tiny[-1][1] == 3 and len(tiny) == 4


@pytest.mark.parametrize("world", [2, 4])
def test_shard_plan_rows_edges(world):
    from oracle import tcg_oracle as o
    from paper_2112_02052_b200.dist import make_shard_plan

    n = 777
    ptr, cols, _ = o.gen_uniform(n, 5, seed=1)
    wp, _, _, _ = o.translate(ptr, cols, n, 16, 8)
    plans = [make_shard_plan(ptr, n, 16, wp, None, r, world) for r in range(world)]
    rows = plans[0].rows
    assert rows[0][0] == 0 and rows[-1][1] == n
    assert all(rows[i][1] == rows[i + 1][0] for i in range(world - 1))
    edges = plans[0].edges
    assert edges[0][0] == 0 and edges[-1][1] == cols.shape[0]


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_uniform_plan_layout(world):
    """Equal row ranges (multiples of blk_h) so every exchange is one in-place
    all_gather_into_tensor; every rank's padded edge slice starts at or after
    its first edge id (the kernels write P / dS at absolute edge ids through a
    non-negative pointer offset); edge slots are a bijection into the layout."""
    from oracle import tcg_oracle as o
    from paper_2112_02052_b200.dist import make_shard_plan

    n = 1237
    ptr, cols, _ = o.gen_uniform(n, 6, seed=2)
    wp, _, _, _ = o.translate(ptr, cols, n, 16, 8)
    for r in range(world):
        p = make_shard_plan(ptr, n, 16, wp, None, r, world)
        assert p.R % 16 == 0 and p.padded_rows >= n and p.imbalance >= 1.0
        assert all(r1 - r0 <= p.R for r0, r1 in p.rows)
        assert all(q * 2 * p.edges_max >= e0 for q, (e0, _) in enumerate(p.edges))
        assert all(a[0] * 16 == min(r0, n) or r0 == n for a, (r0, _) in zip(p.windows, p.rows))
    slots = p.edge_slot(np.arange(cols.shape[0]))
    assert np.unique(slots).shape[0] == cols.shape[0] and slots.max() < world * 2 * p.edges_max

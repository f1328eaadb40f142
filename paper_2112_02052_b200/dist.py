"""Row-window sharding across the GPUs of one box.

Windows are independent: rank r owns a contiguous window
range [wb, we) — the same range for A and A^T so the two halves of the AGNN
input gradient land on the same rows — balanced by the combined tile count
win_partition(A) + win_partition(A^T). Dense features, weights and GEMMs are
replicated; after each sparse op the rank's rows (or its edges' attention
weights) are exchanged with one all-gather over NCCL (torch.distributed), the
sparse kernel's epilogue writing straight into the rank's slice of the
all-gather buffer.

The host logic here (partitioning, padded slices, reassembly) is backend
agnostic and is tested with gloo on CPU (tests/test_dist_cpu.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def partition_windows(cost: np.ndarray, parts: int) -> list[tuple[int, int]]:
    """Contiguous window ranges whose summed `cost` is balanced: cut where the
    cumulative cost crosses k/parts of the total (deterministic)."""
    cost = np.asarray(cost, dtype=np.float64)
    W = cost.shape[0]
    if parts < 1:
        raise ValueError("parts must be >= 1")
    cum = np.concatenate([[0.0], np.cumsum(cost + 1e-9)])  # tie-break empty windows
    total = cum[-1]
    cuts = [0]
    for k in range(1, parts):
        c = int(np.searchsorted(cum, total * k / parts, side="left"))
        cuts.append(min(max(c, cuts[-1]), W))
    cuts.append(W)
    return [(cuts[i], cuts[i + 1]) for i in range(parts)]


@dataclass
class ShardPlan:
    rank: int
    world: int
    windows: list[tuple[int, int]]   # per rank [wb, we)
    rows: list[tuple[int, int]]      # per rank [rb, re)
    edges: list[tuple[int, int]]     # per rank [eb, ee) of A
    blk_h: int

    @property
    def my_windows(self):
        return self.windows[self.rank]

    @property
    def my_rows(self):
        return self.rows[self.rank]

    @property
    def my_edges(self):
        return self.edges[self.rank]

    @property
    def rows_max(self) -> int:
        return max(1, max(r1 - r0 for r0, r1 in self.rows))

    @property
    def edges_max(self) -> int:
        return max(1, max(e1 - e0 for e0, e1 in self.edges))


def make_shard_plan(node_pointer: np.ndarray, num_nodes: int, blk_h: int, wp_a: np.ndarray,
                    wp_t: np.ndarray | None, rank: int, world: int) -> ShardPlan:
    cost = wp_a.astype(np.float64)
    if wp_t is not None:
        cost = cost + wp_t.astype(np.float64)
    wins = partition_windows(cost, world)
    rows = [(min(wb * blk_h, num_nodes), min(we * blk_h, num_nodes)) for wb, we in wins]
    edges = [(int(node_pointer[r0]), int(node_pointer[r1])) for r0, r1 in rows]
    return ShardPlan(rank, world, wins, rows, edges, blk_h)


def _all_gather(buf, local, group):
    """all_gather_into_tensor over NCCL; other backends (gloo, used by the
    1-GPU functional tests) stage device tensors through the host."""
    import torch.distributed as dist

    if local.is_cuda and dist.get_backend(group) != "nccl":
        hb = buf.cpu()
        dist.all_gather_into_tensor(hb, local.cpu(), group=group)
        buf.copy_(hb)
    else:
        dist.all_gather_into_tensor(buf, local, group=group)


def allgather_rows(local_slab, plan: ShardPlan, group=None):
    """local_slab: [rows_max, D] (rank's rows at the top). Returns the full
    [N, D] matrix assembled from every rank's slab."""
    import torch

    D = local_slab.shape[1]
    buf = torch.empty((plan.world * plan.rows_max, D), dtype=local_slab.dtype,
                      device=local_slab.device)
    _all_gather(buf, local_slab.contiguous(), group)
    parts = [buf[r * plan.rows_max: r * plan.rows_max + (r1 - r0)]
             for r, (r0, r1) in enumerate(plan.rows)]
    return torch.cat(parts, 0)


def allgather_edges(local_vec, plan: ShardPlan, group=None):
    """local_vec: [edges_max] (rank's edges first). Returns the full [M]."""
    import torch

    buf = torch.empty(plan.world * plan.edges_max, dtype=local_vec.dtype, device=local_vec.device)
    _all_gather(buf, local_vec.contiguous(), group)
    parts = [buf[r * plan.edges_max: r * plan.edges_max + (e1 - e0)]
             for r, (e0, e1) in enumerate(plan.edges)]
    return torch.cat(parts, 0)

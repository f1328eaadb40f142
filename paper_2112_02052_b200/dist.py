"""Row-window sharding across the GPUs of one box.

Windows are independent, so rank r owns the row windows of
one contiguous row range and runs every sparse kernel -- and SGT itself -- on
those windows only:

* **Uniform row ranges** of R rows (R a multiple of blk_h): rank r owns rows
  [rR, (r+1)R). Equal ranges are what lets every exchange be one in-place
  ``all_gather_into_tensor`` over a persistent padded buffer whose rows ARE
  the node ids (rows >= N are padding): a rank copies its rows into its slice
  and the collective fills the rest, with no reassembly and no allocation per
  call. On the uniform-degree BASELINE graphs equal rows are within a few
  percent of equal tile counts (``ShardPlan.imbalance`` reports it).
* **SGT per shard** (``translate_sharded``): each rank translates its own
  windows of A and of A^T (``sgt.ShardSgt``); the only exchange is the P
  shard totals (one all-gather of P int64) for the global col_offsets base.
* **Dense GEMMs by rows**: every rank transforms only its own rows; the
  layer's input rows are all-gathered where a sparse op needs neighbours, and
  the (tiny) weight gradients are all-reduced once per step
  (``Shard.allreduce_grads``).
* **AGNN edge weights**: P and dS of a rank's edges live in its slice of one
  padded edge buffer ([P, dS] per rank, 2 * Emax floats), exchanged by one
  in-place all-gather per layer backward; the A^T pass reads them through a
  precomputed A^T-edge -> padded-slot index (``perm_pad``).

The host logic (plan, padded layout, index remap, in-place gathers) is
backend agnostic and runs under gloo on CPU in tests/test_dist_cpu.py; the
GPU path runs under NCCL (tests/test_gpu_dist.py: gloo world 2 on one GPU
and an NCCL world-1 communicator inside a captured CUDA graph).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def partition_windows(cost: np.ndarray, parts: int) -> list[tuple[int, int]]:
    """Contiguous window ranges whose summed `cost` is balanced: cut where the
    cumulative cost crosses k/parts of the total (deterministic). Used to
    report how far the uniform row ranges are from cost balance."""
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
    blk_h: int
    num_nodes: int
    num_edges: int
    R: int                            # rows per rank (multiple of blk_h)
    windows: list[tuple[int, int]]    # per rank [wb, we)
    rows: list[tuple[int, int]]       # per rank [rb, re) = [min(rR, N), min((r+1)R, N))
    edges: list[tuple[int, int]]      # per rank [eb, ee) of A
    imbalance: float = 1.0            # max / mean tile count over ranks (when costs given)

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
        return self.R

    @property
    def padded_rows(self) -> int:
        return self.world * self.R

    @property
    def edges_max(self) -> int:
        return max(1, max(e1 - e0 for e0, e1 in self.edges))

    def edge_slot(self, e: np.ndarray) -> np.ndarray:
        """Slot of A edge e in the padded per-rank edge layout (rank q's edges
        at [q * 2 Emax, q * 2 Emax + m_q); the second Emax half holds dS)."""
        e = np.asarray(e, dtype=np.int64)
        starts = np.array([e0 for e0, _ in self.edges], dtype=np.int64)
        q = np.searchsorted(starts, e, side="right") - 1
        return q * 2 * self.edges_max + (e - starts[q])


def make_shard_plan(node_pointer: np.ndarray, num_nodes: int, blk_h: int, wp_a=None, wp_t=None,
                    rank: int = 0, world: int = 1) -> ShardPlan:
    """Uniform row ranges (see the module docstring). `wp_a` / `wp_t`
    (win_partition of A / A^T), when given, only feed `imbalance`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    n = int(num_nodes)
    W = -(-n // blk_h)
    R = max(1, -(-W // world)) * blk_h
    rows = [(min(r * R, n), min((r + 1) * R, n)) for r in range(world)]
    wins = [(-(-r0 // blk_h), -(-r1 // blk_h)) for r0, r1 in rows]
    edges = [(int(node_pointer[r0]), int(node_pointer[r1])) for r0, r1 in rows]
    imb = 1.0
    if wp_a is not None:
        cost = np.asarray(wp_a, dtype=np.float64)
        if wp_t is not None:
            cost = cost + np.asarray(wp_t, dtype=np.float64)
        per = np.array([cost[a:b].sum() for a, b in wins])
        imb = float(per.max() / per.mean()) if per.mean() > 0 else 1.0
    m = int(node_pointer[n]) if n else 0
    return ShardPlan(rank, world, blk_h, n, m, R, wins, rows, edges, imb)


def _all_gather_inplace(buf, plan: ShardPlan, group=None):
    """buf: [world * chunk, ...] contiguous; rank r's chunk r is filled, the
    collective fills the others in place (NCCL). Other backends (gloo, used by
    the functional tests) stage device tensors through the host."""
    import torch.distributed as dist

    chunk = buf.shape[0] // plan.world
    mine = buf[plan.rank * chunk:(plan.rank + 1) * chunk]
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(buf, mine, group=group)
        return
    hb = buf.cpu() if buf.is_cuda else buf
    dist.all_gather_into_tensor(hb, hb[plan.rank * chunk:(plan.rank + 1) * chunk].clone(), group=group)
    if buf.is_cuda:
        buf.copy_(hb)


def allgather_rows(buf, plan: ShardPlan, group=None):
    """In-place row all-gather of a padded [world * R, D] buffer whose slice
    [rank R, (rank+1) R) holds this rank's rows; returns buf (rows = node ids)."""
    _all_gather_inplace(buf, plan, group)
    return buf


def allgather_edges(buf, plan: ShardPlan, group=None):
    """In-place all-gather of a padded [world * 2 Emax] edge buffer (per rank:
    its edges' P in the first Emax slots, dS in the second)."""
    _all_gather_inplace(buf, plan, group)
    return buf


def translate_sharded(g, cfg, win_range, group=None, device=None):
    """SGT of this rank's windows only (sgt.ShardSgt) with the global
    col_offsets base from one all-gather of the shard totals: bit for bit the
    whole-graph SGT restricted to the shard."""
    import torch
    import torch.distributed as dist

    from .sgt import ShardSgt

    sh = ShardSgt(g, cfg, win_range, device).count()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    tot = sh.total.clone()
    if world > 1:
        allt = torch.empty(world, dtype=torch.int64, device=tot.device)
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(allt, tot, group=group)
        else:
            ht = torch.empty(world, dtype=torch.int64)
            dist.all_gather_into_tensor(ht, tot.cpu(), group=group)
            allt.copy_(ht)
        host = allt.cpu().numpy()
    else:
        host = tot.cpu().numpy()
    t = sh.fill(int(host[:rank].sum()))
    t.dev["num_unique"] = int(host.sum())
    return t


@dataclass
class Shard:
    """Everything one rank needs for the sharded step: the plan, its SGT
    shards of A and A^T, the A^T edge -> padded edge slot index of its own
    A^T edges, persistent gather buffers and the process group."""

    plan: ShardPlan
    t: object                 # TiledGraph: SGT of A on this rank's windows
    tt: object                # TiledGraph: SGT of A^T on this rank's windows
    perm: object              # A^T edge k -> A edge perm[k] (device int32, all edges)
    perm_pad: object          # padded slot of the A edge of each of this rank's A^T edges
    t_edges: tuple            # [kb, ke) A^T edges of this rank's windows
    group: object = None
    _bufs: dict = field(default_factory=dict)

    @staticmethod
    def build(g, cfg, plan: ShardPlan, group=None, device=None) -> "Shard":
        import torch

        from .sgt import csr_transpose_device

        t = translate_sharded(g, cfg, plan.my_windows, group, device)
        gt, perm = csr_transpose_device(g, device)
        tt = translate_sharded(gt, cfg, plan.my_windows, group, device)
        r0, r1 = plan.my_rows
        ptr_t = gt._ptr_d
        kb, ke = int(ptr_t[r0].item()), int(ptr_t[r1].item())
        src = perm[kb:ke].to(torch.int64)
        starts = torch.tensor([e0 for e0, _ in plan.edges], dtype=torch.int64, device=src.device)
        q = torch.searchsorted(starts, src, right=True) - 1
        pad = (q * 2 * plan.edges_max + (src - starts[q])).to(torch.int32)
        perm_pad = torch.zeros(max(g.num_edges, 1), dtype=torch.int32, device=src.device)
        perm_pad[kb:ke] = pad
        return Shard(plan, t, tt, perm, perm_pad, (kb, ke), group)

    # ---- persistent buffers -------------------------------------------------
    def rows_buffer(self, key, d: int):
        """[world * R, Dp] zero-initialised, contiguous (Dp = d rounded up to 4
        for 16-B rows); returns (buffer, [N x d] view, own-rows view)."""
        import torch

        got = self._bufs.get(("rows", key, d))
        if got is None:
            p = self.plan
            dp = d if d <= 16 or d % 4 == 0 else (d + 3) // 4 * 4
            buf = torch.zeros((p.padded_rows, dp), dtype=torch.float32, device=self.t.device)
            r0, r1 = p.my_rows
            got = (buf, buf[: p.num_nodes, :d], buf[r0:r1, :d])
            self._bufs[("rows", key, d)] = got
        return got

    def edge_buffer(self, key):
        """[world * 2 Emax] zero-initialised; returns (buffer, P view, dS view),
        the views indexed by absolute A edge id for this rank's edges."""
        import torch

        got = self._bufs.get(("edges", key))
        if got is None:
            p = self.plan
            em = p.edges_max
            buf = torch.zeros(p.world * 2 * em, dtype=torch.float32, device=self.t.device)
            e0, _ = p.my_edges
            off = p.rank * 2 * em - e0  # >= 0: every rank's edge count is <= Emax
            got = (buf, buf[off: off + p.num_edges + 1], buf[off + em: off + em + p.num_edges + 1])
            self._bufs[("edges", key)] = got
        return got

    def at_buffers(self):
        """A^T-edge-indexed P / dS arrays (this rank's A^T edges filled)."""
        import torch

        got = self._bufs.get("at")
        if got is None:
            m = max(self.plan.num_edges, 1)
            got = (torch.zeros(m, dtype=torch.float32, device=self.t.device),
                   torch.zeros(m, dtype=torch.float32, device=self.t.device))
            self._bufs["at"] = got
        return got

    def comm_stream(self):
        """Side stream for collectives that overlap kernels (NCCL only: gloo
        stages through the host synchronously); None when not overlapping."""
        import torch
        import torch.distributed as dist

        if not dist.is_initialized() or dist.get_backend(self.group) != "nccl":
            return None
        st = self._bufs.get("comm_stream")
        if st is None:
            st = torch.cuda.Stream(device=self.t.device)
            self._bufs["comm_stream"] = st
        return st

    def allreduce_grads(self, params):
        """Sum the row-sharded weight gradients over the ranks (one collective
        over the flattened gradients)."""
        import torch
        import torch.distributed as dist

        grads = [p.grad for p in params if p.grad is not None]
        if self.plan.world == 1 or not grads:
            return
        flat = self._bufs.get(("flat", sum(g.numel() for g in grads)))
        if flat is None:
            flat = torch.empty(sum(g.numel() for g in grads), dtype=torch.float32,
                               device=grads[0].device)
            self._bufs[("flat", flat.numel())] = flat
        o = 0
        for gr in grads:
            flat[o:o + gr.numel()].copy_(gr.reshape(-1))
            o += gr.numel()
        if dist.get_backend(self.group) == "nccl":
            dist.all_reduce(flat, group=self.group)
        else:
            h = flat.cpu()
            dist.all_reduce(h, group=self.group)
            flat.copy_(h)
        o = 0
        for gr in grads:
            gr.copy_(flat[o:o + gr.numel()].view_as(gr))
            o += gr.numel()

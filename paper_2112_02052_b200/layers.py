"""torch.autograd layers over the B200 kernels: GCNConv / AGNNConv and the
two models of the paper's evaluation.

The reference has forward functions only (gcn_layer, agnn_layer,
kernels.py:559-601; backprop is a non-goal there). The layers
here keep those forward semantics and add the backward passes:

  GCNConv(X)  = A (X W) + b            (update-first reordering of
                                         gcn_layer's (A X) W + b: same maths,
                                         fp32 reassociation only)
      dH = A^T G (SpMM on SGT(A^T), weights through the edge permutation)
  AGNNConv(X) = agnn_layer(t, X W):  S_e = <Z_i, Z_j>, P = rowsoftmax(S),
                Y_i = sum_e P_e Z_j
      dS = P * (<G_i, Z_j> - rowsum(P <G_i, Z_j>))   (SDDMM2 + fused softmax bwd)
      dZ = A_dS Z + A^T_{P} G + A^T_{dS} Z            (one SpMM on A, one dual
                                                       SpMM on A^T)

Every sparse op is a libtcg_b200.so kernel; the dense GEMMs are fp32
libtcg_b200.so kernels too (TF32 disabled). With a Shard
(dist.py) each rank runs its row windows and its rows of every dense op, the
inputs of the sparse ops are all-gathered in place, and the weight gradients
are all-reduced (Shard.allreduce_grads).
"""

from __future__ import annotations

import math
import os

import torch
import torch.nn as nn
import torch.nn.functional as F

from . import _lib
from .dist import Shard, allgather_edges, allgather_rows
from .dense import (  # noqa: F401  (re-exported)
    DenseFn,
    dense_backward,
    Linear,
    SoftmaxXentFn,
    colsum,
    LinearXentFn,
    colsum_gate,
    cross_entropy,
    linear_cross_entropy,
    rows_empty,
    rows_ok,
)
from .kernels import (
    agnn_forward_next_device,
    agnn_backward_device,
    agnn_forward_device,
    invert_perm_device,
    permute2_device,
    permute_device,
    sddmm_device,
    spmm_device,
)
from .sgt import TiledGraph


def _edge_weights(t: TiledGraph):
    g = t._require_graph()
    return None if g.edge_values is None else g.device_arrays(t.device)[2]


def _rows_out(t: TiledGraph, d: int, like: torch.Tensor):
    return rows_empty(t.num_nodes, d, like.device)


def _rows16(x):
    """x with 16-B aligned rows: the TF32 engine stages rows in 16/8-byte slices,
    so an odd width (GCN class counts, e.g. products' 47) is copied once into a
    padded-stride buffer instead of falling back to 4-byte slices."""
    d = x.shape[1]
    if x.stride(1) == 1 and x.stride(0) % 4 == 0 and x.data_ptr() % 16 == 0:
        return x  # already 16-B aligned rows (padded stride from rows_empty)
    x = x.contiguous()
    if d <= 16 or d % 4 == 0:
        return x
    buf = torch.empty((x.shape[0], (d + 3) // 4 * 4), dtype=x.dtype, device=x.device)
    v = buf[:, :d]
    v.copy_(x)
    return v


class GcnAggregate(torch.autograd.Function):
    """Y = A_w H + b, w = stored edge values (or 1); relu=True gives relu(Y)
    with the ReLU in the SpMM epilogue and its backward fused with the bias
    gradient (tcg_colsum_gate)."""

    @staticmethod
    def forward(ctx, h, bias, t: TiledGraph, mode: str, relu: bool = False):
        h = _rows16(h) if mode == "tf32" else h.contiguous()
        out = _rows_out(t, h.shape[1], h)
        spmm_device(t, h, _edge_weights(t), mode=mode, out=out, bias=bias, relu=relu)
        ctx.t, ctx.mode, ctx.relu = t, mode, relu
        ctx.has_bias = bias is not None
        if relu:
            ctx.save_for_backward(out)
        return out

    @staticmethod
    def backward(ctx, g):
        t = ctx.t
        db = None
        if ctx.relu:  # g .* [Y > 0] and its column sums in one pass
            (y,) = ctx.saved_tensors
            g, cs = colsum_gate(g, y)
            db = cs if ctx.has_bias else None
        g = _rows16(g) if ctx.mode == "tf32" else g.contiguous()
        tt = t.transpose()
        out = _rows_out(t, g.shape[1], g)
        spmm_device(tt.tiled, g, _edge_weights_t(t, tt.perm), mode=ctx.mode, out=out)
        if ctx.has_bias and not ctx.relu:
            db = colsum(g)
        return out, db, None, None, None


def _edge_weights_t(t: TiledGraph, perm):
    """Stored edge values in A^T edge order (cached per tiling), or None."""
    wt = _edge_weights(t)
    if wt is None:
        return None
    key = ("edge_values_T", wt.data_ptr())
    if key not in t._aux:
        t._aux[key] = permute_device(wt, perm)
    return t._aux[key]


class GcnAggShard(torch.autograd.Function):
    """Sharded Y_r = A_w H + b over this rank's row windows: H's rows are
    all-gathered in place (persistent buffer), Y_r = the rank's rows. Backward:
    G's rows all-gathered, dH_r = (A^T)_w G on this rank's A^T windows."""

    @staticmethod
    def forward(ctx, h_local, bias, sh: Shard, key, mode: str):
        d = h_local.shape[1]
        buf, full, mine = sh.rows_buffer(("gcn_in", key), d)
        mine.copy_(h_local)
        allgather_rows(buf, sh.plan, sh.group)
        r0, r1 = sh.plan.my_rows
        out = rows_empty(r1 - r0, d, h_local.device)
        spmm_device(sh.t, full, _edge_weights(sh.t), mode=mode, out=out, bias=bias,
                    win_range=sh.plan.my_windows, y_row0=r0)
        ctx.sh, ctx.mode, ctx.has_bias = sh, mode, bias is not None
        return out

    @staticmethod
    def backward(ctx, g):
        sh = ctx.sh
        d = g.shape[1]
        buf, full, mine = sh.rows_buffer("grad", d)
        mine.copy_(g)
        allgather_rows(buf, sh.plan, sh.group)
        r0, r1 = sh.plan.my_rows
        out = rows_empty(r1 - r0, d, g.device)
        spmm_device(sh.tt, full, _edge_weights_t(sh.t, sh.perm), mode=ctx.mode, out=out,
                    win_range=sh.plan.my_windows, y_row0=r0)
        db = colsum(rows_ok(g)) if ctx.has_bias else None
        return out, db, None, None, None


# measured: permuting P / dS once (2 x 9 us) beats gathering them through perm
# inside the A^T SpMM (+20 us per layer); TCG_GATHER_WEIGHTS=1 opts into the latter
_PERMUTE_WEIGHTS = os.environ.get("TCG_GATHER_WEIGHTS") is None


# P / dS in A^T edge order: by default a gather (tcg_permute_f32) in the
# backward; TCG_FUSED_PT=1 switches to scatters right after the producing
# kernels (tcg_agnn_forward_t / ds_t). Writing them from the kernel epilogues
# was measured slower (1.22 vs 1.15 ms / epoch) and is not offered.
_FUSED_PT = os.environ.get("TCG_FUSED_PT") is not None

# AGNNConv: Z = X W stored on the tf32 grid for the tensor-core aggregation (TCG_Z_TF32=0: off)
_Z_TF32 = os.environ.get("TCG_Z_TF32", "1") != "0"

# AGNN model: the next layer's dense step in the AGNN forward epilogue (opt-in, see AGNN._trunk)
_AGNN_NEXT = os.environ.get("TCG_AGNN_NEXT") == "1"


def _inv_perm(t: TiledGraph):
    """A^T position of every A edge (cached per tiling)."""
    inv = t._aux.get("inv_perm")
    if inv is None:
        inv = invert_perm_device(t.transpose().perm)
        t._aux["inv_perm"] = inv
    return inv


class AgnnAggregate(torch.autograd.Function):
    """Y = spmm(A, P; Z), P = rowsoftmax(sddmm(Z, Z)). z_tf32: Z is already on
    the tf32 grid (AGNNConv's dense step stores it rounded), so the tensor-core
    kernels skip its operand rounding -- same values, 16 fewer cvt per block."""

    @staticmethod
    def forward(ctx, z, t: TiledGraph, mode: str, z_tf32: bool = False):
        z = z.contiguous()
        m = t.num_edges
        p = torch.empty(max(m, 1), dtype=torch.float32, device=z.device)
        out = _rows_out(t, z.shape[1], z)
        p_t = None
        if mode == "tf32" and m and _FUSED_PT:
            # P also written in A^T edge order by the same epilogue (no permute pass)
            p_t = torch.empty(m, dtype=torch.float32, device=z.device)
            agnn_forward_device(t, z, p=p, out=out, p_t=p_t, inv_perm=_inv_perm(t))
        elif mode == "tf32":
            agnn_forward_device(t, z, p=p, out=out, z_tf32=z_tf32)
        else:
            if m:
                sddmm_device(t, z, mode=mode, epilogue=_lib.EPI_SOFTMAX, out=p)
            spmm_device(t, z, p if m else None, mode=mode, out=out)
        ctx.save_for_backward(z, p, out if mode == "tf32" else None, p_t)
        ctx.t, ctx.mode, ctx.z_tf32 = t, mode, z_tf32
        return out

    @staticmethod
    def backward(ctx, g):
        z, p, y_fwd, p_t = ctx.saved_tensors
        return _agnn_backward(ctx.t, ctx.mode, z, p, y_fwd, p_t, g, ctx.z_tf32), None, None, None


def _agnn_backward(t: TiledGraph, mode: str, z, p, y_fwd, p_t, g, z_tf32=False):
    """dZ of Y = spmm(A, P; Z) for the incoming gradient g: the A-side
    (dS = P (dP - rowsum), A_dS Z) and one dual SpMM on A^T (A^T_P G + A^T_dS Z)."""
    g = g.contiguous()
    m = t.num_edges
    out = _rows_out(t, z.shape[1], z)
    if m == 0:
        out.zero_()
        return out
    ds = torch.empty(m, dtype=torch.float32, device=z.device)
    ds_t = torch.empty(m, dtype=torch.float32, device=z.device) if p_t is not None else None
    if mode == "tf32":
        # dS and A_dS Z from one gather of Z's neighbour rows (dS also in A^T order)
        agnn_backward_device(t, z, g, p, ds=ds, out=out, y_fwd=y_fwd, ds_t=ds_t,
                             inv_perm=_inv_perm(t) if ds_t is not None else None, z_tf32=z_tf32)
    else:
        sddmm_device(t, g, z, mode=mode, epilogue=_lib.EPI_SOFTMAX_BWD, aux=p, out=ds)
        spmm_device(t, z, ds, mode=mode, out=out)
    tt = t.transpose()
    # one dual SpMM on A^T: A^T_P G + A^T_dS Z
    if p_t is not None:
        spmm_device(tt.tiled, g, p_t, x2=z, weights2=ds_t, mode=mode, out=out, accumulate=True,
                    x2_tf32=z_tf32)
    elif mode == "tf32" and not _PERMUTE_WEIGHTS:
        spmm_device(tt.tiled, g, p, weight_idx=tt.perm, x2=z, weights2=ds, weight_idx2=tt.perm,
                    mode=mode, out=out, accumulate=True, x2_tf32=z_tf32)
    else:
        pt, dst = permute2_device(p, ds, tt.perm)
        spmm_device(tt.tiled, g, pt, x2=z, weights2=dst, mode=mode, out=out, accumulate=True,
                    x2_tf32=z_tf32)
    return out


class AgnnAggregateNext(torch.autograd.Function):
    """Z_next = AGNN(Z) W_next: an AGNN aggregation and the next layer's dense
    step in one launch (tcg_agnn_forward_next; D = 32 on the tensor cores). The
    backward is the dense backward (dY = dZ_next W_nextᵀ, dW_next = Yᵀ dZ_next,
    one pass) followed by the AGNN backward."""

    @staticmethod
    def forward(ctx, z, w_next, t: TiledGraph, mode: str):
        z = z.contiguous()
        y, p, zn = agnn_forward_next_device(t, z, w_next, out=_rows_out(t, z.shape[1], z))
        ctx.save_for_backward(z, p, y, w_next)
        ctx.t, ctx.mode = t, mode
        return zn

    @staticmethod
    def backward(ctx, gzn):
        z, p, y, w = ctx.saved_tensors
        gy, dw = dense_backward(y, rows_ok(gzn), w.contiguous())
        return _agnn_backward(ctx.t, ctx.mode, z, p, y, None, gy), dw, None, None


class AgnnAggShard(torch.autograd.Function):
    """Sharded AGNN aggregation of this rank's rows.

    Forward: Z's rows all-gathered in place; the fused kernel runs on the
    rank's windows, writing Y's rows into a persistent row buffer (the
    backward reads them at absolute row ids) and P of the rank's edges into
    its slice of the layer's padded edge buffer.
    Backward: G's rows all-gathered; the A-side kernel writes dS of the rank's
    edges and dZ_r = A_dS Z; one in-place all-gather exchanges [P | dS] of all
    ranks; both are permuted into A^T edge order for the rank's own A^T edges
    only (perm_pad) and one dual SpMM on its A^T windows adds
    A^T_P G + A^T_dS Z."""

    @staticmethod
    def forward(ctx, z_local, sh: Shard, key, mode: str, z_tf32: bool = False):
        d = z_local.shape[1]
        zbuf, zf, zmine = sh.rows_buffer(("z", key), d)
        zmine.copy_(z_local)
        allgather_rows(zbuf, sh.plan, sh.group)
        _, yf, ymine = sh.rows_buffer(("y", key), d)
        ebuf, pv, dsv = sh.edge_buffer(key)
        wr = sh.plan.my_windows
        if mode == "tf32":
            agnn_forward_device(sh.t, zf, p=pv, out=yf, win_range=wr, y_row0=0, z_tf32=z_tf32)
        else:
            sddmm_device(sh.t, zf, mode=mode, epilogue=_lib.EPI_SOFTMAX, out=pv, win_range=wr)
            spmm_device(sh.t, zf, pv, mode=mode, out=yf, win_range=wr, y_row0=0)
        ctx.sh, ctx.key, ctx.mode, ctx.z_tf32 = sh, key, mode, z_tf32
        return ymine.clone()

    @staticmethod
    def backward(ctx, g):
        sh, key, mode = ctx.sh, ctx.key, ctx.mode
        d = g.shape[1]
        _, zf, _ = sh.rows_buffer(("z", key), d)
        _, yf, _ = sh.rows_buffer(("y", key), d)
        gbuf, gf, gmine = sh.rows_buffer("grad", d)
        gmine.copy_(g)
        # The A-side kernel reads only this rank's rows of G (the SDDMM's own-row
        # operand) and the already gathered Z, so under NCCL the G all-gather runs
        # on a side stream beside it; the A^T pass below needs every row of G.
        side = sh.comm_stream()
        if side is not None:
            cur = torch.cuda.current_stream()
            side.wait_stream(cur)
            with torch.cuda.stream(side):
                allgather_rows(gbuf, sh.plan, sh.group)
        else:
            allgather_rows(gbuf, sh.plan, sh.group)
        ebuf, pv, dsv = sh.edge_buffer(key)
        wr = sh.plan.my_windows
        r0, r1 = sh.plan.my_rows
        out = rows_empty(r1 - r0, d, g.device)
        if mode == "tf32":
            agnn_backward_device(sh.t, zf, gf, pv, ds=dsv, out=out, win_range=wr, y_row0=r0,
                                 y_fwd=yf, z_tf32=ctx.z_tf32)
        else:
            sddmm_device(sh.t, gf, zf, mode=mode, epilogue=_lib.EPI_SOFTMAX_BWD, aux=pv, out=dsv,
                         win_range=wr)
            spmm_device(sh.t, zf, dsv, mode=mode, out=out, win_range=wr, y_row0=r0)
        if side is not None:
            torch.cuda.current_stream().wait_stream(side)
        allgather_edges(ebuf, sh.plan, sh.group)
        pt, dst = sh.at_buffers()
        kb, ke = sh.t_edges
        if ke > kb:
            _lib.check(_lib.load().tcg_permute2_f32(
                ebuf.data_ptr(), ebuf.data_ptr() + 4 * sh.plan.edges_max,
                sh.perm_pad.data_ptr() + 4 * kb, pt.data_ptr() + 4 * kb, dst.data_ptr() + 4 * kb,
                ke - kb, _lib.current_stream()), "tcg_permute2_f32")
        spmm_device(sh.tt, gf, pt, x2=zf, weights2=dst, mode=mode, out=out, accumulate=True,
                    win_range=wr, y_row0=r0, x2_tf32=ctx.z_tf32)
        return out, None, None, None, None


def _glorot(fan_in, fan_out, gen=None):
    return torch.randn(fan_in, fan_out, generator=gen) / math.sqrt(fan_in)


class GCNConv(nn.Module):
    """TC-GNN GCNConv: Y = A X W + b.

    The sparse product runs at the narrower of the two widths: A (X W) + b when
    the layer narrows (in_dim >= out_dim), (A X) W + b -- the reference
    gcn_layer's own order, `spmm(t, x) @ w + b` (kernels.py:559-583) -- when
    it widens (e.g. 16 -> 47 classes: one 16-wide aggregation instead of a
    32-wide and a 16-wide pass, forward and backward). Same maths; only the
    fp32 association differs. `order` = "auto" | "transform_first" |
    "aggregate_first"."""

    def __init__(self, in_dim: int, out_dim: int, mode: str = "tf32", gen=None,
                 order: str = "auto"):
        super().__init__()
        if order not in ("auto", "transform_first", "aggregate_first"):
            raise ValueError(f"unknown order {order!r}")
        self.weight = nn.Parameter(_glorot(in_dim, out_dim, gen))
        self.bias = nn.Parameter(torch.zeros(out_dim))
        self.mode = mode
        self.aggregate_first = (order == "aggregate_first"
                                or (order == "auto" and in_dim < out_dim))

    def forward(self, x, t: TiledGraph, shard: Shard | None = None, key=None, relu: bool = False):
        """The layer's output (relu=True: relu of it, fused into the last kernel)."""
        if shard is not None:  # x: this rank's rows
            if self.aggregate_first:
                h = GcnAggShard.apply(x, None, shard, key, self.mode)
                return DenseFn.apply(h, self.weight, self.bias, relu)
            h = DenseFn.apply(x, self.weight, None, False)
            y = GcnAggShard.apply(h, self.bias, shard, key, self.mode)
            return F.relu(y) if relu else y
        if self.aggregate_first:
            h = GcnAggregate.apply(x, None, t, self.mode, False)
            return DenseFn.apply(h, self.weight, self.bias, relu)
        h = DenseFn.apply(x, self.weight, None, False)
        return GcnAggregate.apply(h, self.bias, t, self.mode, relu)

    def loss(self, x, t: TiledGraph, labels, shard: Shard | None = None, key=None, div=None):
        """cross_entropy(self(x, t), labels) (sum / div with `div`); aggregate-first,
        the dense step runs inside the loss kernel (logits never stored)."""
        if not self.aggregate_first:
            logits = self(x, t, shard, key)
            n = logits.shape[0]
            ce = SoftmaxXentFn.apply(logits, labels)
            return ce if div is None or div == n else ce * (n / div)
        if shard is not None:
            h = GcnAggShard.apply(x, None, shard, key, self.mode)
        else:
            h = GcnAggregate.apply(x, None, t, self.mode, False)
        return linear_cross_entropy(h, self.weight, self.bias, labels, div)


class AGNNConv(nn.Module):
    """TC-GNN AGNNConv: agnn_layer(t, X W) (kernels.py:586-601 + a linear map)."""

    def __init__(self, in_dim: int, out_dim: int, mode: str = "tf32", gen=None):
        super().__init__()
        self.weight = nn.Parameter(_glorot(in_dim, out_dim, gen))
        self.mode = mode

    def forward(self, x, t: TiledGraph, shard: Shard | None = None, key=None):
        # Z on the tf32 grid: every consumer (the fused forward, the A-side backward,
        # the dual A^T SpMM) rounds it to tf32 anyway, so the results are unchanged
        rz = self.mode == "tf32" and _Z_TF32
        z = DenseFn.apply(x, self.weight, None, False, rz)
        if shard is not None:  # x: this rank's rows
            return AgnnAggShard.apply(z, shard, key, self.mode, rz)
        return AgnnAggregate.apply(z, t, self.mode, rz)


class GCN(nn.Module):
    """X -> GCNConv(F,h) -> ReLU -> GCNConv(h,C) -> logits;
    train with `GCN.loss` (the last dense step fused into the loss) or
    `cross_entropy` of the logits."""

    def __init__(self, f_in, hidden, classes, mode="tf32", seed=3):
        super().__init__()
        gen = torch.Generator().manual_seed(seed)
        self.c1 = GCNConv(f_in, hidden, mode, gen)
        self.c2 = GCNConv(hidden, classes, mode, gen)

    def forward(self, x, t, shard=None):
        """Logits of all rows, or with a Shard of this rank's rows (x: all rows)."""
        if shard is not None:
            r0, r1 = shard.plan.my_rows
            x = x[r0:r1]
        return self.c2(self.c1(x, t, shard, 1, relu=True), t, shard, 2)

    def loss(self, x, t, labels, shard=None):
        """Mean cross-entropy of the logits against labels (all N rows), the last
        dense step fused into the loss; with a Shard, this rank's share (its
        rows' NLL / N: the sum over ranks is the loss)."""
        if shard is not None:
            r0, r1 = shard.plan.my_rows
            x, labels = x[r0:r1], labels[r0:r1]
            div = shard.plan.num_nodes
        else:
            div = None
        return self.c2.loss(self.c1(x, t, shard, 1, relu=True), t, labels, shard, 2, div)


class AGNN(nn.Module):
    """X -> Linear(F,h) -> ReLU -> L x AGNNConv(h,h) -> Linear(h,C) -> logits
    (PAPER.md:688-689); train with `AGNN.loss` (lin_out fused into the loss)
    or `cross_entropy` of the logits."""

    def __init__(self, f_in, hidden, classes, layers=4, mode="tf32", seed=3):
        super().__init__()
        gen = torch.Generator().manual_seed(seed)
        self.lin_in = Linear(f_in, hidden, bias=True, relu=True, gen=gen)
        self.convs = nn.ModuleList([AGNNConv(hidden, hidden, mode, gen) for _ in range(layers)])
        self.lin_out = Linear(hidden, classes, bias=True, gen=gen)

    def _trunk(self, x, t, shard=None):
        """The last AGNN layer's output. With TCG_AGNN_NEXT=1 (unsharded, TF32)
        each aggregation also computes the next layer's Z = Y W in its epilogue
        (AgnnAggregateNext); measured even with the separate GEMM at arxiv
        (0.900-0.915 vs 0.910 ms / epoch: the epilogue adds 11.4 us to each
        forward launch, the GEMM it replaces took 11), so it is opt-in."""
        h = self.lin_in(x)
        convs = list(self.convs)
        if (not _AGNN_NEXT or shard is not None or not convs
                or any(c.mode != "tf32" for c in convs)):
            for i, c in enumerate(convs):
                h = c(h, t, shard, i)
            return h
        z = DenseFn.apply(h, convs[0].weight, None, False)
        for c in convs[1:]:
            z = AgnnAggregateNext.apply(z, c.weight, t, c.mode)
        return AgnnAggregate.apply(z, t, convs[-1].mode)

    def forward(self, x, t, shard=None):
        """Logits of all rows, or with a Shard of this rank's rows (x: all rows)."""
        if shard is not None:
            r0, r1 = shard.plan.my_rows
            x = x[r0:r1]
        return self.lin_out(self._trunk(x, t, shard))

    def loss(self, x, t, labels, shard=None):
        """Mean cross-entropy of the logits against labels with lin_out fused
        into the loss; with a Shard, this rank's share (see GCN.loss)."""
        div = None
        if shard is not None:
            r0, r1 = shard.plan.my_rows
            x, labels = x[r0:r1], labels[r0:r1]
            div = shard.plan.num_nodes
        h = self._trunk(x, t, shard)
        lo = self.lin_out
        if lo.relu:
            return cross_entropy(lo(h), labels) if div is None else \
                SoftmaxXentFn.apply(lo(h), labels) * (h.shape[0] / div)
        return linear_cross_entropy(h, lo.weight, lo.bias, labels, div)


def cross_entropy_sharded(logits_local, labels, shard: Shard):
    """This rank's share of the mean cross-entropy over all N rows: the mean
    over its rows scaled by n_r / N, so that the sum over ranks is the loss
    and each rank's dlogits are exactly its rows of the full gradient."""
    r0, r1 = shard.plan.my_rows
    n = shard.plan.num_nodes
    return SoftmaxXentFn.apply(logits_local, labels[r0:r1]) * ((r1 - r0) / n)

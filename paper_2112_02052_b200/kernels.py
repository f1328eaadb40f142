"""SpMM / SDDMM / segment softmax / GCN and AGNN layers on the B200.

Drop-in for the reference `tcgraph.kernels` (/root/reference/pkg/src/tcgraph/
kernels.py): same function names, arguments, validation order and error
messages, same `TaskPlan` / `Counters` contract. The engine dispatch seam
(kernels.py:242-248, 396-402) is where the reference's numpy engines are
replaced by the GPU engine "b200"; the reference engine names are accepted as
aliases of it (there is no CPU engine).

Inputs may be numpy arrays (results come back as numpy, host<->device copies
included) or CUDA torch tensors (results stay on the device; this is the path
the torch layers and the benchmark use).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .sgt import PRECISION_MODES, TiledGraph, paired_block_counts

ENGINES = ("b200", "vectorized", "tilewise")
TF32_TILE = (16, 8)


@dataclass
class Counters:
    """Work counters (kernels.py:30-47), computed with the reference formulas."""

    tiles_visited: int = 0
    mma_calls: int = 0
    bytes_gathered: int = 0

    def add(self, other: "Counters") -> None:
        self.tiles_visited += other.tiles_visited
        self.mma_calls += other.mma_calls
        self.bytes_gathered += other.bytes_gathered


@dataclass
class TaskPlan:
    """Disjoint (window, dim_start, dim_count) rectangles covering the output."""

    tasks: list[tuple[int, int, int]]
    warps_per_block: int


def _dim_chunks(dim: int, parts: int, align: int) -> list[tuple[int, int]]:
    """D split into `parts` chunks aligned to `align` (kernels.py:58-86)."""
    if dim < 1:
        raise ValueError(f"embedding dimension must be >= 1, got {dim}")
    parts = max(1, parts)
    nsub = -(-dim // align)
    if nsub >= parts:
        base, rem = divmod(nsub, parts)
        out, start = [], 0
        for i in range(parts):
            end = min(start + (base + (1 if i < rem else 0)) * align, dim)
            out.append((start, end - start))
            start = end
        return out
    if nsub > 1:
        return [(s, min(align, dim - s)) for s in range(0, dim, align)]
    k = min(parts, dim)
    base, rem = divmod(dim, k)
    out, start = [], 0
    for i in range(k):
        w = base + (1 if i < rem else 0)
        out.append((start, w))
        start += w
    return out


def make_plan(t: TiledGraph, dim: int, requested_workers: int | None = None) -> TaskPlan:
    """warpPerBlock = max(1, floor(avg edges per window / 32)) (kernels.py:89-109,
    PAPER.md:854) and the (window, dim chunk) task list."""
    W = t.num_row_windows
    if requested_workers is not None:
        if requested_workers < 1:
            raise ValueError(f"requested_workers must be >= 1, got {requested_workers}")
        wpb = int(requested_workers)
    else:
        wpb = max(1, math.floor((t.num_edges / W if W else 0.0) / 32.0))
    chunks = _dim_chunks(dim, wpb, t.config.blk_h)
    return TaskPlan(tasks=[(w, d0, dc) for w in range(W) for d0, dc in chunks],
                    warps_per_block=wpb)


def validate_plan(plan: TaskPlan, num_windows: int, dim: int) -> None:
    """Reject overlapping / non-covering plans (kernels.py:112-133)."""
    per: dict[int, list[tuple[int, int]]] = {}
    for w, d0, dc in plan.tasks:
        if not 0 <= w < num_windows:
            raise ValueError(f"plan window {w} out of range [0, {num_windows})")
        if dc < 1 or d0 < 0 or d0 + dc > dim:
            raise ValueError(f"plan dim range [{d0}, {d0 + dc}) invalid for D={dim}")
        per.setdefault(w, []).append((d0, dc))
    if len(per) != num_windows:
        missing = next(w for w in range(num_windows) if w not in per)
        raise ValueError(f"plan covers no dims of window {missing}")
    for w, spans in per.items():
        spans.sort()
        cur = 0
        for d0, dc in spans:
            if d0 != cur:
                raise ValueError(f"plan {'overlap' if d0 < cur else 'gap'} at window {w}, dim {d0}")
            cur += dc
        if cur != dim:
            raise ValueError(f"plan covers dims [0, {cur}) of window {w}, need {dim}")


# ---------------------------------------------------------------------------
# argument handling
# ---------------------------------------------------------------------------


def _is_torch(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def _stream():
    import torch

    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _resolve_mode(t: TiledGraph, mode: str | None) -> str:
    mode = mode if mode is not None else t.config.precision_mode
    if mode not in PRECISION_MODES:
        raise ValueError(f"precision mode must be one of {PRECISION_MODES}, got {mode!r}")
    if mode == "tf32" and (t.config.blk_h, t.config.blk_w) != TF32_TILE:
        raise ValueError(
            f"tf32 mode requires the 16x8 tile shape, got {t.config.blk_h}x{t.config.blk_w}")
    return mode


def _check_engine(engine: str) -> None:
    if engine not in ENGINES:
        raise ValueError(f"engine must be one of {ENGINES}, got {engine!r}")


def _embeddings(t: TiledGraph, x):
    """Validate like kernels._check_embeddings (kernels.py:136-144) and return
    (device tensor f32 2-D with unit column stride, came_from_numpy)."""
    import torch

    if _is_torch(x):
        if x.dim() != 2:
            raise ValueError(f"embedding matrix must be 2-D, got shape {tuple(x.shape)}")
        if x.dtype != torch.float32:
            x = x.float()
        if not x.is_cuda:
            x = x.to(t.device)
        if x.stride(1) != 1:
            x = x.contiguous()
        host = False
    else:
        a = np.ascontiguousarray(x, dtype=np.float32)
        if a.ndim != 2:
            raise ValueError(f"embedding matrix must be 2-D, got shape {a.shape}")
        x = torch.from_numpy(a).to(t.device)
        host = True
    if x.shape[0] != t.num_nodes:
        raise ValueError(f"embedding rows {x.shape[0]} != graph nodes {t.num_nodes}")
    if x.shape[1] < 1:
        raise ValueError("embedding dimension must be >= 1")
    return x, host


def _edge_vector(t: TiledGraph, f, what="edge value list"):
    import torch

    if f is None:
        return None
    if _is_torch(f):
        f = f.reshape(-1)
        if f.dtype != torch.float32:
            f = f.float()
        f = f.to(t.device).contiguous()
    else:
        f = torch.from_numpy(np.ascontiguousarray(f, dtype=np.float32).reshape(-1)).to(t.device)
    if f.shape[0] != t.num_edges:
        raise ValueError(f"{what} has {f.shape[0]} entries, expected {t.num_edges}")
    return f


def _ptr(x):
    return None if x is None else x.data_ptr()


# ---------------------------------------------------------------------------
# counters (reference formulas: kernels.py:306-311, 511-513)
# ---------------------------------------------------------------------------


def _spmm_counters(t: TiledGraph, plan: TaskPlan) -> Counters:
    c = Counters()
    wp = t.win_partition.astype(np.int64)
    uc = np.diff(t.col_offsets).astype(np.int64)
    bh = t.config.blk_h
    groups: dict[tuple[int, int], list[int]] = {}
    for w, d0, dc in plan.tasks:
        groups.setdefault((d0, dc), []).append(w)
    for (d0, dc), ws in groups.items():
        ws = np.asarray(ws, dtype=np.int64)
        c.bytes_gathered += int(uc[ws].sum()) * dc * 4
        c.mma_calls += int(wp[ws].sum()) * (-(-dc // bh))
        if d0 == 0:
            c.tiles_visited += int(wp[ws].sum())
    return c


def _sddmm_counters(t: TiledGraph, d: int) -> Counters:
    bh, bw, n = t.config.blk_h, t.config.blk_w, t.num_nodes
    paired = paired_block_counts(t)
    W = t.num_row_windows
    rows_real = np.minimum(bh, n - np.arange(W, dtype=np.int64) * bh)
    tiles = int(paired.sum())
    gather_rows = int((paired * rows_real).sum()) + int(t.col_offsets[-1])
    return Counters(tiles, tiles * (-(-d // bw)), gather_rows * d * 4)


# ---------------------------------------------------------------------------
# device entry points (torch tensors in/out; used by layers.py and the bench)
# ---------------------------------------------------------------------------


def spmm_device(t: TiledGraph, x, weights=None, *, mode="tf32", out=None, bias=None,
                accumulate=False, weight_idx=None, x2=None, weights2=None, weight_idx2=None,
                win_range=None, y_row0=None, relu=False, x2_tf32=False):
    """Raw SpMM launch: Y = A_w X (+ A_w2 X2) (+ bias), rows of `win_range`;
    relu=True (single operand) stores relu(Y) (tcg_spmm_act); x2_tf32: x2 is
    already on the tf32 grid (TCG_PREC_X2_TF32, tf32 mode)."""
    import torch

    lib = _lib.load()
    d = x.shape[1]
    wb, we = win_range if win_range is not None else (0, t.num_row_windows)
    if out is None:
        out = torch.empty((t.num_nodes, d), dtype=torch.float32, device=x.device)
        y_row0 = 0
    elif y_row0 is None:
        y_row0 = 0
    if relu:
        if x2 is not None:
            raise ValueError("relu is supported for single-operand SpMM only")
        _lib.check(lib.tcg_spmm_act(
            C.byref(t.abi()), x.data_ptr(), x.stride(0), d, _ptr(weights), _ptr(weight_idx), _ptr(bias),
            out.data_ptr(), out.stride(0), y_row0, wb, we,
            _lib.PREC_TF32 if mode == "tf32" else _lib.PREC_F32, int(bool(accumulate)), _lib.ACT_RELU,
            _stream()), "tcg_spmm_act")
        return out
    _lib.check(lib.tcg_spmm(
        C.byref(t.abi()), x.data_ptr(), x.stride(0), d, _ptr(weights), _ptr(weight_idx),
        _ptr(x2), x2.stride(0) if x2 is not None else 0, _ptr(weights2), _ptr(weight_idx2),
        _ptr(bias), out.data_ptr(), out.stride(0), y_row0, wb, we,
        (_lib.PREC_TF32 | (_lib.PREC_X2_TF32 if x2_tf32 and x2 is not None else 0)) if mode == "tf32"
        else _lib.PREC_F32, int(bool(accumulate)), _stream()),
        "tcg_spmm")
    return out


def sddmm_device(t: TiledGraph, xa, xb=None, *, mode="tf32", epilogue=_lib.EPI_NONE, aux=None,
                 out=None, win_range=None):
    import torch

    lib = _lib.load()
    if out is None:
        out = torch.empty(max(t.num_edges, 0), dtype=torch.float32, device=xa.device)
    wb, we = win_range if win_range is not None else (0, t.num_row_windows)
    xb_ = xa if xb is None else xb
    _lib.check(lib.tcg_sddmm(
        C.byref(t.abi()), xa.data_ptr(), xa.stride(0), xb_.data_ptr(), xb_.stride(0), xa.shape[1],
        _ptr(aux), out.data_ptr() if t.num_edges else None, wb, we,
        _lib.PREC_TF32 if mode == "tf32" else _lib.PREC_F32, epilogue, _stream()), "tcg_sddmm")
    return out


def invert_perm_device(perm):
    """inv[perm[k]] = k (tcg_invert_perm)."""
    import torch

    inv = torch.empty_like(perm)
    _lib.check(_lib.load().tcg_invert_perm(perm.data_ptr(), perm.shape[0], inv.data_ptr(),
                                           _stream()), "tcg_invert_perm")
    return inv


def permute2_device(a, b, idx):
    """(a[idx], b[idx]) in one pass (tcg_permute2_f32)."""
    import torch

    n = idx.shape[0]
    da = torch.empty(n, dtype=torch.float32, device=a.device)
    db = torch.empty(n, dtype=torch.float32, device=a.device)
    _lib.check(_lib.load().tcg_permute2_f32(a.data_ptr(), b.data_ptr(), idx.data_ptr(),
                                            da.data_ptr(), db.data_ptr(), n, _stream()),
               "tcg_permute2_f32")
    return da, db


def permute_device(src, idx, out=None):
    """out[k] = src[idx[k]] (tcg_permute_f32)."""
    import torch

    n = idx.shape[0]
    if out is None:
        out = torch.empty(n, dtype=torch.float32, device=src.device)
    _lib.check(_lib.load().tcg_permute_f32(src.data_ptr(), idx.data_ptr(), out.data_ptr(), n,
                                           _stream()), "tcg_permute_f32")
    return out


def agnn_forward_device(t: TiledGraph, z, *, p=None, out=None, win_range=None, y_row0=0,
                        p_t=None, inv_perm=None, z_tf32=False):
    """Fused TF32 AGNN aggregation (tcg_agnn_forward): returns (Y, P). With
    `p_t` / `inv_perm` P is also written in A^T edge order (tcg_agnn_forward_t);
    z_tf32: z is already on the tf32 grid (tcg_agnn_forward_ex, TCG_AGNN_Z_TF32)."""
    import torch

    lib = _lib.load()
    wb, we = win_range if win_range is not None else (0, t.num_row_windows)
    if p is None:
        p = torch.empty(max(t.num_edges, 1), dtype=torch.float32, device=z.device)
    if out is None:
        out = torch.empty((t.num_nodes, z.shape[1]), dtype=torch.float32, device=z.device)
        y_row0 = 0
    if p_t is not None:
        _lib.check(lib.tcg_agnn_forward_t(C.byref(t.abi()), z.data_ptr(), z.stride(0), z.shape[1],
                                          p.data_ptr(), p_t.data_ptr(), inv_perm.data_ptr(),
                                          out.data_ptr(), out.stride(0), y_row0, wb, we,
                                          _stream()), "tcg_agnn_forward_t")
        return out, p
    if z_tf32:
        _lib.check(lib.tcg_agnn_forward_ex(C.byref(t.abi()), z.data_ptr(), z.stride(0), z.shape[1],
                                           p.data_ptr(), out.data_ptr(), out.stride(0), y_row0, wb, we,
                                           _lib.AGNN_Z_TF32, _stream()), "tcg_agnn_forward_ex")
        return out, p
    _lib.check(lib.tcg_agnn_forward(C.byref(t.abi()), z.data_ptr(), z.stride(0), z.shape[1],
                                    p.data_ptr(), out.data_ptr(), out.stride(0), y_row0, wb, we,
                                    _stream()), "tcg_agnn_forward")
    return out, p


def agnn_forward_next_device(t: TiledGraph, z, w_next, *, p=None, out=None, z_next=None):
    """tcg_agnn_forward_next: (Y, P, Y @ w_next), the next layer's dense step in
    the forward kernel's epilogue at D = 32 (3xTF32)."""
    import torch

    from .dense import rows_empty

    lib = _lib.load()
    n = t.num_nodes
    co = w_next.shape[1]
    if p is None:
        p = torch.empty(max(t.num_edges, 1), dtype=torch.float32, device=z.device)
    if out is None:
        out = torch.empty((n, z.shape[1]), dtype=torch.float32, device=z.device)
    if z_next is None:
        z_next = rows_empty(n, co, z.device)
    w_next = w_next.contiguous()
    _lib.check(lib.tcg_agnn_forward_next(C.byref(t.abi()), z.data_ptr(), z.stride(0), z.shape[1],
                                         p.data_ptr(), out.data_ptr(), out.stride(0), 0, 0,
                                         t.num_row_windows, w_next.data_ptr(), co, z_next.data_ptr(),
                                         z_next.stride(0), _stream()), "tcg_agnn_forward_next")
    return out, p, z_next


def agnn_backward_device(t: TiledGraph, z, gy, p, *, ds=None, out=None, win_range=None,
                         y_row0=0, y_fwd=None, ds_t=None, inv_perm=None, z_tf32=False):
    """A-side half of the AGNN backward (tcg_agnn_backward): returns (dZ_A, dS)
    with dS = P (dP - rowsum(P dP)), dP = <G_i, Z_j>, dZ_A = A_dS Z. With the
    forward output `y_fwd` the one-pass form (tcg_agnn_backward_fused,
    rowsum(P dP)_i = <G_i, Y_i>) runs."""
    import torch

    lib = _lib.load()
    wb, we = win_range if win_range is not None else (0, t.num_row_windows)
    if ds is None:
        ds = torch.empty(max(t.num_edges, 1), dtype=torch.float32, device=z.device)
    if out is None:
        out = torch.empty((t.num_nodes, z.shape[1]), dtype=torch.float32, device=z.device)
        y_row0 = 0
    if y_fwd is not None:
        _lib.check(lib.tcg_agnn_backward_fused_ex(
            C.byref(t.abi()), z.data_ptr(), z.stride(0), gy.data_ptr(), gy.stride(0),
            y_fwd.data_ptr(), y_fwd.stride(0), z.shape[1], p.data_ptr(), ds.data_ptr(),
            ds_t.data_ptr() if ds_t is not None else None,
            inv_perm.data_ptr() if ds_t is not None else None,
            out.data_ptr(), out.stride(0), y_row0, wb, we, _lib.AGNN_Z_TF32 if z_tf32 else 0,
            _stream()), "tcg_agnn_backward_fused_ex")
        return out, ds
    _lib.check(lib.tcg_agnn_backward(C.byref(t.abi()), z.data_ptr(), z.stride(0), gy.data_ptr(),
                                     gy.stride(0), z.shape[1], p.data_ptr(), ds.data_ptr(),
                                     out.data_ptr(), out.stride(0), y_row0, wb, we, _stream()),
               "tcg_agnn_backward")
    return out, ds


# ---------------------------------------------------------------------------
# reference-compatible API
# ---------------------------------------------------------------------------


def spmm(t: TiledGraph, x, f=None, mode: str | None = None, plan: TaskPlan | None = None,
         workers: int = 1, counters: Counters | None = None, engine: str = "b200"):
    """out = (F .* A) @ X on the GPU (kernels.py:213-251). f32 mode is bitwise
    equal to the reference; tf32 mode runs on the tensor cores."""
    g = t._require_graph()
    xd, host = _embeddings(t, x)
    d = xd.shape[1]
    fd = _edge_vector(t, f)
    mode = _resolve_mode(t, mode)
    if plan is None:
        plan = make_plan(t, d)
    validate_plan(plan, t.num_row_windows, d)
    _check_engine(engine)
    if fd is None and g.edge_values is not None:
        fd = g.device_arrays(t.device)[2]
    out = spmm_device(t, xd, fd, mode=mode)
    if counters is not None:
        counters.add(_spmm_counters(t, plan))
    return out.cpu().numpy() if host else out


def sddmm(t: TiledGraph, x, mode: str | None = None, workers: int = 1,
          counters: Counters | None = None, engine: str = "b200"):
    """F = (X X^T) .* A on the GPU (kernels.py:377-405)."""
    t._require_graph()
    xd, host = _embeddings(t, x)
    mode = _resolve_mode(t, mode)
    _check_engine(engine)
    out = sddmm_device(t, xd, mode=mode)
    if counters is not None:
        counters.add(_sddmm_counters(t, xd.shape[1]))
    return out.cpu().numpy() if host else out


def segment_softmax(values, indptr):
    """Per-row stable softmax over edge segments (kernels.py:541-556)."""
    import torch

    lib = _lib.load()
    host = not _is_torch(values)
    if host:
        v = np.ascontiguousarray(values, dtype=np.float32)
        if v.size == 0:
            return v.copy()
        vd = torch.from_numpy(v).cuda()
    else:
        vd = values.float().contiguous()
        if vd.numel() == 0:
            return vd.clone()
    if _is_torch(indptr):
        pd = indptr.to(device=vd.device, dtype=torch.int64).contiguous()
    else:
        pd = torch.from_numpy(np.ascontiguousarray(indptr, dtype=np.int64)).to(vd.device)
    out = torch.empty_like(vd)
    _lib.check(lib.tcg_segment_softmax(pd.data_ptr(), pd.shape[0] - 1, vd.data_ptr(),
                                       out.data_ptr(), _stream()), "tcg_segment_softmax")
    return out.cpu().numpy() if host else out


def gcn_layer(t: TiledGraph, x, w, b=None, mode: str | None = None, plan: TaskPlan | None = None,
              workers: int = 1, counters: Counters | None = None, engine: str = "b200"):
    """Aggregate then update: spmm(t, x) @ w + b (kernels.py:559-583); the
    update is the fp32 tall-skinny GEMM tcg_dense (no TF32), the same kernel
    GCNConv runs."""
    import torch

    from .dense import dense, rows_ok

    host = not _is_torch(x)
    agg = spmm(t, x if host else x, mode=mode, plan=plan, workers=workers, counters=counters,
               engine=engine)
    aggd = torch.from_numpy(agg).to(t.device) if host else agg
    wd = torch.as_tensor(np.ascontiguousarray(w, dtype=np.float32)) if not _is_torch(w) else w
    if wd.dim() != 2 or wd.shape[0] != aggd.shape[1]:
        raise ValueError(
            f"weight shape {tuple(wd.shape)} incompatible with aggregated dim {aggd.shape[1]}")
    wd = wd.to(aggd.device, torch.float32).contiguous()
    bd = None
    if b is not None:
        bd = torch.as_tensor(np.ascontiguousarray(b, dtype=np.float32)) if not _is_torch(b) else b
        if tuple(bd.shape) != (wd.shape[1],):
            raise ValueError(f"bias shape {tuple(bd.shape)} != ({wd.shape[1]},)")
        bd = bd.to(aggd.device, torch.float32).contiguous()
    out = dense(rows_ok(aggd.to(torch.float32)), wd, bias=bd)
    return out.cpu().numpy() if host else out


def agnn_layer(t: TiledGraph, x, mode: str | None = None, workers: int = 1,
               counters: Counters | None = None, engine: str = "b200"):
    """sddmm -> row softmax -> weighted spmm (kernels.py:586-601), with the
    softmax fused into the SDDMM epilogue."""
    g = t._require_graph()
    xd, host = _embeddings(t, x)
    mode = _resolve_mode(t, mode)
    _check_engine(engine)
    if mode == "tf32":
        out, _ = agnn_forward_device(t, xd)  # one gather serves SDDMM and SpMM
    else:
        p = sddmm_device(t, xd, mode=mode, epilogue=_lib.EPI_SOFTMAX) if t.num_edges else None
        out = spmm_device(t, xd, p, mode=mode)
    if counters is not None:
        counters.add(_sddmm_counters(t, xd.shape[1]))
        counters.add(_spmm_counters(t, make_plan(t, xd.shape[1])))
    _ = g
    return out.cpu().numpy() if host else out

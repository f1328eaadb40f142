"""Dense companions of the GNN layers on the B200 (csrc/dense.cu via the C ABI).

The models' tall-skinny fp32 GEMMs (N x F times F x C with F, C <= a few
hundred) and the softmax cross-entropy loss, as torch.autograd Functions:

  DenseFn       y = act(x W + b);  dx = (g .* [y > 0]) W^T,
                dW = x^T (g .* [y > 0]), db = colsum(g .* [y > 0])
  SoftmaxXentFn loss = mean -log_softmax(logits)[label];
                dlogits = (softmax - onehot) / n * g  (recomputed in the backward)

All reductions are fixed-order (deterministic); no TF32.
"""

from __future__ import annotations

import ctypes as C
import math

import torch
import torch.nn as nn

from . import _lib


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _p(t):
    return None if t is None else t.data_ptr()


def rows_empty(n: int, d: int, device):
    """[n x d] f32 with 16-B aligned rows: widths above 16 that are not a
    multiple of 4 (class counts such as 47 or 22) get a padded row stride, so
    the sparse engine and the dense kernels read them with vector slices and
    nothing has to be copied into an aligned buffer later."""
    if d > 16 and d % 4:
        return torch.empty((n, (d + 3) // 4 * 4), dtype=torch.float32, device=device)[:, :d]
    return torch.empty((n, d), dtype=torch.float32, device=device)


def rows_ok(x):
    """x as is when its rows are unit-stride (any row stride), else a copy."""
    return x if x.dim() == 2 and x.stride(1) == 1 else x.contiguous()


def rows16(x):
    """x with 16-B aligned rows (a padded-stride copy when they are not): the
    tensor-core dense kernels stage rows in 16-B pieces. Used for the wide input
    layers (Cora's 1433 features), where the copy is small next to the GEMM."""
    x = rows_ok(x)
    if x.stride(0) % 4 == 0 and x.data_ptr() % 16 == 0:
        return x
    out = rows_empty(x.shape[0], x.shape[1], x.device) if x.shape[1] > 16 else None
    if out is None or out.stride(0) % 4:
        buf = torch.empty((x.shape[0], (x.shape[1] + 3) // 4 * 4), dtype=x.dtype, device=x.device)
        out = buf[:, :x.shape[1]]
    out.copy_(x)
    return out


def dense(x, w, bias=None, relu=False, mask=None, transposed=False, out=None, out_tf32=False):
    """y = act((x .* [mask>0]) M + bias), M = w ([ci x co]) or w^T when
    `transposed` (w then [co x ci]); out_tf32 stores y RN-rounded to tf32
    (TCG_DENSE_OUT_TF32), for operands whose every consumer rounds them anyway."""
    lib = _lib.load()
    n, ci = x.shape
    co = w.shape[0] if transposed else w.shape[1]
    if out is None:
        out = rows_empty(n, co, x.device)
    _lib.check(lib.tcg_dense(x.data_ptr(), x.stride(0), n, ci, w.data_ptr(), co, int(transposed),
                             _p(bias), int(relu) | (_lib.DENSE_OUT_TF32 if out_tf32 else 0), _p(mask),
                             mask.stride(0) if mask is not None else 0,
                             out.data_ptr(), out.stride(0), _stream()), "tcg_dense")
    return out


def gemm_tn(a, b, mask=None, colsum=False):
    """(a^T (b .* [mask>0]), colsum(b .* [mask>0]) or None)."""
    lib = _lib.load()
    n, k = a.shape
    c = b.shape[1]
    out = torch.empty((k, c), dtype=torch.float32, device=a.device)
    cs = torch.empty(c, dtype=torch.float32, device=a.device) if colsum else None
    wsb = int(lib.tcg_gemm_tn_workspace_bytes(n, k, c))
    ws = torch.empty(max(wsb // 4, 1), dtype=torch.float32, device=a.device)
    _lib.check(lib.tcg_gemm_tn(a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), _p(mask),
                               mask.stride(0) if mask is not None else 0, n, k, c, out.data_ptr(),
                               _p(cs), ws.data_ptr(), wsb, _stream()), "tcg_gemm_tn")
    return out, cs


def dense_backward(x, g, w):
    """(g W^T, x^T g) for y = x W: one fused pass at 32 x 32 (tcg_dense_backward)."""
    lib = _lib.load()
    n, ci = x.shape
    co = g.shape[1]
    dx = torch.empty((n, ci), dtype=torch.float32, device=x.device)
    dw = torch.empty((ci, co), dtype=torch.float32, device=x.device)
    wsb = int(lib.tcg_dense_backward_workspace_bytes(n, ci, co))
    ws = torch.empty(max(wsb // 4, 1), dtype=torch.float32, device=x.device)
    _lib.check(lib.tcg_dense_backward(x.data_ptr(), x.stride(0), g.data_ptr(), g.stride(0), n, ci,
                                      co, w.data_ptr(), dx.data_ptr(), dx.stride(0),
                                      dw.data_ptr(), ws.data_ptr(), wsb, _stream()),
               "tcg_dense_backward")
    return dx, dw


def colsum(x):
    """Column sums of a 2-D device tensor (fixed-order, deterministic)."""
    lib = _lib.load()
    n, c = x.shape
    if x.stride(1) != 1:
        x = x.contiguous()
    out = torch.empty(c, dtype=torch.float32, device=x.device)
    wsb = int(lib.tcg_colsum_workspace_bytes(n, c))
    ws = torch.empty(max(wsb // 4, 1), dtype=torch.float32, device=x.device)
    _lib.check(lib.tcg_colsum(x.data_ptr(), x.stride(0), n, c, out.data_ptr(), ws.data_ptr(), wsb,
                              _stream()), "tcg_colsum")
    return out


def colsum_gate(x, gate):
    """(x .* [gate > 0], its column sums): the ReLU backward fused with the bias
    gradient (tcg_colsum_gate; fixed-order, deterministic)."""
    lib = _lib.load()
    n, c = x.shape
    x = rows_ok(x)
    gate = rows_ok(gate)
    gout = rows_empty(n, c, x.device)
    out = torch.empty(c, dtype=torch.float32, device=x.device)
    wsb = int(lib.tcg_colsum_workspace_bytes(n, c))
    ws = torch.empty(max(wsb // 4, 1), dtype=torch.float32, device=x.device)
    _lib.check(lib.tcg_colsum_gate(x.data_ptr(), x.stride(0), gate.data_ptr(), gate.stride(0), n, c,
                                   gout.data_ptr(), gout.stride(0), out.data_ptr(), ws.data_ptr(), wsb,
                                   _stream()), "tcg_colsum_gate")
    return gout, out


def _labels(labels, n: int, device):
    """Class labels as the kernel reads them: int64, contiguous, 1-D of length
    n on the logits' device (int32 / host labels are converted, anything
    else is rejected). Labels outside [0, C) turn the loss into NaN."""
    if not torch.is_tensor(labels):
        raise TypeError("labels must be a torch tensor")
    if labels.dtype not in (torch.int64, torch.int32, torch.int16, torch.uint8):
        raise TypeError(f"labels must be an integer tensor, got {labels.dtype}")
    if labels.dim() != 1 or labels.shape[0] != n:
        raise ValueError(f"labels must be 1-D of length {n}, got shape {tuple(labels.shape)}")
    return labels.to(device=device, dtype=torch.int64).contiguous()


def softmax_xent(logits, labels, grad=True):
    """(mean NLL of log_softmax, dlogits or None)."""
    lib = _lib.load()
    n, c = logits.shape
    labels = _labels(labels, n, logits.device)
    loss = torch.empty((), dtype=torch.float32, device=logits.device)
    dl = torch.empty((n, c), dtype=torch.float32, device=logits.device) if grad else None
    wsb = int(lib.tcg_softmax_xent_workspace_bytes(n))
    ws = torch.empty(max(wsb // 4, 1), dtype=torch.float32, device=logits.device)
    _lib.check(lib.tcg_softmax_xent(logits.data_ptr(), logits.stride(0), labels.data_ptr(), n, c,
                                    loss.data_ptr(), _p(dl), ws.data_ptr(), wsb, _stream()),
               "tcg_softmax_xent")
    return loss, dl


def softmax_xent_backward(logits, labels, grad_scale=None):
    """(softmax(logits) - onehot(labels)) / n * grad_scale (a device scalar)."""
    lib = _lib.load()
    n, c = logits.shape
    labels = _labels(labels, n, logits.device)
    dl = rows_empty(n, c, logits.device)
    gs = None if grad_scale is None else grad_scale.float().contiguous()
    _lib.check(lib.tcg_softmax_xent_backward(logits.data_ptr(), logits.stride(0),
                                             labels.data_ptr(), n, c, _p(gs), dl.data_ptr(),
                                             dl.stride(0), _stream()),
               "tcg_softmax_xent_backward")
    return dl


class DenseFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, b, relu: bool, out_tf32: bool = False):
        # out_tf32: y stored on the tf32 grid (its consumers all round it: the
        # AGNN aggregation's Z); the backward treats the rounding as identity
        x = rows16(x) if x.shape[1] > 128 and w.shape[1] in (16, 32) else rows_ok(x)
        y = dense(x, w.contiguous(), bias=b, relu=relu, out_tf32=out_tf32)
        ctx.relu = relu
        ctx.has_b = b is not None
        ctx.save_for_backward(x, w, y if relu else None)
        return y

    @staticmethod
    def backward(ctx, g):
        x, w, y = ctx.saved_tensors
        g = rows_ok(g)
        if not ctx.relu and not ctx.has_b and ctx.needs_input_grad[0]:
            dx, dw = dense_backward(x, g, w.contiguous())
            return dx, dw, None, None, None
        mask = y if ctx.relu else None
        dx = None
        if ctx.needs_input_grad[0]:
            dx = dense(g, w.contiguous(), mask=mask, transposed=True)
        dw, db = gemm_tn(x, g, mask=mask, colsum=ctx.has_b)
        return dx, dw, db, None, None


class SoftmaxXentFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, logits, labels):
        # loss only; the backward recomputes the softmax from the logits
        # (one read of the logits instead of writing dlogits, re-reading and
        # scaling it by the incoming gradient)
        logits = rows_ok(logits)
        loss, _ = softmax_xent(logits, labels, grad=False)
        ctx.save_for_backward(logits, labels)
        return loss

    @staticmethod
    def backward(ctx, g):
        logits, labels = ctx.saved_tensors
        return softmax_xent_backward(logits, labels, g), None


class Linear(nn.Module):
    """fp32 Linear over DenseFn (weight stored [in x out])."""

    def __init__(self, in_dim: int, out_dim: int, bias: bool = True, relu: bool = False,
                 gen=None):
        super().__init__()
        self.weight = nn.Parameter(torch.randn(in_dim, out_dim, generator=gen) / math.sqrt(in_dim))
        self.bias = nn.Parameter(torch.zeros(out_dim)) if bias else None
        self.relu = relu

    def forward(self, x):
        return DenseFn.apply(x, self.weight, self.bias, self.relu)


def cross_entropy(logits, labels):
    return SoftmaxXentFn.apply(logits, labels)


def linear_xent(x, w, bias, labels, div=None, grad=True):
    """(sum NLL / div, dlogits = (softmax - onehot) / div or None) of logits =
    x w + bias, fused (csrc/dense_mma.cu linear_xent; the logits never reach
    memory), or None when the shape is outside the fused kernel's coverage."""
    lib = _lib.load()
    n, kin = x.shape
    c = w.shape[1]
    labels = _labels(labels, n, x.device)
    div = n if div is None else int(div)
    loss = torch.empty((), dtype=torch.float32, device=x.device)
    dl = rows_empty(n, c, x.device) if grad else None
    wsb = int(lib.tcg_linear_xent_workspace_bytes(n))
    ws = torch.empty(max(wsb // 4, 1), dtype=torch.float32, device=x.device)
    rc = lib.tcg_linear_xent(x.data_ptr(), x.stride(0), n, kin, w.data_ptr(), c, _p(bias),
                             labels.data_ptr(), div, loss.data_ptr(), _p(dl),
                             dl.stride(0) if grad else 0, ws.data_ptr(), wsb, _stream())
    if rc == _lib.TCG_E_UNSUPPORTED:
        return None
    _lib.check(rc, "tcg_linear_xent")
    return loss, dl


def linear_xent_backward(x, w, bias, labels, div=None, grad_scale=None, need_dx=True):
    """(dx, dw, db) of linear_xent's loss for an incoming gradient grad_scale
    (device scalar), recomputing the logits (no stored dlogits); None outside
    the fused coverage."""
    lib = _lib.load()
    n, kin = x.shape
    c = w.shape[1]
    labels = _labels(labels, n, x.device)
    div = n if div is None else int(div)
    dx = rows_empty(n, kin, x.device) if need_dx else None
    dw = torch.empty((kin, c), dtype=torch.float32, device=x.device)
    db = torch.empty(c, dtype=torch.float32, device=x.device) if bias is not None else None
    gs = None if grad_scale is None else grad_scale.float().contiguous()
    wsb = int(lib.tcg_linear_xent_backward_workspace_bytes(n, kin, c))
    ws = torch.empty(max(wsb // 4, 1), dtype=torch.float32, device=x.device)
    rc = lib.tcg_linear_xent_backward(x.data_ptr(), x.stride(0), n, kin, w.data_ptr(), c, _p(bias),
                                      labels.data_ptr(), div, _p(gs), _p(dx),
                                      dx.stride(0) if need_dx else 0, dw.data_ptr(), _p(db),
                                      ws.data_ptr(), wsb, _stream())
    if rc == _lib.TCG_E_UNSUPPORTED:
        return None
    _lib.check(rc, "tcg_linear_xent_backward")
    return dx, dw, db


class LinearXentFn(torch.autograd.Function):
    """loss = sum_i NLL(x_i w + b, label_i) / div, the output layer and the loss
    in one kernel; the backward recomputes the logits in the kernel that
    produces dx, dw and db (no dlogits in memory). Shapes outside the fused
    coverage run the two-kernel form (dense, then softmax_xent with dlogits
    kept for the dense backward)."""

    @staticmethod
    def forward(ctx, x, w, b, labels, div):
        x = rows_ok(x)
        w = w.contiguous()
        n = x.shape[0]
        labels = _labels(labels, n, x.device)
        r = linear_xent(x, w, b, labels, div, grad=False)
        ctx.dl = None
        if r is None:  # outside the fused coverage: the two-kernel form, same maths
            logits = dense(x, w, bias=b)
            loss, dl = softmax_xent(logits, labels, grad=True)
            if div != n:
                loss, dl = loss * (n / div), dl * (n / div)
            ctx.dl = dl
        else:
            loss = r[0]
        ctx.div = div
        ctx.has_b = b is not None
        ctx.save_for_backward(x, w, b, labels)
        return loss

    @staticmethod
    def backward(ctx, g):
        x, w, b, labels = ctx.saved_tensors
        need_dx = ctx.needs_input_grad[0]
        if ctx.dl is None:
            dx, dw, db = linear_xent_backward(x, w, b, labels, ctx.div, g, need_dx)
            return dx, dw, db, None, None
        dl = rows_empty(*ctx.dl.shape, ctx.dl.device)  # keeps the 16-B row stride
        torch.mul(ctx.dl, g, out=dl)
        dx = dense(dl, w, transposed=True) if need_dx else None
        dw, db = gemm_tn(x, dl, colsum=ctx.has_b)
        return dx, dw, db, None, None


def linear_cross_entropy(x, weight, bias, labels, div=None):
    """F.cross_entropy(x @ weight + bias, labels) (mean; sum / div with `div`)
    with the output layer fused into the loss."""
    return LinearXentFn.apply(x, weight, bias, labels, x.shape[0] if div is None else int(div))

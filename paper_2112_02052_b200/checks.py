"""The reference's oracle API (tcgraph.oracle, oracle.py:17-137), B200 edition.

`ref_spmm` / `ref_sddmm` evaluate the CSR directly, without tiling, on the
GPU (`tcg_csr_spmm` / `tcg_csr_sddmm`): f32 accumulation is the reference's
fold bit for bit (product rounded, then add; CSR edge order / k ascending);
"f64" accumulates in double (tolerance checks; summation order is the
sequential one, not numpy's pairwise sum). `compare` is the host-side
element-wise agreement report of oracle.py:95-137.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .graph import CsrGraph


def _stream():
    import ctypes as C

    import torch

    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _check_embeddings(g: CsrGraph, x):
    import torch

    host = not torch.is_tensor(x)
    if host:
        x = np.ascontiguousarray(x, dtype=np.float32)
    if x.ndim != 2:
        raise ValueError(f"embedding matrix must be 2-D, got shape {tuple(x.shape)}")
    if x.shape[0] != g.num_nodes:
        raise ValueError(f"embedding rows {x.shape[0]} != graph nodes {g.num_nodes}")
    return x, host


def _accumulate(acc: str):
    if acc not in ("f32", "f64"):
        raise ValueError(f"unknown accumulate mode {acc!r}")
    return acc == "f64"


def ref_spmm(g: CsrGraph, x, f=None, accumulate: str = "f32"):
    """out[i] = sum over row i's edges e, in CSR order, of f[e] * x[col e];
    f defaults to the graph's edge values (all ones when unweighted)."""
    import torch

    x, host = _check_embeddings(g, x)
    wide = _accumulate(accumulate)
    ptr, cols, vals = g.device_arrays()
    dev = ptr.device
    if f is None:
        fd = vals
    else:
        fh = f if torch.is_tensor(f) else np.asarray(f, dtype=np.float32)
        if fh.shape[0] != g.num_edges:
            raise ValueError(f"edge value list has {fh.shape[0]} entries, expected {g.num_edges}")
        fd = torch.as_tensor(fh, dtype=torch.float32).to(dev).contiguous()
    xd = torch.as_tensor(x, dtype=torch.float32).to(dev).contiguous()
    d = int(xd.shape[1])
    out = torch.empty(g.num_nodes, d, dtype=torch.float64 if wide else torch.float32, device=dev)
    if d and g.num_nodes:
        _lib.check(_lib.load().tcg_csr_spmm(
            ptr.data_ptr(), cols.data_ptr() if g.num_edges else None,
            fd.data_ptr() if fd is not None and g.num_edges else None, g.num_nodes,
            xd.data_ptr(), d, d, out.data_ptr(), d, int(wide), _stream()), "tcg_csr_spmm")
    return out.cpu().numpy() if host else out


def ref_sddmm(g: CsrGraph, x, accumulate: str = "f32"):
    """F[e] = <x[row e], x[col e]>, the embedding dimension folded ascending."""
    import torch

    x, host = _check_embeddings(g, x)
    wide = _accumulate(accumulate)
    ptr, cols, _ = g.device_arrays()
    dev = ptr.device
    xd = torch.as_tensor(x, dtype=torch.float32).to(dev).contiguous()
    d = int(xd.shape[1])
    m = g.num_edges
    out = torch.zeros(m, dtype=torch.float64 if wide else torch.float32, device=dev)
    if m and d:
        rows = torch.empty(m, dtype=torch.int32, device=dev)
        _lib.check(_lib.load().tcg_csr_sddmm(
            ptr.data_ptr(), cols.data_ptr(), g.num_nodes, m, xd.data_ptr(), d, d,
            rows.data_ptr(), out.data_ptr(), int(wide), _stream()), "tcg_csr_sddmm")
    return out.cpu().numpy() if host else out


@dataclass
class CompareReport:
    """Element-wise agreement of a result with its reference."""

    passed: bool
    max_abs_err: float
    max_rel_err: float
    num_mismatch: int
    first_mismatch: tuple[int, ...] | None

    def __str__(self) -> str:
        status = "pass" if self.passed else "FAIL"
        loc = "" if self.first_mismatch is None else f" first at {self.first_mismatch}"
        return (f"{status}: max_abs={self.max_abs_err:.3e} max_rel={self.max_rel_err:.3e} "
                f"mismatches={self.num_mismatch}{loc}")


def compare(a, b, rel_tol: float = 0.0, abs_tol: float = 0.0) -> CompareReport:
    """|a - b| <= abs_tol + rel_tol * |b| element-wise, b the reference."""
    a = np.asarray(a.cpu() if hasattr(a, "cpu") else a, dtype=np.float64)
    b = np.asarray(b.cpu() if hasattr(b, "cpu") else b, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    if a.size == 0:
        return CompareReport(True, 0.0, 0.0, 0, None)
    diff = np.abs(a - b)
    bad = ~(diff <= abs_tol + rel_tol * np.abs(b))
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(diff == 0.0, 0.0, diff / np.abs(b))
    nbad = int(bad.sum())
    first = (tuple(int(v) for v in np.unravel_index(int(np.argmax(bad)), a.shape))
             if nbad else None)
    return CompareReport(passed=nbad == 0, max_abs_err=float(diff.max()),
                         max_rel_err=float(np.nanmax(rel)), num_mismatch=nbad,
                         first_mismatch=first)

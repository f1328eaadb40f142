"""TF32 operand rounding on the device.

`quantize_tf32` keeps the reference signature (tcgraph.tiles.quantize_tf32,
/root/reference/pkg/src/tcgraph/tiles.py:67-82) and runs `tcg_quantize_tf32`,
i.e. the same `cvt.rn.tf32.f32` instruction that rounds every tensor-core
operand inside spmm/sddmm — so the golden-vector test of this function is
also the test of the kernels' operand rounding. The other tile primitives
of the reference (Tile, mma, init_sparse, fetch_dense, store_*) are a
semantic spec realised inside the CUDA kernels (csrc/spmm.cu, sddmm.cu).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

TF32_MMA_M = 16
TF32_MMA_N = 16
TF32_MMA_K = 8


def quantize_tf32(x):
    """Round-to-nearest-even onto 10 explicit mantissa bits; Inf/NaN pass
    through. numpy in -> numpy out; CUDA tensor in -> CUDA tensor out."""
    import torch

    lib = _lib.load()
    if isinstance(x, torch.Tensor):
        xd = x.float().contiguous()
        out = torch.empty_like(xd)
        _lib.check(lib.tcg_quantize_tf32(xd.data_ptr(), out.data_ptr(), xd.numel(),
                                          C.c_void_p(torch.cuda.current_stream().cuda_stream)),
                   "tcg_quantize_tf32")
        return out
    arr = np.asarray(x, dtype=np.float32)
    flat = np.ascontiguousarray(arr.reshape(-1))
    if flat.size == 0:
        return arr.copy()
    xd = torch.from_numpy(flat).cuda()
    out = torch.empty_like(xd)
    _lib.check(lib.tcg_quantize_tf32(xd.data_ptr(), out.data_ptr(), xd.numel(),
                                      C.c_void_p(torch.cuda.current_stream().cuda_stream)),
               "tcg_quantize_tf32")
    res = out.cpu().numpy().reshape(arr.shape)
    if arr.ndim == 0:
        return np.float32(res[()])
    return res

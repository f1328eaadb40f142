"""ctypes binding of the C ABI in include/tcg.h (libtcg_b200.so).

The library is the only compute path: if it is missing or cannot be loaded,
every entry point raises — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("TCG_B200_LIB", _PKG / "libtcg_b200.so"))

TCG_OK = 0
ACT_NONE, ACT_RELU = 0, 1
TCG_E_UNSUPPORTED = -4
PREC_F32 = 0
PREC_TF32 = 1
PREC_X2_TF32 = 0x10  # TCG_PREC_X2_TF32: x2 already on the tf32 grid
DENSE_OUT_TF32 = 0x2  # TCG_DENSE_OUT_TF32
AGNN_Z_TF32 = 0x1  # TCG_AGNN_Z_TF32
EPI_NONE = 0
EPI_SOFTMAX = 1
EPI_SOFTMAX_BWD = 2
STREAM_PAD = 16  # TCG_STREAM_PAD


class TcgTiling(C.Structure):
    """Mirror of `tcg_tiling` (include/tcg.h)."""

    _fields_ = [
        ("num_nodes", C.c_int64),
        ("num_edges", C.c_int64),
        ("num_windows", C.c_int64),
        ("num_unique", C.c_int64),
        ("blk_h", C.c_int32),
        ("blk_w", C.c_int32),
        ("node_ptr", C.c_void_p),
        ("edge_list", C.c_void_p),
        ("edge_to_col", C.c_void_p),
        ("col_offsets", C.c_void_p),
        ("col_to_node", C.c_void_p),
        ("win_partition", C.c_void_p),
        ("edge_frag", C.c_void_p),
        ("max_window_edges", C.c_int64),
        ("max_window_unique", C.c_int64),
        ("block_offsets", C.c_void_p),
        ("col_stream", C.c_void_p),
        ("pair_offsets", C.c_void_p),
        ("pair_stream", C.c_void_p),
    ]


_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32
_SZ = C.c_size_t

# symbol -> (restype, argtypes); the exact set include/tcg.h declares
SIGNATURES = {
    "tcg_last_error": (C.c_char_p, []),
    "tcg_version": (C.c_char_p, []),
    "tcg_launch_count": (_I64, []),
    "tcg_device_info": (C.c_int, [C.POINTER(_I64), C.POINTER(_I64)]),
    "tcg_from_edges_workspace_bytes": (_SZ, [_I64]),
    "tcg_from_edges": (C.c_int, [_P, _P, _P, _I64, _I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "tcg_validate": (C.c_int, [_P, _P, _I64, _I64, _P, _P, _SZ, _P]),
    "tcg_structure_blocks": (C.c_int, [C.POINTER(TcgTiling), _I64, _P, _P, _P]),
    "tcg_sgt_workspace_bytes": (_SZ, [_I64, _I64, _I32]),
    "tcg_sgt": (C.c_int, [_P, _P, _I64, _I64, _I32, _I32, _P, _P, _P, _P, _P, _SZ, _P]),
    "tcg_sgt_count": (C.c_int, [_P, _P, _I64, _I64, _I32, _I32, _P, _P, _P, _SZ, _P]),
    "tcg_sgt_fill": (C.c_int, [_P, _P, _I64, _I64, _I32, _I32, _P, _P, _P, _P, _P]),
    "tcg_sgt_count_range": (C.c_int, [_P, _P, _I64, _I64, _I32, _I32, _I64, _I64, _P, _P, _P, _P, _SZ,
                                      _P]),
    "tcg_sgt_fill_range": (C.c_int, [_P, _P, _I64, _I64, _I32, _I64, _I64, _I64, _P, _P, _P, _P]),
    "tcg_edge_frag": (C.c_int, [C.POINTER(TcgTiling), _P, _P]),
    "tcg_edge_to_row": (C.c_int, [_P, _I64, _I32, _P, _P]),
    "tcg_block_stream": (C.c_int, [C.POINTER(TcgTiling), _P, _P, _P]),
    "tcg_block_stream_pairs": (C.c_int, [C.POINTER(TcgTiling), _P, _P, _P]),
    "tcg_permute_f32": (C.c_int, [_P, _P, _P, _I64, _P]),
    "tcg_permute2_f32": (C.c_int, [_P, _P, _P, _P, _P, _I64, _P]),
    "tcg_csr_transpose_workspace_bytes": (_SZ, [_I64, _I64]),
    "tcg_csr_transpose": (C.c_int, [_P, _P, _I64, _I64, _P, _P, _P, _P, _SZ, _P]),
    "tcg_spmm": (C.c_int, [C.POINTER(TcgTiling), _P, _I64, _I64, _P, _P, _P, _I64, _P, _P, _P,
                           _P, _I64, _I64, _I64, _I64, _I32, _I32, _P]),
    "tcg_sddmm": (C.c_int, [C.POINTER(TcgTiling), _P, _I64, _P, _I64, _I64, _P, _P, _I64, _I64,
                            _I32, _I32, _P]),
    "tcg_segment_softmax": (C.c_int, [_P, _I64, _P, _P, _P]),
    "tcg_segment_softmax_backward": (C.c_int, [_P, _I64, _P, _P, _P, _P]),
    "tcg_softmax_fwd": (C.c_int, [_P, _I64, _P, _P, _P]),
    "tcg_softmax_bwd": (C.c_int, [_P, _I64, _P, _P, _P, _P]),
    "tcg_agnn_fused_fwd": (C.c_int, [C.POINTER(TcgTiling), _P, _I64, _P, _P, _I64, _P]),
    "tcg_agnn_forward": (C.c_int, [C.POINTER(TcgTiling), _P, _I64, _I64, _P, _P, _I64, _I64,
                                   _I64, _I64, _P]),
    "tcg_agnn_backward": (C.c_int, [C.POINTER(TcgTiling), _P, _I64, _P, _I64, _I64, _P, _P,
                                    _P, _I64, _I64, _I64, _I64, _P]),
    "tcg_agnn_backward_fused": (C.c_int, [C.POINTER(TcgTiling), _P, _I64, _P, _I64, _P, _I64,
                                          _I64, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _P]),
    "tcg_agnn_forward_ex": (C.c_int, [C.POINTER(TcgTiling), _P, _I64, _I64, _P, _P, _I64, _I64,
                                      _I64, _I64, _I32, _P]),
    "tcg_agnn_backward_fused_ex": (C.c_int, [C.POINTER(TcgTiling), _P, _I64, _P, _I64, _P, _I64,
                                             _I64, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64,
                                             _I32, _P]),
    "tcg_agnn_forward_t": (C.c_int, [C.POINTER(TcgTiling), _P, _I64, _I64, _P, _P, _P, _P, _I64,
                                     _I64, _I64, _I64, _P]),
    "tcg_scatter_f32": (C.c_int, [_P, _P, _P, _I64, _P]),
    "tcg_invert_perm": (C.c_int, [_P, _I64, _P, _P]),
    "tcg_quantize_tf32": (C.c_int, [_P, _P, _I64, _P]),
    "tcg_csr_spmm": (C.c_int, [_P, _P, _P, _I64, _P, _I64, _I64, _P, _I64, _I32, _P]),
    "tcg_csr_sddmm": (C.c_int, [_P, _P, _I64, _I64, _P, _I64, _I64, _P, _P, _I32, _P]),
    "tcg_dense": (C.c_int, [_P, _I64, _I64, _I64, _P, _I64, _I32, _P, _I32, _P, _I64, _P, _I64,
                            _P]),
    "tcg_gemm_tn_workspace_bytes": (_SZ, [_I64, _I64, _I64]),
    "tcg_gemm_tn": (C.c_int, [_P, _I64, _P, _I64, _P, _I64, _I64, _I64, _I64, _P, _P, _P, _SZ,
                              _P]),
    "tcg_dense_backward_workspace_bytes": (_SZ, [_I64, _I64, _I64]),
    "tcg_dense_backward": (C.c_int, [_P, _I64, _P, _I64, _I64, _I64, _I64, _P, _P, _I64, _P, _P,
                                     _SZ, _P]),
    "tcg_colsum_workspace_bytes": (_SZ, [_I64, _I64]),
    "tcg_colsum": (C.c_int, [_P, _I64, _I64, _I64, _P, _P, _SZ, _P]),
    "tcg_agnn_forward_next": (C.c_int, [C.POINTER(TcgTiling), _P, _I64, _I64, _P, _P, _I64, _I64, _I64, _I64,
                                        _P, _I64, _P, _I64, _P]),
    "tcg_colsum_gate": (C.c_int, [_P, _I64, _P, _I64, _I64, _I64, _P, _I64, _P, _P, _SZ, _P]),
    "tcg_spmm_act": (C.c_int, [C.POINTER(TcgTiling), _P, _I64, _I64, _P, _P, _P, _P, _I64, _I64, _I64,
                               _I64, _I32, _I32, _I32, _P]),
    "tcg_softmax_xent_workspace_bytes": (_SZ, [_I64]),
    "tcg_softmax_xent": (C.c_int, [_P, _I64, _P, _I64, _I64, _P, _P, _P, _SZ, _P]),
    "tcg_linear_xent_workspace_bytes": (_SZ, [_I64]),
    "tcg_linear_xent": (C.c_int, [_P, _I64, _I64, _I64, _P, _I64, _P, _P, _I64, _P, _P, _I64, _P, _SZ, _P]),
    "tcg_linear_xent_backward_workspace_bytes": (_SZ, [_I64, _I64, _I64]),
    "tcg_linear_xent_backward": (C.c_int, [_P, _I64, _I64, _I64, _P, _I64, _P, _P, _I64, _P, _P, _I64,
                                           _P, _P, _P, _SZ, _P]),
    "tcg_softmax_xent_backward": (C.c_int, [_P, _I64, _P, _I64, _I64, _P, _P, _I64, _P]),
}

_lib = None
_load_error: str | None = None


def load() -> C.CDLL:
    """Load (once) and type the library; raise loudly if it is unavailable."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        _load_error = (f"{LIB_PATH} not found: build it with "
                       "`python -m paper_2112_02052_b200._build` (no CPU fallback exists)")
        raise RuntimeError(_load_error)
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class TcgError(RuntimeError):
    pass


def check(rc: int, what: str) -> None:
    if rc != TCG_OK:
        msg = load().tcg_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(msg)
        raise TcgError(f"{what} failed ({rc}): {msg}")


def launch_count() -> int:
    return int(load().tcg_launch_count())


def version() -> str:
    return load().tcg_version().decode()


def current_stream():
    """torch's current CUDA stream as the ABI's `void* stream`."""
    import torch

    return C.c_void_p(torch.cuda.current_stream().cuda_stream)

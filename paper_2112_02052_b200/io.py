"""TCGT / TCEM binary formats: cache a GPU SGT result
and embedding matrices across runs.

Same on-disk layout as the reference `tcgraph.io` (io.py:208-291), so files
are interchangeable byte for byte (tests/golden/*.tcgt, *.tcem):

  TCGT  'TCGT' | u32 version=1 | u32 blk_h | u32 blk_w | u64 N | u64 M |
        u64 W | u32 win_partition[W] | u32 edge_to_col[M] |
        u64 col_offsets[W+1] | u32 col_to_node[col_offsets[W]]
  TCEM  'TCEM' | u32 version=1 | u64 N | u64 D | f32 data[N*D] (row-major)

all little-endian. A loaded tiling is structure-only (graph=None): kernels
refuse it, the tile accounting works on it; `device=` also uploads it.
"""

from __future__ import annotations

import struct

import numpy as np

from .sgt import BlockConfig, TiledGraph

TCGT_MAGIC = b"TCGT"
TCEM_MAGIC = b"TCEM"
FORMAT_VERSION = 1
_TCGT_HEAD = struct.Struct("<IIIQQQ")
_TCEM_HEAD = struct.Struct("<IQQ")


class GraphFormatError(ValueError):
    """Malformed or unsupported graph/matrix file content (reference io.py:24)."""


def _take(buf: memoryview, off: int, nbytes: int, what: str, path) -> tuple[memoryview, int]:
    if off + nbytes > len(buf):
        raise GraphFormatError(f"{path}: truncated file while reading {what}")
    return buf[off:off + nbytes], off + nbytes


def _array(buf, off, dtype, count, what, path):
    dt = np.dtype(dtype)
    raw, off = _take(buf, off, dt.itemsize * int(count), what, path)
    return np.frombuffer(raw, dtype=dt).copy(), off


def tcgt_bytes(t: TiledGraph) -> bytes:
    """The serialised tiling (reference write_tcgt layout)."""
    W = t.num_row_windows
    parts = [TCGT_MAGIC,
             _TCGT_HEAD.pack(FORMAT_VERSION, t.config.blk_h, t.config.blk_w, t.num_nodes,
                             t.num_edges, W),
             np.asarray(t.win_partition, dtype="<u4").tobytes(),
             np.asarray(t.edge_to_col, dtype="<u4").tobytes(),
             np.asarray(t.col_offsets, dtype="<u8").tobytes(),
             np.asarray(t.col_to_node, dtype="<u4").tobytes()]
    return b"".join(parts)


def write_tcgt(t: TiledGraph, path) -> None:
    """Serialise the tiling structure (not the source graph); device-resident
    SGT arrays are copied to the host once."""
    with open(path, "wb") as fh:
        fh.write(tcgt_bytes(t))


def read_tcgt(path, device=None) -> TiledGraph:
    """Load a tiling structure (graph=None); `device` also uploads it."""
    with open(path, "rb") as fh:
        buf = memoryview(fh.read())
    magic, off = _take(buf, 0, 4, "magic", path)
    if bytes(magic) != TCGT_MAGIC:
        raise GraphFormatError(f"{path}: bad magic {bytes(magic)!r}, expected {TCGT_MAGIC!r}")
    head, off = _take(buf, off, _TCGT_HEAD.size, "header", path)
    version, blk_h, blk_w, n, m, W = _TCGT_HEAD.unpack(head)
    if version != FORMAT_VERSION:
        raise GraphFormatError(f"{path}: unsupported format version {version}")
    wp, off = _array(buf, off, "<u4", W, "win_partition", path)
    e2c, off = _array(buf, off, "<u4", m, "edge_to_col", path)
    co, off = _array(buf, off, "<u8", W + 1, "col offsets", path)
    co = co.astype(np.int64)
    c2n, off = _array(buf, off, "<u4", int(co[-1]) if W else 0, "col_to_node", path)
    if off != len(buf):
        raise GraphFormatError(f"{path}: trailing bytes after tiling payload")
    t = TiledGraph(None, BlockConfig(blk_h=blk_h, blk_w=blk_w), int(n), int(m), int(W))
    t._host.update(win_partition=wp.astype(np.uint32), edge_to_col=e2c.astype(np.uint32),
                   col_offsets=co, col_to_node=c2n.astype(np.uint32))
    if device is not None:
        import torch

        dev = torch.device(device)
        t.dev.update(
            win_partition=torch.from_numpy(wp.view(np.int32)).to(dev),
            edge_to_col=torch.from_numpy(e2c.view(np.int32)).to(dev),
            col_offsets=torch.from_numpy(co).to(dev),
            col_to_node=torch.from_numpy(c2n.view(np.int32)).to(dev),
            num_unique=int(co[-1]) if W else 0)
    return t


def write_tcem(x, path) -> None:
    """Serialise an embedding matrix (f32 row-major; torch tensors accepted)."""
    if hasattr(x, "detach"):
        x = x.detach().cpu().numpy()
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.ndim != 2:
        raise ValueError(f"embedding matrix must be 2-D, got shape {x.shape}")
    with open(path, "wb") as fh:
        fh.write(TCEM_MAGIC)
        fh.write(_TCEM_HEAD.pack(FORMAT_VERSION, x.shape[0], x.shape[1]))
        fh.write(x.astype("<f4").tobytes())


def read_tcem(path) -> np.ndarray:
    with open(path, "rb") as fh:
        buf = memoryview(fh.read())
    magic, off = _take(buf, 0, 4, "magic", path)
    if bytes(magic) != TCEM_MAGIC:
        raise GraphFormatError(f"{path}: bad magic {bytes(magic)!r}, expected {TCEM_MAGIC!r}")
    head, off = _take(buf, off, _TCEM_HEAD.size, "header", path)
    version, n, d = _TCEM_HEAD.unpack(head)
    if version != FORMAT_VERSION:
        raise GraphFormatError(f"{path}: unsupported format version {version}")
    data, off = _array(buf, off, "<f4", n * d, "embedding data", path)
    if off != len(buf):
        raise GraphFormatError(f"{path}: trailing bytes after embedding payload")
    return data.reshape(int(n), int(d)).astype(np.float32)

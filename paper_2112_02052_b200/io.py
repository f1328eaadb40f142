"""Graph and matrix files.

TCGT / TCEM binary formats cache a GPU SGT result and embedding matrices
across runs; the text loaders (edge lists, Matrix Market coordinate files)
feed the command-line harness (cli.py).

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
from pathlib import Path

import numpy as np

from .graph import CsrGraph
from .sgt import BlockConfig, TiledGraph

MAX_NODE_ID = 0xFFFFFFFF

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
    t = TiledGraph(None, BlockConfig(blk_h=blk_h, blk_w=blk_w), int(n), int(m), int(W),
                   wp.astype(np.uint32), e2c.astype(np.uint32), co, c2n.astype(np.uint32))
    if device is not None:
        t._upload(device)
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


# ---- text formats (reference io.py:28-193) ----------------------------------

def _node_id(token: str, path, lineno: int) -> int:
    try:
        v = int(token)
    except ValueError:
        raise GraphFormatError(
            f"{path}:{lineno}: expected a non-negative integer node id, got {token!r}"
        ) from None
    if v < 0:
        raise GraphFormatError(f"{path}:{lineno}: negative node id {v}")
    if v > MAX_NODE_ID:
        raise GraphFormatError(f"{path}:{lineno}: node id {v} exceeds the 32-bit id width")
    return v


def _data_lines(fh, first_lineno: int):
    """(lineno, fields) of the non-blank, non-comment lines."""
    for lineno, line in enumerate(fh, first_lineno):
        st = line.strip()
        if st and st[0] not in "#%":
            yield lineno, st.split()


def load_edge_list(path, num_nodes_hint: int | None = None) -> CsrGraph:
    """'src dst' lines ('#' / '%' comments) -> normalised CsrGraph; N is the
    largest id + 1 unless the hint is larger (reference io.py:44-68)."""
    src, dst = [], []
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, parts in _data_lines(fh, 1):
            if len(parts) != 2:
                raise GraphFormatError(
                    f"{path}:{lineno}: expected 'src dst', got {len(parts)} fields")
            src.append(_node_id(parts[0], path, lineno))
            dst.append(_node_id(parts[1], path, lineno))
    n = max(max(src, default=-1), max(dst, default=-1)) + 1
    if num_nodes_hint is not None:
        n = max(n, int(num_nodes_hint))
    return CsrGraph.from_edges(np.asarray(src, np.int64), np.asarray(dst, np.int64), n)


def save_edge_list(g: CsrGraph, path) -> None:
    """'src dst' lines in CSR order (weights are not representable)."""
    rows = np.repeat(np.arange(g.num_nodes, dtype=np.int64), np.diff(g.node_pointer))
    with open(path, "w", encoding="utf-8") as fh:
        for i, j in zip(rows.tolist(), g.edge_list.tolist()):
            fh.write(f"{i} {j}\n")


def load_matrix_market(path) -> CsrGraph:
    """Matrix Market coordinate file (pattern / real, general / symmetric) as
    an adjacency: 1-based -> 0-based, symmetric off-diagonals mirrored, real
    values kept (duplicates summed by from_edges) (reference io.py:79-172)."""
    with open(path, "r", encoding="utf-8") as fh:
        header = fh.readline()
        if not header.startswith("%%MatrixMarket"):
            raise GraphFormatError(f"{path}:1: missing %%MatrixMarket header")
        tok = header.split()
        if len(tok) != 5:
            raise GraphFormatError(f"{path}:1: malformed header {header.strip()!r}")
        obj, fmt, field, sym = (x.lower() for x in tok[1:])
        if obj != "matrix" or fmt != "coordinate":
            raise GraphFormatError(
                f"{path}:1: unsupported object/format '{obj} {fmt}' (need matrix coordinate)")
        if field not in ("pattern", "real"):
            raise GraphFormatError(f"{path}:1: unsupported field {field!r}")
        if sym not in ("general", "symmetric"):
            raise GraphFormatError(f"{path}:1: unsupported symmetry {sym!r}")
        lines = _data_lines(fh, 2)
        first = next(lines, None)
        if first is None:
            raise GraphFormatError(f"{path}: missing size line")
        lineno, parts = first
        size_line = " ".join(parts)
        if len(parts) != 3:
            raise GraphFormatError(f"{path}:{lineno}: malformed size line {size_line!r}")
        try:
            rows, cols, nnz = (int(x) for x in parts)
        except ValueError:
            raise GraphFormatError(f"{path}:{lineno}: malformed size line {size_line!r}") from None
        if rows != cols:
            raise GraphFormatError(
                f"{path}:{lineno}: adjacency matrix must be square, got {rows}x{cols}")
        if rows > MAX_NODE_ID + 1:
            raise GraphFormatError(f"{path}:{lineno}: {rows} nodes exceed the 32-bit id width")
        real = field == "real"
        want = 3 if real else 2
        src, dst, vals = [], [], ([] if real else None)
        seen = 0
        for lineno, parts in lines:
            if len(parts) != want:
                raise GraphFormatError(f"{path}:{lineno}: expected {want} fields, got {len(parts)}")
            try:
                i, j = int(parts[0]), int(parts[1])
            except ValueError:
                raise GraphFormatError(f"{path}:{lineno}: malformed entry indices") from None
            if not (1 <= i <= rows and 1 <= j <= cols):
                raise GraphFormatError(
                    f"{path}:{lineno}: index ({i}, {j}) out of declared bounds {rows}x{cols}")
            if real:
                try:
                    v = float(parts[2])
                except ValueError:
                    raise GraphFormatError(f"{path}:{lineno}: malformed entry value") from None
            seen += 1
            src.append(i - 1)
            dst.append(j - 1)
            if real:
                vals.append(v)
            if sym == "symmetric" and i != j:
                src.append(j - 1)
                dst.append(i - 1)
                if real:
                    vals.append(v)
        if seen != nnz:
            raise GraphFormatError(f"{path}: declared {nnz} entries, found {seen}")
    return CsrGraph.from_edges(np.asarray(src, np.int64), np.asarray(dst, np.int64), rows,
                               values=None if vals is None else np.asarray(vals, np.float64))


def detect_format(path) -> str:
    suffix = Path(path).suffix.lower()
    return {".mtx": "mtx", ".tcgt": "tcgt"}.get(suffix, "edgelist")


def load_graph(path, fmt: str = "auto", num_nodes_hint: int | None = None) -> CsrGraph:
    """Edge-list or Matrix Market file -> CsrGraph (reference io.py:184-193)."""
    if fmt == "auto":
        fmt = detect_format(path)
    if fmt == "edgelist":
        return load_edge_list(path, num_nodes_hint)
    if fmt == "mtx":
        return load_matrix_market(path)
    raise GraphFormatError(f"format {fmt!r} does not describe a loadable graph")

"""Sparse Graph Translation on the GPU and the tiled-graph container.

`translate` keeps the reference signature (`tcgraph.sgt.translate(g, cfg)`,
/root/reference/pkg/src/tcgraph/sgt.py:101-137) but runs on the B200 through
`tcg_sgt` (csrc/sgt.cu). The TiledGraph keeps its four SGT arrays resident in
HBM (the per-epoch kernels read them there) and materialises the numpy views
the reference exposes (`win_partition`, `edge_to_col`, `col_offsets`,
`col_to_node`) lazily, on first host access.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .graph import CsrGraph

PRECISION_MODES = ("f32", "tf32")


@dataclass(frozen=True)
class BlockConfig:
    """Tile shape and numeric mode (sgt.py:21-40)."""

    blk_h: int = 16
    blk_w: int = 8
    precision_mode: str = "f32"

    def __post_init__(self):
        if self.blk_h < 1 or self.blk_w < 1:
            raise ValueError(f"tile shape must be >= 1, got {self.blk_h}x{self.blk_w}")
        if self.precision_mode not in PRECISION_MODES:
            raise ValueError(
                f"precision_mode must be one of {PRECISION_MODES}, got {self.precision_mode!r}"
            )


def _to_np_u32(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint32)


_SGT_ARRAYS = ("win_partition", "edge_to_col", "col_offsets", "col_to_node")


class TiledGraph:
    """SGT result (sgt.py:43-98), constructed with the reference's positional
    fields: (graph, config, num_nodes, num_edges, num_row_windows,
    win_partition, edge_to_col, col_offsets, col_to_node, _aux).

    The four arrays are resident in HBM in `dev` (node_ptr i64[N+1];
    edge_list / edge_to_col / col_to_node / win_partition as int32 tensors
    holding u32 bits; col_offsets i64[W+1]); the numpy views the reference
    exposes are materialised lazily. A TiledGraph built from host arrays (as
    reference code does) uploads them on first kernel use. `graph=None` means
    structure only: kernels raise (sgt.py:92-98)."""

    def __init__(self, graph: CsrGraph | None, config: BlockConfig, num_nodes: int,
                 num_edges: int, num_row_windows: int, win_partition=None, edge_to_col=None,
                 col_offsets=None, col_to_node=None, _aux: dict | None = None, *,
                 dev: dict | None = None):
        self.graph = graph
        self.config = config
        self.num_nodes = int(num_nodes)
        self.num_edges = int(num_edges)
        self.num_row_windows = int(num_row_windows)
        self.dev = {} if dev is None else dev
        self._host = {}
        self._aux = {} if _aux is None else _aux
        given = dict(zip(_SGT_ARRAYS, (win_partition, edge_to_col, col_offsets, col_to_node)))
        for k, v in given.items():
            if v is not None:
                self._host[k] = (np.asarray(v, dtype=np.int64) if k == "col_offsets"
                                 else np.asarray(v, dtype=np.uint32))

    def __repr__(self) -> str:
        return (f"TiledGraph(config={self.config}, num_nodes={self.num_nodes}, "
                f"num_edges={self.num_edges}, num_row_windows={self.num_row_windows})")

    def _upload(self, device=None) -> None:
        """Host arrays (constructed from numpy / read from a file) -> HBM."""
        import torch

        if all(k in self.dev for k in _SGT_ARRAYS):
            return
        dev = torch.device(device) if device is not None else torch.device("cuda")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        for k in _SGT_ARRAYS:
            a = self._host[k]
            self.dev[k] = torch.from_numpy(
                np.ascontiguousarray(a if k == "col_offsets" else a.view(np.int32))).to(dev)
        self.dev["num_unique"] = int(self._host["col_offsets"][-1]) if self.num_row_windows else 0

    # ---- host views (reference attribute names) ---------------------------
    def _host_array(self, name, conv):
        a = self._host.get(name)
        if a is None:
            a = conv(self.dev[name])
            self._host[name] = a
        return a

    @property
    def win_partition(self) -> np.ndarray:
        return self._host_array("win_partition", _to_np_u32)

    @property
    def edge_to_col(self) -> np.ndarray:
        return self._host_array("edge_to_col", _to_np_u32)

    @property
    def col_offsets(self) -> np.ndarray:
        return self._host_array("col_offsets", lambda t: t.cpu().numpy())

    @property
    def col_to_node(self) -> np.ndarray:
        # the device array may be allocated at its upper bound (GPU SGT): U first
        return self._host_array("col_to_node", lambda t: _to_np_u32(t[: self.num_unique]))

    @property
    def num_unique(self) -> int:
        if "num_unique" not in self.dev:
            if "col_offsets" in self.dev:
                co = self.dev["col_offsets"]
                self.dev["num_unique"] = int(co[-1].item()) if self.num_row_windows else 0
            else:
                return int(self.col_offsets[-1]) if self.num_row_windows else 0
        return int(self.dev["num_unique"])

    def unique_count(self, window: int) -> int:
        return int(self.col_offsets[window + 1] - self.col_offsets[window])

    def window_nodes(self, window: int) -> np.ndarray:
        return self.col_to_node[self.col_offsets[window]:self.col_offsets[window + 1]]

    def window_edge_range(self, window: int) -> tuple[int, int]:
        g = self._require_graph()
        bh = self.config.blk_h
        r0, r1 = min(window * bh, g.num_nodes), min((window + 1) * bh, g.num_nodes)
        return int(g.node_pointer[r0]), int(g.node_pointer[r1])

    def window_edge_rows(self, window: int) -> np.ndarray:
        """edgeToRow: row offset within the window of each of its edges."""
        g = self._require_graph()
        bh = self.config.blk_h
        r0, r1 = min(window * bh, g.num_nodes), min((window + 1) * bh, g.num_nodes)
        return np.repeat(np.arange(r1 - r0, dtype=np.int64), np.diff(g.node_pointer[r0:r1 + 1]))

    @property
    def edge_to_row(self) -> np.ndarray:
        """edgeToRow for every edge (the window_edge_rows of all windows,
        concatenated), computed on the GPU (tcg_edge_to_row)."""
        a = self._host.get("edge_to_row")
        if a is None:
            import torch

            self._require_graph()
            ptr = self.dev["node_ptr"]
            e2r = torch.empty(max(self.num_edges, 1), dtype=torch.int32, device=ptr.device)
            _lib.check(_lib.load().tcg_edge_to_row(ptr.data_ptr(), self.num_nodes,
                                                   self.config.blk_h, e2r.data_ptr(),
                                                   _stream_ptr()), "tcg_edge_to_row")
            a = _to_np_u32(e2r[: self.num_edges])
            self._host["edge_to_row"] = a
        return a

    def _require_graph(self) -> CsrGraph:
        if self.graph is None:
            raise ValueError(
                "this TiledGraph holds tiling structure only (no source graph); "
                "reload the original edge list or matrix file to run kernels"
            )
        return self.graph

    # ---- device descriptor --------------------------------------------------
    def abi(self) -> _lib.TcgTiling:
        """The `tcg_tiling` descriptor handed to every kernel call."""
        s = self._aux.get("abi")
        if s is None:
            g = self._require_graph()
            self._upload()
            d = self.dev
            if "node_ptr" not in d:
                ptr, cols, _ = g.device_arrays()
                d.update(node_ptr=ptr, edge_list=cols)
            s = _lib.TcgTiling(
                self.num_nodes, self.num_edges, self.num_row_windows, self.num_unique,
                self.config.blk_h, self.config.blk_w,
                d["node_ptr"].data_ptr(), d["edge_list"].data_ptr() if self.num_edges else None,
                d["edge_to_col"].data_ptr() if self.num_edges else None,
                d["col_offsets"].data_ptr(),
                d["col_to_node"].data_ptr() if self.num_unique else None,
                d["win_partition"].data_ptr() if self.num_row_windows else None,
                None,
                *self.window_maxima(),
            )
            if (self.config.blk_h, self.config.blk_w) == (16, 8) and self.num_edges:
                import torch

                ef = torch.empty(self.num_edges, dtype=torch.int32, device=self.device)
                _lib.check(_lib.load().tcg_edge_frag(C.byref(s), ef.data_ptr(), _stream_ptr()),
                           "tcg_edge_frag")
                d["edge_frag"] = ef
                s.edge_frag = ef.data_ptr()
                # block stream for the SpMM engine (tcg_block_stream)
                W = self.num_row_windows
                bo = torch.empty(W + 1, dtype=torch.int32, device=self.device)
                lib = _lib.load()
                _lib.check(lib.tcg_block_stream(C.byref(s), bo.data_ptr(), None, _stream_ptr()),
                           "tcg_block_stream")
                tb = int(bo[W].item())
                cs = torch.empty(8 * (tb + _lib.STREAM_PAD), dtype=torch.int32, device=self.device)
                _lib.check(lib.tcg_block_stream(C.byref(s), bo.data_ptr(), cs.data_ptr(),
                                                _stream_ptr()), "tcg_block_stream")
                d["block_offsets"] = bo
                d["col_stream"] = cs
                s.block_offsets = bo.data_ptr()
                s.col_stream = cs.data_ptr()
                # pair stream for the 16-wide SpMM (two blocks per step)
                po = torch.empty(W + 1, dtype=torch.int32, device=self.device)
                _lib.check(lib.tcg_block_stream_pairs(C.byref(s), po.data_ptr(), None,
                                                      _stream_ptr()), "tcg_block_stream_pairs")
                tp = int(po[W].item())
                ps = torch.empty(8 * (tp + _lib.STREAM_PAD), dtype=torch.int32, device=self.device)
                _lib.check(lib.tcg_block_stream_pairs(C.byref(s), po.data_ptr(), ps.data_ptr(),
                                                      _stream_ptr()), "tcg_block_stream_pairs")
                d["pair_offsets"] = po
                d["pair_stream"] = ps
                s.pair_offsets = po.data_ptr()
                s.pair_stream = ps.data_ptr()
            self._aux["abi"] = s
        return s

    def window_maxima(self) -> tuple[int, int]:
        """(max edges, max condensed columns) over the windows: decides
        whether the fused AGNN kernels can keep a whole window on chip."""
        mx = self._aux.get("maxima")
        if mx is None:
            wb, we = getattr(self, "shard_windows", (0, self.num_row_windows))
            if we <= wb:
                mx = (0, 0)
            else:
                ptr = self.dev["node_ptr"]
                bh = self.config.blk_h
                idx = np.minimum(np.arange(wb, we + 1) * bh, self.num_nodes)
                import torch

                eb = ptr[torch.from_numpy(idx).to(ptr.device)]
                me = int((eb[1:] - eb[:-1]).max().item())
                co = self.dev["col_offsets"][wb: we + 1]
                mu = int((co[1:] - co[:-1]).max().item())
                mx = (me, mu)
            self._aux["maxima"] = mx
        return mx

    @property
    def device(self):
        return self.dev["node_ptr"].device

    def block_offsets(self) -> np.ndarray:
        """Per-window TC-block offsets: exclusive cumsum of win_partition
        (the 'counts and offsets' of north_star; the reference derives the
        SDDMM analogue tile_base at kernels.py:461-462)."""
        out = np.zeros(self.num_row_windows + 1, dtype=np.int64)
        np.cumsum(self.win_partition.astype(np.int64), out=out[1:])
        return out

    def transpose(self) -> "TransposedTiling":
        """A^T tiled with the same BlockConfig, plus the edge permutation
        (backward passes; cached)."""
        tt = self._aux.get("transpose")
        if tt is None:
            tt = _transpose(self)
            self._aux["transpose"] = tt
        return tt


@dataclass
class TransposedTiling:
    tiled: TiledGraph
    perm: object  # torch int32 tensor (u32 bits): edge k of A^T is edge perm[k] of A


def _stream_ptr():
    import torch

    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _sgt_device(ptr, cols, n: int, m: int, cfg: BlockConfig, graph) -> TiledGraph:
    import torch

    lib = _lib.load()
    dev = ptr.device
    W = -(-n // cfg.blk_h)
    wp = torch.empty(max(W, 1), dtype=torch.int32, device=dev)
    e2c = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    offs = torch.empty(W + 1, dtype=torch.int64, device=dev)
    wsb = int(lib.tcg_sgt_workspace_bytes(n, m, cfg.blk_h))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    cp = cols.data_ptr() if m else None
    # one ABI call (count + scan + fill enqueued back to back from C), no host
    # round trip: col_to_node is allocated at its upper bound M (U <= M) and
    # U = col_offsets[W] is read lazily, on the first use that needs it as a
    # host integer (TiledGraph.num_unique)
    c2n = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    _lib.check(lib.tcg_sgt(ptr.data_ptr(), cp, n, m, cfg.blk_h, cfg.blk_w, wp.data_ptr(),
                           e2c.data_ptr(), offs.data_ptr(), c2n.data_ptr(), ws.data_ptr(), wsb,
                           _stream_ptr()), "tcg_sgt")
    t = TiledGraph(graph, cfg, n, m, W)
    t.dev.update(node_ptr=ptr, edge_list=cols, win_partition=wp[:W], edge_to_col=e2c[:m],
                 col_offsets=offs, col_to_node=c2n)
    return t


class ShardSgt:
    """SGT of one row-window shard [wb, we) (windows are
    independent, so a rank translates only its own). Phase 1 (`count`) ranks
    the shard's edges and scans its unique counts from 0; the shard's total U_r
    is `total` (a device scalar). Phase 2 (`fill`) writes col_to_node at the
    global offsets once `base` = sum of the lower shards' totals is known (an
    exclusive scan of P integers: dist.translate_sharded all-gathers them).
    The result is a TiledGraph with global-sized arrays of which only the
    shard's windows / edges are filled -- bit for bit the whole-graph SGT
    restricted to the shard; kernels run on it with win_range = (wb, we)."""

    def __init__(self, g: CsrGraph, cfg: BlockConfig, win_range: tuple[int, int], device=None):
        import torch

        if not isinstance(cfg, BlockConfig):
            raise TypeError("cfg must be a BlockConfig")
        self.g, self.cfg = g, cfg
        self.ptr, self.cols, _ = g.device_arrays(device)
        n, m = g.num_nodes, g.num_edges
        self.W = -(-n // cfg.blk_h)
        wb, we = (int(win_range[0]), int(win_range[1]))
        if not 0 <= wb <= we <= self.W:
            raise IndexError(f"window range [{wb}, {we}) outside [0, {self.W})")
        self.wb, self.we = wb, we
        dev = self.ptr.device
        self.wp = torch.zeros(max(self.W, 1), dtype=torch.int32, device=dev)
        self.e2c = torch.zeros(max(m, 1), dtype=torch.int32, device=dev)
        self.offs = torch.zeros(self.W + 1, dtype=torch.int64, device=dev)
        self.c2n = torch.zeros(max(m, 1), dtype=torch.int32, device=dev)
        self._counted = self._filled = False

    def count(self) -> "ShardSgt":
        import torch

        lib = _lib.load()
        n, m = self.g.num_nodes, self.g.num_edges
        wsb = int(lib.tcg_sgt_workspace_bytes(n, m, self.cfg.blk_h))
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=self.ptr.device)
        _lib.check(lib.tcg_sgt_count_range(
            self.ptr.data_ptr(), self.cols.data_ptr() if m else None, n, m, self.cfg.blk_h,
            self.cfg.blk_w, self.wb, self.we, self.e2c.data_ptr(), self.offs.data_ptr(),
            self.wp.data_ptr(), ws.data_ptr(), wsb, _stream_ptr()), "tcg_sgt_count_range")
        self._counted = True
        return self

    @property
    def total(self):
        """U_r, the shard's unique-column count (device int64 scalar tensor)."""
        return self.offs[self.we: self.we + 1]

    def fill(self, base: int) -> TiledGraph:
        if not self._counted:
            self.count()
        n, m = self.g.num_nodes, self.g.num_edges
        _lib.check(_lib.load().tcg_sgt_fill_range(
            self.ptr.data_ptr(), self.cols.data_ptr() if m else None, n, m, self.cfg.blk_h,
            self.wb, self.we, int(base), self.e2c.data_ptr(), self.offs.data_ptr(),
            self.c2n.data_ptr(), _stream_ptr()), "tcg_sgt_fill_range")
        t = TiledGraph(self.g, self.cfg, n, m, self.W)
        t.dev.update(node_ptr=self.ptr, edge_list=self.cols, win_partition=self.wp[: self.W],
                     edge_to_col=self.e2c[:m], col_offsets=self.offs, col_to_node=self.c2n)
        t.shard_windows = (self.wb, self.we)
        return t


def translate_range(g: CsrGraph, cfg: BlockConfig, win_range, base: int = 0, device=None) -> TiledGraph:
    """SGT of the windows in `win_range` only, col_offsets shifted by `base`
    (see ShardSgt; base=0 with the full range is `translate`)."""
    return ShardSgt(g, cfg, win_range, device).count().fill(base)


def translate(g: CsrGraph, cfg: BlockConfig, device=None) -> TiledGraph:
    """GPU Sparse Graph Translation; bit-exact with the reference translate
    (sgt.py:101-137) for any BlockConfig."""
    if not isinstance(cfg, BlockConfig):
        raise TypeError("cfg must be a BlockConfig")
    ptr, cols, _ = g.device_arrays(device)
    return _sgt_device(ptr, cols, g.num_nodes, g.num_edges, cfg, g)


def csr_transpose_device(g: CsrGraph, device=None):
    """(A^T as a device-resident CsrGraph, perm): A^T edge k is A edge perm[k]
    (tcg_csr_transpose; the backward's graph)."""
    ptr, cols, _ = g.device_arrays(device)
    return _csr_transpose(ptr, cols, g.num_nodes, g.num_edges, g)


def _transpose(t: TiledGraph) -> TransposedTiling:
    g = t._require_graph()
    gt, perm = _csr_transpose(t.dev["node_ptr"], t.dev["edge_list"], t.num_nodes, t.num_edges, g)
    tt = _sgt_device(gt._ptr_d, gt._cols_d, t.num_nodes, t.num_edges, t.config, gt)
    return TransposedTiling(tt, perm)


def _csr_transpose(ptr, cols, n: int, m: int, g):
    import torch

    lib = _lib.load()
    dev = ptr.device
    ptr_t = torch.empty(n + 1, dtype=torch.int64, device=dev)
    cols_t = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    perm = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    wsb = int(lib.tcg_csr_transpose_workspace_bytes(n, m))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    _lib.check(lib.tcg_csr_transpose(ptr.data_ptr(), cols.data_ptr() if m else None, n, m,
                                     ptr_t.data_ptr(), cols_t.data_ptr(), perm.data_ptr(),
                                     ws.data_ptr(), wsb, _stream_ptr()), "tcg_csr_transpose")
    cols_t, perm = cols_t[:m], perm[:m]
    return _DeviceCsr(n, ptr_t, cols_t, g), perm


class _DeviceCsr(CsrGraph):
    """A CsrGraph whose arrays were built on the device (A^T); host views are
    materialised on demand."""

    def __init__(self, n, ptr_d, cols_d, parent):
        self.num_nodes = int(n)
        self._dev = {("csr", ptr_d.device.index): (ptr_d, cols_d, None)}
        self._ptr_d, self._cols_d = ptr_d, cols_d
        self.edge_values = None
        self._np = None

    def _host(self):
        if self._np is None:
            self._np = (self._ptr_d.cpu().numpy(), self._cols_d.cpu().numpy().view(np.uint32))
        return self._np

    @property
    def node_pointer(self):
        return self._host()[0]

    @node_pointer.setter
    def node_pointer(self, v):
        pass

    @property
    def edge_list(self):
        return self._host()[1]

    @edge_list.setter
    def edge_list(self, v):
        pass

    @property
    def num_edges(self) -> int:
        return int(self._cols_d.shape[0])


# ---- tile accounting (sgt.py:140-217; reporting, host-side) -----------------


def count_blocks_before(g: CsrGraph, cfg: BlockConfig, device=None) -> tuple[int, np.ndarray]:
    """Occupied blk_w-wide original-column buckets per window (sgt.py:140-157).
    With `device` it is the GPU structure count on the (GPU) SGT of g — the
    condensed columns keep each window's distinct neighbour set. The default
    is the GPU whenever CUDA is present; `device="cpu"` keeps the host count."""
    from .graph import _on_device

    if _on_device(device):
        t = translate(g, cfg, None if device in (None, "auto") else device)
        return structure_blocks_device(t, cfg.blk_w)
    n, bh, bw = g.num_nodes, cfg.blk_h, cfg.blk_w
    W = -(-n // bh)
    if g.num_edges == 0:
        return 0, np.zeros(W, dtype=np.int64)
    win = np.repeat(np.arange(n, dtype=np.int64), g.degrees()) // bh
    nb = -(-n // bw)
    uniq = np.unique(win * nb + g.edge_list.astype(np.int64) // bw)
    return int(uniq.shape[0]), np.bincount(uniq // nb, minlength=W)


def structure_blocks_device(t: TiledGraph, tile_width: int) -> tuple[int, np.ndarray]:
    """(total, per-window) distinct col_to_node // tile_width buckets on the
    GPU (tcg_structure_blocks)."""
    import torch

    if tile_width < 1:
        raise ValueError("tile_width must be >= 1")
    W = t.num_row_windows
    dev = t.dev["col_offsets"].device
    per = torch.zeros(max(W, 1), dtype=torch.int64, device=dev)
    tot = torch.zeros(1, dtype=torch.int64, device=dev)
    s = _lib.TcgTiling(t.num_nodes, t.num_edges, W, t.num_unique, t.config.blk_h, t.config.blk_w,
                       None, None, None, t.dev["col_offsets"].data_ptr(),
                       t.dev["col_to_node"].data_ptr() if t.num_unique else None,
                       None, None, 0, 0, None, None)
    _lib.check(_lib.load().tcg_structure_blocks(C.byref(s), int(tile_width), per.data_ptr(),
                                                tot.data_ptr(), _stream_ptr()),
               "tcg_structure_blocks")
    return int(tot.item()), per[:W].cpu().numpy()


def structure_blocks_before(t: TiledGraph, tile_width: int) -> int:
    """Occupied original-column buckets per window from the tiling structure
    alone (sgt.py:199-217); equals count_blocks_before on the source graph.
    Device-resident tilings count on the GPU."""
    if tile_width < 1:
        raise ValueError("tile_width must be >= 1")
    if t.dev:
        return structure_blocks_device(t, tile_width)[0]
    c2n = t.col_to_node
    if c2n.size == 0:
        return 0
    win = np.repeat(np.arange(t.num_row_windows, dtype=np.int64), np.diff(t.col_offsets))
    nb = -(-t.num_nodes // tile_width)
    return int(np.unique(win * nb + c2n.astype(np.int64) // tile_width).shape[0])


def count_blocks_after(t: TiledGraph) -> int:
    return int(t.win_partition.astype(np.int64).sum())


def reduction_ratio(before: int, after: int) -> float:
    return 0.0 if before == 0 else 1.0 - after / before


def block_columns(t: TiledGraph, window: int, block: int) -> np.ndarray:
    if not 0 <= window < t.num_row_windows:
        raise IndexError(f"window {window} out of range [0, {t.num_row_windows})")
    if not 0 <= block < int(t.win_partition[window]):
        raise IndexError(
            f"block {block} out of range [0, {int(t.win_partition[window])}) in window {window}")
    bw = t.config.blk_w
    lo = t.col_offsets[window] + block * bw
    hi = min(lo + bw, t.col_offsets[window + 1])
    return t.col_to_node[lo:hi].copy()


def paired_block_counts(t: TiledGraph) -> np.ndarray:
    """ceil(wp * blk_w / blk_h) square output tiles per window (sgt.py:190-198)."""
    bh, bw = t.config.blk_h, t.config.blk_w
    return (t.win_partition.astype(np.int64) * bw + bh - 1) // bh

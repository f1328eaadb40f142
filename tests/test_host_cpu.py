"""Host-side layout helpers and layer configuration (no GPU needed)."""

from __future__ import annotations

import pytest
import torch

from paper_2112_02052_b200 import dense, layers


@pytest.mark.parametrize("d,ld", [(47, 48), (22, 24), (16, 16), (40, 40), (7, 7), (3, 3)])
def test_rows_empty_padding(d, ld):
    x = dense.rows_empty(5, d, "cpu")
    assert x.shape == (5, d) and x.stride() == (ld, 1)
    assert dense.rows_ok(x) is x
    y = torch.zeros(d, 5).t()  # column-major view: copied into unit-stride rows
    z = dense.rows_ok(y)
    assert z is not y and z.stride(1) == 1 and torch.equal(z, y)


@pytest.mark.parametrize("fin,fout,order,agg_first", [
    (16, 47, "auto", True), (128, 16, "auto", False), (16, 16, "auto", False),
    (16, 7, "auto", False), (128, 16, "aggregate_first", True), (16, 47, "transform_first", False),
])
def test_gcnconv_order(fin, fout, order, agg_first):
    conv = layers.GCNConv(fin, fout, order=order)
    assert conv.aggregate_first is agg_first


def test_gcnconv_order_rejects_unknown():
    with pytest.raises(ValueError):
        layers.GCNConv(4, 4, order="sideways")


# ---- reference host API (no GPU): plan validation, metrics, compare, TiledGraph

import numpy as np  # noqa: E402

import paper_2112_02052_b200 as tcg  # noqa: E402
from paper_2112_02052_b200 import kernels  # noqa: E402


def test_validate_plan_messages():
    """The reference's messages (kernels.py:112-133; tests/test_kernels.py:259-269)."""
    TP = tcg.TaskPlan
    with pytest.raises(ValueError, match="overlap"):
        tcg.validate_plan(TP([(0, 0, 4), (0, 2, 2)], 1), 1, 4)
    with pytest.raises(ValueError, match="gap"):
        tcg.validate_plan(TP([(0, 0, 1), (0, 2, 2)], 1), 1, 4)
    with pytest.raises(ValueError, match="window 1"):
        tcg.validate_plan(TP([(0, 0, 4)], 1), 2, 4)
    with pytest.raises(ValueError, match=r"out of range \[0, 1\)"):
        tcg.validate_plan(TP([(1, 0, 4)], 1), 1, 4)
    with pytest.raises(ValueError, match=r"dim range \[2, 6\) invalid for D=4"):
        tcg.validate_plan(TP([(0, 0, 2), (0, 2, 4)], 1), 1, 4)
    with pytest.raises(ValueError, match=r"covers dims \[0, 3\) of window 0, need 4"):
        tcg.validate_plan(TP([(0, 0, 3)], 1), 1, 4)
    tcg.validate_plan(TP([(0, 0, 2), (0, 2, 2), (1, 0, 4)], 2), 2, 4)


def test_dim_chunks_reference_cases():
    """reference tests/test_kernels.py:250-256"""
    assert kernels._dim_chunks(40, 2, 16) == [(0, 32), (32, 8)]
    assert kernels._dim_chunks(64, 2, 16) == [(0, 32), (32, 32)]
    assert kernels._dim_chunks(40, 4, 16) == [(0, 16), (16, 16), (32, 8)]
    assert kernels._dim_chunks(16, 4, 16) == [(0, 4), (4, 4), (8, 4), (12, 4)]
    assert kernels._dim_chunks(3, 8, 16) == [(0, 1), (1, 1), (2, 1)]


def test_graph_stats_and_dense_memory():
    g = tcg.CsrGraph.from_edges([0, 0, 1, 2], [0, 3, 3, 1], 4, device="cpu")
    s = tcg.graph_stats(g, 2)
    assert (s.num_nodes, s.num_edges, s.avg_degree) == (4, 4, 1.0)
    assert s.dense_memory_bytes == tcg.dense_memory_bytes(4) == 64
    assert s.effective_computation == 0.25 and s.avg_edges_per_row_window == 2.0
    z = tcg.graph_stats(tcg.CsrGraph.from_edges([], [], 0, device="cpu"), 16)
    assert (z.avg_degree, z.effective_computation, z.avg_edges_per_row_window) == (0.0, 0.0, 0.0)
    with pytest.raises(ValueError, match="window_height"):
        tcg.graph_stats(g, 0)
    # reference criterion 6 (test_acceptance.py:183-187): 14,302.48 GB at N = 1,890,931
    n = 1_890_931
    big = tcg.CsrGraph(n, np.zeros(n + 1, dtype=np.int64), np.array([], dtype=np.uint32))
    assert abs(tcg.graph_stats(big, 16).dense_memory_bytes / 1e9 - 14302.48) <= 0.01


def test_compare_report():
    a = np.array([1.0, 2.0, 3.0], np.float32)
    r = tcg.compare(a, a)
    assert r.passed and r.max_abs_err == 0.0 and r.first_mismatch is None
    b = np.array([1.0, 2.5, 3.0], np.float32)
    r = tcg.compare(b, a, rel_tol=0.1)
    assert not r.passed and r.num_mismatch == 1 and r.first_mismatch == (1,)
    assert abs(r.max_rel_err - 0.25) < 1e-12 and "FAIL" in str(r)
    assert tcg.compare(b, a, abs_tol=0.5).passed
    with pytest.raises(ValueError, match="shape mismatch"):
        tcg.compare(a, a[:2])
    assert tcg.compare(np.zeros(0), np.zeros(0)).passed


def test_tiled_graph_reference_constructor():
    """TiledGraph(graph, config, num_nodes, num_edges, num_row_windows,
    win_partition, edge_to_col, col_offsets, col_to_node) as the reference
    dataclass orders its fields (sgt.py:43-66); structure-only accounting runs
    on the host arrays."""
    wp = np.array([1, 1], np.uint32)
    e2c = np.array([0, 1, 1, 0], np.uint32)
    co = np.array([0, 2, 3], np.int64)
    c2n = np.array([0, 3, 1], np.uint32)
    t = tcg.TiledGraph(None, tcg.BlockConfig(2, 2), 4, 4, 2, wp, e2c, co, c2n)
    assert np.array_equal(t.win_partition, wp) and np.array_equal(t.col_to_node, c2n)
    assert t.num_unique == 3 and t.unique_count(0) == 2
    assert np.array_equal(t.window_nodes(0), [0, 3])
    assert tcg.count_blocks_after(t) == 2
    assert np.array_equal(t.block_offsets(), [0, 1, 2])
    with pytest.raises(ValueError, match="structure only"):
        t.window_edge_range(0)

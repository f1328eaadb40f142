"""GPU parity: the CUDA path (through the C ABI) against the reference's own
outputs (golden fixtures) and the CPU oracle.

Bars: SGT arrays bit-exact; f32 SpMM/SDDMM bit-exact (the reference's exact
f32 contract); TF32 outputs within relative L2 <= 5e-3 (north_star) and the
reference's own per-element TF32 bound |tf32 - f32| <= 10*2^-10*sum|products|
+ 1e-7 (tests/test_kernels.py:124-134 of the reference)."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import GOLDEN, TF32_REL_L2, rel_l2

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def tcg():
    import paper_2112_02052_b200 as tcg

    return tcg


def _graph(tcg, ptr, cols, n):
    return tcg.CsrGraph(n, ptr, cols)


def test_quantize_tf32_bitwise(tcg):
    z = np.load(GOLDEN / "tf32_vectors.npz")
    got = tcg.quantize_tf32(z["x"])
    assert np.array_equal(got.view(np.uint32), z["q"].view(np.uint32))


def test_sgt_small_cases_bitwise(tcg, small_cases):
    for c in small_cases:
        g = _graph(tcg, small_cases.arr(c, "ptr"), small_cases.arr(c, "cols"), c["n"])
        t = tcg.translate(g, tcg.BlockConfig(c["blk_h"], c["blk_w"]))
        for k in ("win_partition", "edge_to_col", "col_offsets", "col_to_node"):
            assert np.array_equal(getattr(t, k), small_cases.arr(c, k)), (c["name"], k)
        assert np.array_equal(tcg.paired_block_counts(t), small_cases.arr(c, "paired"))


def test_sgt_big_window_path(tcg, oracle):
    """Windows with > 4096 edges take the bitmap path (csrc/sgt.cu)."""
    rng = np.random.default_rng(3)
    n = 30000
    src = np.concatenate([rng.integers(0, 16, 90000), rng.integers(0, n, 60000)])
    dst = rng.integers(0, n, src.shape[0])
    g = tcg.CsrGraph.from_edges(src, dst, n)
    for bh, bw in ((16, 8), (5, 3), (64, 8)):
        t = tcg.translate(g, tcg.BlockConfig(bh, bw))
        ref = oracle.translate(g.node_pointer, g.edge_list, n, bh, bw)
        for k, v in zip(("win_partition", "edge_to_col", "col_offsets", "col_to_node"), ref):
            assert np.array_equal(getattr(t, k), v), (bh, bw, k)


@pytest.mark.parametrize("shape", ["pubmed", "arxiv", "amazon0601"])
def test_sgt_full_shape_digests(tcg, digests, shape):
    d = digests[shape]
    g = tcg.synth.shaped_graph(shape)
    assert sha(g.node_pointer) == d["ptr"] and sha(g.edge_list) == d["cols"]
    t = tcg.translate(g, tcg.BlockConfig())
    for k in ("win_partition", "edge_to_col", "col_offsets", "col_to_node"):
        assert sha(getattr(t, k)) == d[k], k


def test_tcgt_golden_bytes(tcg, oracle):
    g = tcg.synth.gen_uniform(100, 4, 42)
    t = tcg.translate(g, tcg.BlockConfig())
    b = oracle.write_tcgt_bytes(16, 8, 100, g.num_edges, t.win_partition, t.edge_to_col,
                                t.col_offsets, t.col_to_node)
    assert b == (GOLDEN / "uniform100.tcgt").read_bytes()


def test_exact_f32_small_cases_bitwise(tcg, small_cases):
    for c in small_cases:
        g = _graph(tcg, small_cases.arr(c, "ptr"), small_cases.arr(c, "cols"), c["n"])
        t = tcg.translate(g, tcg.BlockConfig(c["blk_h"], c["blk_w"]))
        x, xs, f = small_cases.inputs(c)
        nm = (c["name"], c["blk_h"], c["blk_w"])
        assert np.array_equal(tcg.spmm(t, x), small_cases.arr(c, "spmm_f32")), nm
        assert np.array_equal(tcg.spmm(t, x, f=f), small_cases.arr(c, "spmm_w_f32")), nm
        s = tcg.sddmm(t, xs)
        assert np.array_equal(s, small_cases.arr(c, "sddmm_f32")), nm
        sm = tcg.segment_softmax(small_cases.arr(c, "sddmm_f32"), g.node_pointer)
        np.testing.assert_allclose(sm, small_cases.arr(c, "softmax"), rtol=2e-6, atol=1e-7)
        np.testing.assert_allclose(tcg.agnn_layer(t, x), small_cases.arr(c, "agnn_f32"),
                                   rtol=1e-5, atol=1e-5)


def _tf32_bound_ok(got, exact, scale):
    return np.all(np.abs(got.astype(np.float64) - exact) <= 10 * 2.0**-10 * scale + 1e-7)


def test_tf32_small_cases(tcg, small_cases, oracle):
    for c in small_cases:
        if not small_cases.has(c, "spmm_tf32"):
            continue
        ptr, cols = small_cases.arr(c, "ptr"), small_cases.arr(c, "cols")
        g = _graph(tcg, ptr, cols, c["n"])
        t = tcg.translate(g, tcg.BlockConfig())
        x, xs, f = small_cases.inputs(c)
        nm = c["name"]
        got = tcg.spmm(t, x, mode="tf32")
        ref = small_cases.arr(c, "spmm_tf32")
        assert rel_l2(got, ref) <= TF32_REL_L2, nm
        assert _tf32_bound_ok(got, small_cases.arr(c, "spmm_f32"),
                              oracle.spmm(ptr, cols, np.abs(x)).astype(np.float64)), nm
        got = tcg.spmm(t, x, f=f, mode="tf32")
        assert rel_l2(got, small_cases.arr(c, "spmm_w_tf32")) <= TF32_REL_L2, nm
        got = tcg.sddmm(t, xs, mode="tf32")
        assert rel_l2(got, small_cases.arr(c, "sddmm_tf32")) <= TF32_REL_L2, nm
        assert _tf32_bound_ok(got, small_cases.arr(c, "sddmm_f32"),
                              oracle.sddmm(ptr, cols, np.abs(xs)).astype(np.float64)), nm
        got = tcg.agnn_layer(t, x, mode="tf32")
        assert rel_l2(got, small_cases.arr(c, "agnn_tf32")) <= TF32_REL_L2, nm
        w, b = small_cases.gcn_params(c)
        got = tcg.gcn_layer(t, x, w, b)
        np.testing.assert_allclose(got, small_cases.arr(c, "gcn_f32"), rtol=1e-4, atol=1e-4)


def test_cora_golden(tcg, cora_golden):
    gd = cora_golden
    g = tcg.CsrGraph(2708, gd["ptr"], gd["cols"])
    t = tcg.translate(g, tcg.BlockConfig())
    x, f = gd["x"], gd["f"]
    assert np.array_equal(tcg.spmm(t, x), gd["spmm_f32"])
    assert np.array_equal(tcg.spmm(t, x, f=f), gd["spmm_w_f32"])
    assert np.array_equal(tcg.sddmm(t, x), gd["sddmm_f32"])
    assert rel_l2(tcg.spmm(t, x, mode="tf32"), gd["spmm_tf32"]) <= TF32_REL_L2
    assert rel_l2(tcg.spmm(t, x, f=f, mode="tf32"), gd["spmm_w_tf32"]) <= TF32_REL_L2
    assert rel_l2(tcg.sddmm(t, x, mode="tf32"), gd["sddmm_tf32"]) <= TF32_REL_L2
    assert rel_l2(tcg.agnn_layer(t, x, mode="tf32"), gd["agnn_tf32"]) <= TF32_REL_L2


@pytest.mark.parametrize("shape", ["pubmed", "arxiv", "amazon0601"])
def test_full_shape_exact_digests(tcg, digests, shape):
    """f32 SpMM/SDDMM at the full BASELINE shape are bit-identical to the
    reference's outputs (sha256 recorded from the reference itself)."""
    d = digests[shape]
    g = tcg.synth.shaped_graph(shape)
    t = tcg.translate(g, tcg.BlockConfig())
    for dim in (16, 32):
        x = tcg.synth.random_embeddings(g.num_nodes, dim, seed=2)
        assert sha(tcg.spmm(t, x)) == d[f"spmm_f32_d{dim}"], dim
        assert sha(tcg.sddmm(t, x)) == d[f"sddmm_f32_d{dim}"], dim


@pytest.mark.parametrize("dim", [16, 32, 40, 128])
def test_arxiv_tf32_vs_oracle(tcg, oracle, dim):
    g = tcg.synth.shaped_graph("arxiv")
    t = tcg.translate(g, tcg.BlockConfig())
    x = tcg.synth.random_embeddings(g.num_nodes, dim, seed=2)
    ref = oracle.spmm(g.node_pointer, g.edge_list, x, workers=8)
    assert rel_l2(tcg.spmm(t, x, mode="tf32"), ref) <= TF32_REL_L2
    ref_s = oracle.sddmm(g.node_pointer, g.edge_list, x, workers=8)
    assert rel_l2(tcg.sddmm(t, x, mode="tf32"), ref_s) <= TF32_REL_L2
    if dim == 32:
        ref_a = oracle.agnn_layer(g.node_pointer, g.edge_list, x, mode="f32")
        assert rel_l2(tcg.agnn_layer(t, x, mode="tf32"), ref_a) <= TF32_REL_L2


def test_validation_messages(tcg):
    g = tcg.CsrGraph.from_edges([0], [0], 2)
    t = tcg.translate(g, tcg.BlockConfig(2, 2))
    with pytest.raises(ValueError, match="16x8"):
        tcg.spmm(t, np.ones((2, 2), np.float32), mode="tf32")
    with pytest.raises(ValueError, match="embedding rows"):
        tcg.spmm(t, np.ones((3, 2), np.float32))
    with pytest.raises(ValueError, match="entries, expected"):
        tcg.spmm(t, np.ones((2, 2), np.float32), f=np.ones(3, np.float32))
    with pytest.raises(ValueError, match="engine"):
        tcg.spmm(t, np.ones((2, 2), np.float32), engine="cpu")
    t2 = tcg.TiledGraph(None, t.config, t.num_nodes, t.num_edges, t.num_row_windows, dev=t.dev)
    with pytest.raises(ValueError, match="structure only"):
        tcg.spmm(t2, np.ones((2, 2), np.float32))

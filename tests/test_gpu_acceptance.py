"""The reference's acceptance gate (tests/test_acceptance.py of the reference)
re-run against the B200 engine, plus its hypothesis property strategies
(tests/conftest.py:60-88 of the reference) driving GPU SGT and the exact f32
kernels against the oracle (bitwise)."""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN, TF32_REL_L2, rel_l2

pytestmark = pytest.mark.gpu

try:
    from hypothesis import given, settings
    from hypothesis import strategies as st
except ImportError:  # pragma: no cover
    given = None


@pytest.fixture(scope="module")
def tcg():
    import paper_2112_02052_b200 as tcg

    return tcg


CRITERION_1_DIMS = (16, 256, 1, 64, 2)


def criterion_1_cases(tcg):
    """50 seeded uniform graphs, N from 16 to 10,000 (geometric), degree drawn
    from [1, 32], D cycling 16/256/1/64/2 (reference test_acceptance.py:53-60)."""
    for i in range(50):
        n = round(16 * (10000 / 16) ** (i / 49))
        deg = int(np.random.default_rng(5000 + i).integers(1, 33))
        yield i, tcg.synth.gen_uniform(n, deg, 5000 + i), CRITERION_1_DIMS[i % 5]


def test_criterion_1_oracle_equivalence(tcg, oracle):
    """f32 SpMM / SDDMM on the tiled GPU engine bitwise equal to the CSR
    oracle fold on all 50 graphs (test_acceptance.py:76-98)."""
    for i, g, d in criterion_1_cases(tcg):
        t = tcg.translate(g, tcg.BlockConfig())
        x = tcg.synth.random_embeddings(g.num_nodes, d, 6000 + i)
        ref = oracle.spmm(g.node_pointer, g.edge_list, x)
        assert np.array_equal(tcg.spmm(t, x, workers=4), ref), i
        assert np.array_equal(tcg.ref_spmm(g, x), ref), i
        ref_s = oracle.sddmm(g.node_pointer, g.edge_list, x)
        assert np.array_equal(tcg.sddmm(t, x, workers=4), ref_s), i
        assert np.array_equal(tcg.ref_sddmm(g, x), ref_s), i
        if d in (16, 64):  # the TF32 engine on the same graphs, within tolerance
            yt = tcg.spmm(t, x, mode="tf32")
            assert rel_l2(yt, oracle.spmm(g.node_pointer, g.edge_list, x, mode="tf32")) \
                <= TF32_REL_L2, i


def _determinism_corpus(tcg):
    G = tcg.CsrGraph
    return [("four_node", G.from_edges([0, 0, 1, 2], [0, 3, 3, 1], 4)),
            ("empty", G.from_edges([], [], 48)),
            ("identity", G.from_edges(np.arange(37), np.arange(37), 37)),
            ("uniform", tcg.synth.gen_uniform(600, 8, 31)),
            ("powerlaw", tcg.synth.gen_powerlaw(400, 6, 32)),
            ("blockdense", tcg.synth.gen_blockdense(8, 3, 16, 33)),
            ("ragged", tcg.synth.gen_uniform(45, 3, 34))]


def test_criterion_2_sgt_correctness(tcg):
    """Independent re-derivation of each window's sorted unique neighbour set,
    win_partition = ceil(|set| / blk_w), and the bijection
    window_nodes(w)[edge_to_col[e]] == edge_list[e] (test_acceptance.py:101-118)."""
    for name, g in _determinism_corpus(tcg):
        for bh, bw in ((16, 8), (5, 3)):
            t = tcg.translate(g, tcg.BlockConfig(bh, bw))
            ptr, cols = g.node_pointer, g.edge_list
            rows = np.repeat(np.arange(g.num_nodes), np.diff(ptr))
            for w in range(t.num_row_windows):
                sel = (rows // bh) == w
                expect = np.unique(cols[sel].astype(np.int64))
                assert np.array_equal(t.window_nodes(w).astype(np.int64), expect), (name, w)
                assert int(t.win_partition[w]) == -(-expect.size // bw), (name, w)
            win = rows // bh
            got = t.col_to_node[t.col_offsets[win] + t.edge_to_col.astype(np.int64)]
            assert np.array_equal(got, cols), name


def test_criterion_3_block_reduction(tcg):
    """uniform 4096 / degree 8 / seed 97: 29,028 -> 4,147 blocks (the
    reference's published count, test_output.txt:15), and the planted-block
    sweep exact (test_acceptance.py:125-148)."""
    info = json.loads((GOLDEN / "aux.json").read_text())
    g = tcg.synth.gen_uniform(4096, 8, 97)
    cfg = tcg.BlockConfig(16, 8)
    before, _ = tcg.count_blocks_before(g, cfg)
    after = tcg.count_blocks_after(tcg.translate(g, cfg))
    assert (before, after) == (29028, 4147)
    assert (before, after) == (info["criterion3"]["before"], info["criterion3"]["after"])
    for dbw, want in info["criterion3_planted"].items():
        bd = tcg.synth.gen_blockdense(256, int(dbw), 16, 200 + int(dbw))
        t = tcg.translate(bd, cfg)
        assert bd.num_edges == want["edges"]
        assert int(tcg.paired_block_counts(t).sum()) == want["paired"] == 256 * int(dbw)
        assert tcg.count_blocks_after(t) == want["after"] == 2 * 256 * int(dbw)


def test_criterion_5_determinism(tcg):
    """Run-to-run and worker-count bitwise determinism, f32 and tf32
    (test_acceptance.py criterion 5; SURVEY 8(b) threading row)."""
    for name, g in _determinism_corpus(tcg):
        t = tcg.translate(g, tcg.BlockConfig())
        x = tcg.synth.random_embeddings(g.num_nodes, 24, 7)
        for mode in ("f32", "tf32"):
            base = tcg.spmm(t, x, mode=mode)
            for w in (1, 2, 8):
                assert np.array_equal(tcg.spmm(t, x, mode=mode, workers=w), base), (name, mode)
            bs = tcg.sddmm(t, x, mode=mode)
            assert np.array_equal(tcg.sddmm(t, x, mode=mode, workers=8), bs), (name, mode)
            ba = tcg.agnn_layer(t, x, mode=mode)
            assert np.array_equal(tcg.agnn_layer(t, x, mode=mode), ba), (name, mode)


def test_criterion_7_layer_composition(tcg):
    """GCN with identity weights is the aggregation; AGNN rows are convex
    combinations (softmax rows sum to 1); the 4-node hand trace."""
    g = tcg.CsrGraph.from_edges([0, 0, 1, 2], [0, 3, 3, 1], 4)
    t = tcg.translate(g, tcg.BlockConfig())
    x = np.array([[1, 0], [0, 1], [2, 2], [5, 5]], np.float32)
    assert np.array_equal(tcg.gcn_layer(t, x, np.eye(2, dtype=np.float32)), tcg.spmm(t, x))
    a = tcg.agnn_layer(t, x)
    np.testing.assert_allclose(a, [[4.928055, 4.910069], [5, 5], [0, 1], [0, 0]], rtol=1e-6)
    p = tcg.segment_softmax(tcg.sddmm(t, x), g.node_pointer)
    sums = np.add.reduceat(p, g.node_pointer[:-1][np.diff(g.node_pointer) > 0])
    np.testing.assert_allclose(sums, 1.0, rtol=1e-6)


if given is not None:

    @st.composite
    def csr_graphs(draw, max_nodes=40, max_edges=120):
        n = draw(st.integers(1, max_nodes))
        pairs = draw(st.lists(st.tuples(st.integers(0, n - 1), st.integers(0, n - 1)),
                              max_size=max_edges))
        return n, [p[0] for p in pairs], [p[1] for p in pairs]

    @settings(max_examples=60, deadline=None)
    @given(csr_graphs(), st.integers(1, 9), st.integers(1, 9), st.integers(1, 20))
    def test_property_sgt_and_exact_kernels(tcg, oracle, gdef, bh, bw, d):
        """Random graphs x random tile shapes: GPU SGT bitwise the oracle's,
        f32 SpMM / SDDMM bitwise the oracle fold, from_edges on the device
        bitwise the host normalisation."""
        n, src, dst = gdef
        g = tcg.CsrGraph.from_edges(src, dst, n)
        ptr, cols, _ = oracle.from_edges(src, dst, n)
        assert np.array_equal(g.node_pointer, ptr) and np.array_equal(g.edge_list, cols)
        t = tcg.translate(g, tcg.BlockConfig(bh, bw))
        ref = oracle.translate(ptr, cols, n, bh, bw)
        for k, v in zip(("win_partition", "edge_to_col", "col_offsets", "col_to_node"), ref):
            assert np.array_equal(getattr(t, k), v), k
        x = np.random.default_rng(n * 31 + d).standard_normal((n, d)).astype(np.float32)
        assert np.array_equal(tcg.spmm(t, x), oracle.spmm(ptr, cols, x))
        assert np.array_equal(tcg.sddmm(t, x), oracle.sddmm(ptr, cols, x))


def test_criterion_6_metrics_fidelity(tcg):
    """88 edges per 16-row window -> warps_per_block 2 (test_acceptance.py:189-201)."""
    src, dst = [], []
    for w in range(100):
        for r in range(16):
            for j in range(6 if r < 8 else 5):
                src.append(w * 16 + r)
                dst.append(j)
    g = tcg.CsrGraph.from_edges(src, dst, 1600)
    t = tcg.translate(g, tcg.BlockConfig())
    assert tcg.graph_stats(g, 16).avg_edges_per_row_window == pytest.approx(88.0)
    assert tcg.make_plan(t, 64).warps_per_block == 2

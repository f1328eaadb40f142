"""Pin the CPU oracle against the reference's own outputs (CPU, no GPU).

The fixtures were produced by running the reference package itself
(tests/golden/make_golden.py). Forward ops must match bit-for-bit; the
backward restatements (absent from the reference) are checked against a
float64 dense restatement."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import GOLDEN, rel_l2


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_quantize_tf32_golden(oracle):
    z = np.load(GOLDEN / "tf32_vectors.npz")
    got = oracle.quantize_tf32(z["x"])
    assert np.array_equal(got.view(np.uint32), z["q"].view(np.uint32))


def test_quantize_known_answers(oracle):
    assert float(oracle.quantize_tf32(np.float32(0.1))) == 0.0999755859375
    assert float(oracle.quantize_tf32(np.float32(-2.5))) == -2.5
    assert np.isinf(oracle.quantize_tf32(np.float32(3.4028235e38)))


def test_translate_small_cases(oracle, small_cases):
    for c in small_cases:
        ptr, cols = small_cases.arr(c, "ptr"), small_cases.arr(c, "cols")
        wp, e2c, offs, c2n = oracle.translate(ptr, cols, c["n"], c["blk_h"], c["blk_w"])
        assert np.array_equal(wp, small_cases.arr(c, "win_partition")), c["name"]
        assert np.array_equal(e2c, small_cases.arr(c, "edge_to_col")), c["name"]
        assert np.array_equal(offs, small_cases.arr(c, "col_offsets")), c["name"]
        assert np.array_equal(c2n, small_cases.arr(c, "col_to_node")), c["name"]
        assert wp.dtype == np.uint32 and e2c.dtype == np.uint32 and c2n.dtype == np.uint32
        assert offs.dtype == np.int64
        paired = oracle.paired_block_counts(wp, c["blk_h"], c["blk_w"])
        assert np.array_equal(paired, small_cases.arr(c, "paired"))
        assert oracle.count_blocks_before(ptr, cols, c["n"], c["blk_h"], c["blk_w"]) == \
            c["blocks_before"]


def test_kernels_small_cases_bitwise(oracle, small_cases):
    for c in small_cases:
        ptr, cols = small_cases.arr(c, "ptr"), small_cases.arr(c, "cols")
        x, xs, f = small_cases.inputs(c)
        name = c["name"]
        assert np.array_equal(oracle.spmm(ptr, cols, x), small_cases.arr(c, "spmm_f32")), name
        assert np.array_equal(oracle.spmm(ptr, cols, x, f=f),
                              small_cases.arr(c, "spmm_w_f32")), name
        s = oracle.sddmm(ptr, cols, xs)
        assert np.array_equal(s, small_cases.arr(c, "sddmm_f32")), name
        assert np.array_equal(oracle.segment_softmax(s, ptr), small_cases.arr(c, "softmax")), name
        assert np.array_equal(oracle.agnn_layer(ptr, cols, x), small_cases.arr(c, "agnn_f32")), name
        if small_cases.has(c, "spmm_tf32"):
            assert np.array_equal(oracle.spmm(ptr, cols, x, mode="tf32"),
                                  small_cases.arr(c, "spmm_tf32")), name
            assert np.array_equal(oracle.spmm(ptr, cols, x, f=f, mode="tf32"),
                                  small_cases.arr(c, "spmm_w_tf32")), name
            assert np.array_equal(oracle.sddmm(ptr, cols, xs, mode="tf32"),
                                  small_cases.arr(c, "sddmm_tf32")), name
            assert np.array_equal(oracle.agnn_layer(ptr, cols, x, mode="tf32"),
                                  small_cases.arr(c, "agnn_tf32")), name
            w, b = small_cases.gcn_params(c)
            got = oracle.gcn_layer(ptr, cols, x, w, b)
            np.testing.assert_allclose(got, small_cases.arr(c, "gcn_f32"), rtol=1e-5, atol=1e-5)


def test_cora_golden(oracle, cora_golden):
    g = cora_golden
    ptr, cols, _ = oracle.gen_uniform(2708, 10858 / 2708, seed=1)
    assert np.array_equal(ptr, g["ptr"]) and np.array_equal(cols, g["cols"])
    wp, e2c, offs, c2n = oracle.translate(ptr, cols, 2708, 16, 8)
    for k, v in dict(win_partition=wp, edge_to_col=e2c, col_offsets=offs, col_to_node=c2n).items():
        assert np.array_equal(v, g[k]), k
    x = oracle.random_embeddings(2708, 16, seed=2)
    assert np.array_equal(x, g["x"])
    for mode in ("f32", "tf32"):
        assert np.array_equal(oracle.spmm(ptr, cols, x, mode=mode), g[f"spmm_{mode}"])
        assert np.array_equal(oracle.spmm(ptr, cols, x, f=g["f"], mode=mode), g[f"spmm_w_{mode}"])
        assert np.array_equal(oracle.sddmm(ptr, cols, x, mode=mode), g[f"sddmm_{mode}"])
        assert np.array_equal(oracle.agnn_layer(ptr, cols, x, mode=mode), g[f"agnn_{mode}"])


def test_tcgt_bytes(oracle):
    ptr, cols, _ = oracle.gen_uniform(100, 4, 42)
    wp, e2c, offs, c2n = oracle.translate(ptr, cols, 100, 16, 8)
    b = oracle.write_tcgt_bytes(16, 8, 100, cols.shape[0], wp, e2c, offs, c2n)
    assert b == (GOLDEN / "uniform100.tcgt").read_bytes()
    ptr, cols, _ = oracle.from_edges([0, 0, 1, 2], [0, 3, 3, 1], 4)
    wp, e2c, offs, c2n = oracle.translate(ptr, cols, 4, 2, 2)
    assert oracle.write_tcgt_bytes(2, 2, 4, 4, wp, e2c, offs, c2n) == \
        (GOLDEN / "tiny.tcgt").read_bytes()


@pytest.mark.parametrize("shape", ["pubmed", "arxiv"])
def test_full_shape_digests(oracle, digests, shape):
    d = digests[shape]
    ptr, cols, _ = oracle.gen_uniform(d["n"], {"pubmed": 88676, "arxiv": 1166243}[shape] / d["n"],
                                      seed=1)
    assert sha(ptr) == d["ptr"] and sha(cols) == d["cols"]
    wp, e2c, offs, c2n = oracle.translate(ptr, cols, d["n"], 16, 8)
    assert sha(wp) == d["win_partition"] and sha(e2c) == d["edge_to_col"]
    assert sha(offs) == d["col_offsets"] and sha(c2n) == d["col_to_node"]
    x = oracle.random_embeddings(d["n"], 16, seed=2)
    assert sha(oracle.spmm(ptr, cols, x, workers=4)) == d["spmm_f32_d16"]
    assert sha(oracle.sddmm(ptr, cols, x, workers=4)) == d["sddmm_f32_d16"]


def test_hand_traces(oracle):
    ptr, cols, _ = oracle.from_edges([0, 0, 1, 2], [0, 3, 3, 1], 4)
    wp, e2c, offs, c2n = oracle.translate(ptr, cols, 4, 2, 2)
    assert wp.tolist() == [1, 1] and e2c.tolist() == [0, 1, 1, 0]
    assert c2n.tolist() == [0, 3, 1] and offs.tolist() == [0, 2, 3]
    x = np.array([[1, 0], [0, 1], [2, 2], [5, 5]], dtype=np.float32)
    assert oracle.spmm(ptr, cols, x).tolist() == [[6, 5], [5, 5], [0, 1], [0, 0]]
    assert oracle.sddmm(ptr, cols, x).tolist() == [1, 5, 5, 2]


def test_csr_transpose_matches_from_edges(oracle):
    ptr, cols, _ = oracle.gen_uniform(300, 5, seed=7)
    rows = np.repeat(np.arange(300), np.diff(ptr))
    pt, ct, perm = oracle.csr_transpose(ptr, cols, 300)
    p2, c2, _ = oracle.from_edges(cols.astype(np.int64), rows, 300)
    assert np.array_equal(pt, p2) and np.array_equal(ct, c2)
    assert np.array_equal(perm, np.lexsort((rows, cols)))


def _dense_agnn_f64(ptr, cols, z):
    n = ptr.shape[0] - 1
    rows = np.repeat(np.arange(n), np.diff(ptr))
    z = z.astype(np.float64)
    s = (z[rows] * z[cols]).sum(1)
    p = np.zeros_like(s)
    for i in range(n):
        a, b = ptr[i], ptr[i + 1]
        if b > a:
            e = np.exp(s[a:b] - s[a:b].max())
            p[a:b] = e / e.sum()
    y = np.zeros_like(z)
    np.add.at(y, rows, p[:, None] * z[cols])
    return y


def test_agnn_backward_restatement(oracle):
    """Backward parity unpinned by the reference: check the restated
    gradient against central finite differences of a float64 forward."""
    ptr, cols, _ = oracle.gen_uniform(40, 3, seed=5)
    rng = np.random.default_rng(0)
    z = rng.standard_normal((40, 4)).astype(np.float32)
    gy = rng.standard_normal((40, 4)).astype(np.float32)
    p = oracle.segment_softmax(oracle.sddmm(ptr, cols, z), ptr)
    dz = oracle.agnn_backward(ptr, cols, z, p, gy)
    eps = 1e-6
    num = np.zeros((40, 4))
    z64 = z.astype(np.float64)
    for i in range(40):
        for k in range(4):
            zp, zm = z64.copy(), z64.copy()
            zp[i, k] += eps
            zm[i, k] -= eps
            num[i, k] = ((_dense_agnn_f64(ptr, cols, zp) - _dense_agnn_f64(ptr, cols, zm))
                         * gy).sum() / (2 * eps)
    assert rel_l2(dz, num) < 1e-5


def test_spmm_transpose_restatement(oracle):
    ptr, cols, _ = oracle.gen_uniform(200, 4, seed=9)
    n = 200
    a = np.zeros((n, n))
    rows = np.repeat(np.arange(n), np.diff(ptr))
    f = np.random.default_rng(1).random(cols.shape[0]).astype(np.float32)
    a[rows, cols] = f
    g = np.random.default_rng(2).standard_normal((n, 5)).astype(np.float32)
    got = oracle.spmm_transpose(ptr, cols, g, f=f)
    assert rel_l2(got, a.T @ g) < 1e-6


def test_softmax_backward_restatement(oracle):
    ptr = np.array([0, 3, 3, 5], dtype=np.int64)
    p = oracle.segment_softmax(np.array([1, 2, 3, -1, 0.5], np.float32), ptr)
    dp = np.array([0.3, -1, 2, 0.1, 0.4], np.float32)
    ds = oracle.softmax_backward(p, dp, ptr)
    # row-wise Jacobian-vector product of softmax
    for a, b in ((0, 3), (3, 5)):
        pp = p[a:b].astype(np.float64)
        jac = np.diag(pp) - np.outer(pp, pp)
        np.testing.assert_allclose(ds[a:b], jac @ dp[a:b], rtol=1e-5, atol=1e-7)

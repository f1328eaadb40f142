"""Block-stream engine (csrc/stream.cu) against the oracle.

The stream engine takes every TF32 SpMM whose feature chunks are multiples of
8 (NT = 4 / 2 / 1 launches), the dual A^T form of the AGNN backward, and the
fused AGNN forward / one-pass backward / SDDMM at D <= 32 (multiples of 4). These cases pin it: chunk
splits (8 ... 128 features), bias / accumulate / shard row offsets, graphs
with hub windows (> 16 blocks: the fragment re-load path; > 255 edges: the
fused kernels hand over to the window engine), empty windows, the block
stream arrays themselves, and the arxiv shape against the exact-f32 path.
Tolerance: TF32 rel-L2 5e-3 (tests/conftest.py).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import TF32_REL_L2, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_2112_02052_b200 as tcg
    from paper_2112_02052_b200 import kernels, layers

    torch.backends.cuda.matmul.allow_tf32 = False
    return tcg, kernels, layers, torch


def _graph(tcg, kind, n, deg, seed):
    if kind == "uniform":
        return tcg.synth.gen_uniform(n, deg, seed)
    if kind == "powerlaw":
        return tcg.synth.gen_powerlaw(n, deg, seed)
    # hub rows: a few rows with hundreds of neighbours plus empty windows
    rng = np.random.default_rng(seed)
    src = np.concatenate([rng.integers(0, n, n * deg), np.repeat(np.arange(3), 300),
                          np.full(400, n // 2)])
    dst = np.concatenate([rng.integers(0, n, n * deg), rng.integers(0, n, 900),
                          rng.integers(0, n, 400)])
    keep = (src < 64) | (src >= 96)  # rows 64..95: two empty windows
    return tcg.CsrGraph.from_edges(src[keep], dst[keep], n)


def test_block_stream_arrays(env, oracle):
    tcg, _, _, torch = env
    g = tcg.synth.gen_uniform(777, 5, 3)
    t = tcg.translate(g, tcg.BlockConfig())
    t.abi()
    bo = t.dev["block_offsets"].cpu().numpy()
    assert np.array_equal(bo, t.block_offsets())
    cs = t.dev["col_stream"].cpu().numpy().view(np.uint32)
    tb = int(bo[-1])
    for w in range(t.num_row_windows):
        nodes = t.window_nodes(w)
        for b in range(bo[w], bo[w + 1]):
            for i in range(8):
                c = (b - bo[w]) * 8 + (i >> 1) + 4 * (i & 1)
                want = nodes[c] if c < len(nodes) else nodes[0]
                assert cs[8 * b + i] == want
    assert cs.size == 8 * (tb + 16)
    # pair stream (16-wide SpMM, two blocks per step): windows padded to even
    po = t.dev["pair_offsets"].cpu().numpy()
    wp = t.win_partition.astype(np.int64)
    assert np.array_equal(np.diff(po), wp + (wp & 1)) and po[0] == 0
    ps = t.dev["pair_stream"].cpu().numpy().view(np.uint32)
    for w in range(t.num_row_windows):
        nodes = t.window_nodes(w)
        for b in range(po[w], po[w + 1]):
            for i in range(8):
                c = (b - po[w]) * 8 + (i >> 1) + 4 * (i & 1)
                assert ps[8 * b + i] == (nodes[c] if c < len(nodes) else nodes[0])
    assert ps.size == 8 * (int(po[-1]) + 16)


_PAIR_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import torch
import paper_2112_02052_b200 as tcg
from paper_2112_02052_b200.kernels import spmm_device
out = []
for n, deg, d, seed in ((3001, 7, 16, 1), (2000, 40, 16, 2), (777, 3, 12, 3), (1500, 9, 48, 4),
                        (2500, 8, 32, 5), (1200, 11, 64, 6)):
    g = tcg.synth.gen_uniform(n, deg, seed)
    t = tcg.translate(g, tcg.BlockConfig())
    rng = np.random.default_rng(seed)
    x = torch.from_numpy(rng.standard_normal((n, d)).astype(np.float32)).cuda()
    w = torch.from_numpy(rng.random(g.num_edges).astype(np.float32)).cuda()
    out.append(spmm_device(t, x, w, mode="tf32").cpu().numpy())
    if d == 32:  # the dual form of the AGNN backward's A^T pass
        x2 = torch.from_numpy(rng.standard_normal((n, d)).astype(np.float32)).cuda()
        w2 = torch.from_numpy(rng.random(g.num_edges).astype(np.float32)).cuda()
        out.append(spmm_device(t, x, w, x2=x2, weights2=w2, mode="tf32").cpu().numpy())
np.save(sys.argv[2], np.concatenate([o.ravel() for o in out]))
"""


def test_pair_steps_bitwise_equal_single_block_steps(tmp_path):
    """The 16-wide two-blocks-per-step path (pair stream) is the same mma
    sequence per window as the one-block-per-step path (TCG_NO_PAIRS=1): the
    results are bitwise equal, incl. 40-edge windows (BIG staging), a masked
    12-wide chunk, a 48-wide operand's 16-wide tail, 32 / 64-wide operands
    (32-wide pair steps) and the two-operand (dual) form."""
    import os
    import subprocess
    import sys

    from conftest import ROOT

    res = []
    for k, env in enumerate(({}, {"TCG_NO_PAIRS": "1"})):
        f = tmp_path / f"o{k}.npy"
        r = subprocess.run([sys.executable, "-c", _PAIR_SCRIPT, str(ROOT), str(f)],
                           env=dict(os.environ, **env), capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        res.append(np.load(f))
    assert np.array_equal(res[0], res[1])


@pytest.mark.parametrize("dim", [3, 7, 8, 16, 22, 24, 32, 40, 47, 64, 100, 128])
@pytest.mark.parametrize("kind", ["uniform", "hub"])
def test_stream_spmm_dims(env, oracle, dim, kind):
    tcg, kernels, _, torch = env
    g = _graph(tcg, kind, 3000, 6, 5)
    t = tcg.translate(g, tcg.BlockConfig())
    rng = np.random.default_rng(dim)
    x = rng.standard_normal((g.num_nodes, dim)).astype(np.float32)
    w = rng.random(g.num_edges).astype(np.float32)
    y = kernels.spmm_device(t, torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda())
    ref = oracle.spmm(g.node_pointer, g.edge_list, x, f=w)
    assert rel_l2(y.cpu().numpy(), ref) <= TF32_REL_L2


@pytest.mark.parametrize("dim", [7, 47])
def test_stream_spmm_masked_tail_bias_accumulate(env, oracle, dim):
    """Odd widths (GCN class counts): unaligned rows, masked last chunk, bias,
    accumulate and a shard row offset."""
    tcg, kernels, _, torch = env
    g = tcg.synth.gen_uniform(1500, 6, 2)
    t = tcg.translate(g, tcg.BlockConfig())
    rng = np.random.default_rng(dim)
    x = rng.standard_normal((1500, dim)).astype(np.float32)
    b = rng.standard_normal(dim).astype(np.float32)
    y0 = rng.standard_normal((1500, dim)).astype(np.float32)
    ref = oracle.spmm(g.node_pointer, g.edge_list, x) + b + y0
    out = torch.from_numpy(y0.copy()).cuda()
    kernels.spmm_device(t, torch.from_numpy(x).cuda(), out=out, bias=torch.from_numpy(b).cuda(),
                        accumulate=True)
    assert rel_l2(out.cpu().numpy(), ref) <= TF32_REL_L2
    W = t.num_row_windows
    wb, we = W // 2, W
    r0, r1 = wb * 16, 1500
    slab = torch.from_numpy(y0[r0:r1].copy()).cuda()
    kernels.spmm_device(t, torch.from_numpy(x).cuda(), out=slab, bias=torch.from_numpy(b).cuda(),
                        accumulate=True, win_range=(wb, we), y_row0=r0)
    assert rel_l2(slab.cpu().numpy(), ref[r0:r1]) <= TF32_REL_L2


def test_stream_spmm_bias_accumulate_shard(env, oracle):
    tcg, kernels, _, torch = env
    g = tcg.synth.gen_uniform(2500, 7, 9)
    t = tcg.translate(g, tcg.BlockConfig())
    rng = np.random.default_rng(2)
    x = rng.standard_normal((2500, 32)).astype(np.float32)
    b = rng.standard_normal(32).astype(np.float32)
    y0 = rng.standard_normal((2500, 32)).astype(np.float32)
    ref = oracle.spmm(g.node_pointer, g.edge_list, x) + b + y0
    xt, bt = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    # full range, accumulate + bias
    out = torch.from_numpy(y0.copy()).cuda()
    kernels.spmm_device(t, xt, out=out, bias=bt, accumulate=True)
    assert rel_l2(out.cpu().numpy(), ref) <= TF32_REL_L2
    # two shards writing into row slabs at their own row offsets
    W = t.num_row_windows
    for wb, we in ((0, W // 3), (W // 3, W)):
        r0, r1 = wb * 16, min(we * 16, 2500)
        slab = torch.from_numpy(y0[r0:r1].copy()).cuda()
        kernels.spmm_device(t, xt, out=slab, bias=bt, accumulate=True, win_range=(wb, we),
                            y_row0=r0)
        assert rel_l2(slab.cpu().numpy(), ref[r0:r1]) <= TF32_REL_L2


def test_stream_dual_spmm(env, oracle):
    tcg, kernels, _, torch = env
    g = tcg.synth.gen_uniform(3000, 6, 13)
    t = tcg.translate(g, tcg.BlockConfig())
    rng = np.random.default_rng(4)
    x1 = rng.standard_normal((3000, 32)).astype(np.float32)
    x2 = rng.standard_normal((3000, 32)).astype(np.float32)
    w1 = rng.random(g.num_edges).astype(np.float32)
    w2 = rng.standard_normal(g.num_edges).astype(np.float32)
    y = kernels.spmm_device(t, torch.from_numpy(x1).cuda(), torch.from_numpy(w1).cuda(),
                            x2=torch.from_numpy(x2).cuda(), weights2=torch.from_numpy(w2).cuda())
    ref = (oracle.spmm(g.node_pointer, g.edge_list, x1, f=w1)
           + oracle.spmm(g.node_pointer, g.edge_list, x2, f=w2))
    assert rel_l2(y.cpu().numpy(), ref) <= TF32_REL_L2


@pytest.mark.parametrize("kind", ["uniform", "powerlaw", "hub"])
def test_stream_agnn_forward_backward(env, oracle, kind):
    tcg, kernels, layers, torch = env
    g = _graph(tcg, kind, 4000, 7, 21)
    t = tcg.translate(g, tcg.BlockConfig())
    rng = np.random.default_rng(6)
    z = rng.standard_normal((g.num_nodes, 32)).astype(np.float32)
    gy = rng.standard_normal((g.num_nodes, 32)).astype(np.float32)
    zt = torch.from_numpy(z).cuda()
    y, p = kernels.agnn_forward_device(t, zt)
    ptr, cols = g.node_pointer, g.edge_list
    p_ref = oracle.segment_softmax(oracle.sddmm(ptr, cols, z), ptr)
    y_ref = oracle.spmm(ptr, cols, z, f=p_ref)
    assert rel_l2(p.cpu().numpy()[: g.num_edges], p_ref) <= TF32_REL_L2
    assert rel_l2(y.cpu().numpy(), y_ref) <= TF32_REL_L2
    # one-pass backward (rs = <G, Y>) against the restated gradient
    gyt = torch.from_numpy(gy).cuda()
    dz_a, ds = kernels.agnn_backward_device(t, zt, gyt, p, y_fwd=y)
    dp = oracle.sddmm(ptr, cols, gy, z)
    ds_ref = oracle.softmax_backward(p_ref, dp, ptr)
    assert rel_l2(ds.cpu().numpy()[: g.num_edges], ds_ref) <= TF32_REL_L2
    assert rel_l2(dz_a.cpu().numpy(), oracle.spmm(ptr, cols, z, f=ds_ref)) <= TF32_REL_L2
    zt.requires_grad_(True)
    out = layers.AgnnAggregate.apply(zt, t, "tf32")
    out.backward(gyt)
    dz_ref = oracle.agnn_backward(ptr, cols, z, p_ref, gy)
    assert rel_l2(zt.grad.cpu().numpy(), dz_ref) <= TF32_REL_L2


def test_stream_arxiv_against_exact(env):
    """Full arxiv shape: the TF32 stream SpMM / fused AGNN against the exact-f32
    CUDA-core path (itself bitwise = the reference f32 fold on small cases)."""
    tcg, kernels, _, torch = env
    g = tcg.synth.shaped_graph("arxiv")
    t = tcg.translate(g, tcg.BlockConfig())
    gen = torch.Generator(device="cuda").manual_seed(0)
    z = torch.randn(g.num_nodes, 32, device="cuda", generator=gen)
    w = torch.rand(g.num_edges, device="cuda", generator=gen)
    y_tc = kernels.spmm_device(t, z, w)
    y_ex = kernels.spmm_device(t, z, w, mode="f32")
    assert rel_l2(y_tc.cpu().numpy(), y_ex.cpu().numpy()) <= TF32_REL_L2
    y_f, p_f = kernels.agnn_forward_device(t, z)
    from paper_2112_02052_b200 import _lib

    p_ex = kernels.sddmm_device(t, z, mode="f32", epilogue=_lib.EPI_SOFTMAX)
    y_ex = kernels.spmm_device(t, z, p_ex, mode="f32")
    assert rel_l2(p_f.cpu().numpy(), p_ex.cpu().numpy()) <= TF32_REL_L2
    assert rel_l2(y_f.cpu().numpy(), y_ex.cpu().numpy()) <= TF32_REL_L2


@pytest.mark.parametrize("kind", ["uniform", "powerlaw", "hub"])
def test_stream_sddmm_epilogues(env, oracle, kind):
    tcg, kernels, _, torch = env
    from paper_2112_02052_b200 import _lib

    g = _graph(tcg, kind, 3000, 7, 8)
    t = tcg.translate(g, tcg.BlockConfig())
    rng = np.random.default_rng(9)
    xa = rng.standard_normal((g.num_nodes, 32)).astype(np.float32)
    xb = rng.standard_normal((g.num_nodes, 32)).astype(np.float32)
    ptr, cols = g.node_pointer, g.edge_list
    xat, xbt = torch.from_numpy(xa).cuda(), torch.from_numpy(xb).cuda()
    s = kernels.sddmm_device(t, xat, xbt)
    s_ref = oracle.sddmm(ptr, cols, xa, xb)
    assert rel_l2(s.cpu().numpy(), s_ref) <= TF32_REL_L2
    p = kernels.sddmm_device(t, xat, epilogue=_lib.EPI_SOFTMAX)
    p_ref = oracle.segment_softmax(oracle.sddmm(ptr, cols, xa), ptr)
    assert rel_l2(p.cpu().numpy(), p_ref) <= TF32_REL_L2
    ds = kernels.sddmm_device(t, xat, xbt, epilogue=_lib.EPI_SOFTMAX_BWD,
                              aux=torch.from_numpy(p_ref).cuda())
    ds_ref = oracle.softmax_backward(p_ref, s_ref, ptr)
    assert rel_l2(ds.cpu().numpy(), ds_ref) <= TF32_REL_L2


def _kernel_names(torch, fn):
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    return {e.name for e in prof.events()}


@pytest.mark.parametrize("dim", [4, 8, 16, 20, 28])
@pytest.mark.parametrize("kind", ["uniform", "hub"])
def test_stream_agnn_masked_dims(env, oracle, dim, kind):
    """D < 32 (multiples of 4) on the fused AGNN / SDDMM kernels: the D = 32
    layout with the missing features zero-filled by the copies and never
    stored. Forward, one-pass backward and the SDDMM epilogues against the
    oracle; the launches are the stream kernels (not the window engine)."""
    tcg, kernels, layers, torch = env
    from paper_2112_02052_b200 import _lib

    g = _graph(tcg, kind, 3000, 7, 30 + dim)
    t = tcg.translate(g, tcg.BlockConfig())
    rng = np.random.default_rng(dim)
    z = rng.standard_normal((g.num_nodes, dim)).astype(np.float32)
    gy = rng.standard_normal((g.num_nodes, dim)).astype(np.float32)
    ptr, cols = g.node_pointer, g.edge_list
    zt, gyt = torch.from_numpy(z).cuda(), torch.from_numpy(gy).cuda()
    res = {}
    names = _kernel_names(torch, lambda: res.update(fwd=kernels.agnn_forward_device(t, zt)))
    y, p = res["fwd"]
    if kind == "uniform":  # the hub graph's > 255-edge windows go to the window engine
        assert any("agnn_stream" in n for n in names), names
    p_ref = oracle.segment_softmax(oracle.sddmm(ptr, cols, z), ptr)
    assert rel_l2(p.cpu().numpy()[: g.num_edges], p_ref) <= TF32_REL_L2
    assert rel_l2(y.cpu().numpy(), oracle.spmm(ptr, cols, z, f=p_ref)) <= TF32_REL_L2
    dz_a, ds = kernels.agnn_backward_device(t, zt, gyt, p, y_fwd=y)
    ds_ref = oracle.softmax_backward(p_ref, oracle.sddmm(ptr, cols, gy, z), ptr)
    assert rel_l2(ds.cpu().numpy()[: g.num_edges], ds_ref) <= TF32_REL_L2
    assert rel_l2(dz_a.cpu().numpy(), oracle.spmm(ptr, cols, z, f=ds_ref)) <= TF32_REL_L2
    zg = zt.clone().requires_grad_(True)
    layers.AgnnAggregate.apply(zg, t, "tf32").backward(gyt)
    assert rel_l2(zg.grad.cpu().numpy(), oracle.agnn_backward(ptr, cols, z, p_ref, gy)) <= TF32_REL_L2
    s = kernels.sddmm_device(t, zt, gyt)
    s_ref = oracle.sddmm(ptr, cols, z, gy)
    assert rel_l2(s.cpu().numpy(), s_ref) <= TF32_REL_L2
    ps = kernels.sddmm_device(t, zt, epilogue=_lib.EPI_SOFTMAX)
    assert rel_l2(ps.cpu().numpy(), p_ref) <= TF32_REL_L2


@pytest.mark.parametrize("dim", [16, 32, 40, 47])
def test_stream_spmm_big_windows(env, oracle, dim):
    """Products-like windows (~480 edges): the shared-memory edge-staging variant,
    including windows past its 512-edge staging capacity (global fallback)."""
    tcg, kernels, _, torch = env
    rng = np.random.default_rng(dim)
    n = 2000
    src = np.concatenate([rng.integers(0, n, n * 30), np.repeat(np.arange(16), 80)])
    dst = np.concatenate([rng.integers(0, n, n * 30), rng.integers(0, n, 16 * 80)])
    g = tcg.CsrGraph.from_edges(src, dst, n)
    t = tcg.translate(g, tcg.BlockConfig())
    assert g.num_edges > 256 * t.num_row_windows  # the staging variant's threshold
    x = rng.standard_normal((n, dim)).astype(np.float32)
    x2 = rng.standard_normal((n, dim)).astype(np.float32)
    w = rng.random(g.num_edges).astype(np.float32)
    w2 = rng.standard_normal(g.num_edges).astype(np.float32)
    ptr, cols = g.node_pointer, g.edge_list
    y = kernels.spmm_device(t, torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda())
    assert rel_l2(y.cpu().numpy(), oracle.spmm(ptr, cols, x, f=w)) <= TF32_REL_L2
    y1 = kernels.spmm_device(t, torch.from_numpy(x).cuda())
    assert rel_l2(y1.cpu().numpy(), oracle.spmm(ptr, cols, x)) <= TF32_REL_L2
    yd = kernels.spmm_device(t, torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(),
                             x2=torch.from_numpy(x2).cuda(), weights2=torch.from_numpy(w2).cuda())
    ref = oracle.spmm(ptr, cols, x, f=w) + oracle.spmm(ptr, cols, x2, f=w2)
    assert rel_l2(yd.cpu().numpy(), ref) <= TF32_REL_L2


_TMA_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import torch
import paper_2112_02052_b200 as tcg
from paper_2112_02052_b200 import _lib
from oracle import tcg_oracle as oracle
from paper_2112_02052_b200.kernels import spmm_device
worst = 0.0
for n, deg, d, seed in ((3001, 7, 32, 1), (1500, 12, 64, 2), (777, 3, 40, 3)):
    g = tcg.synth.gen_uniform(n, deg, seed)
    t = tcg.translate(g, tcg.BlockConfig())
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, d)).astype(np.float32)
    w = rng.random(g.num_edges).astype(np.float32)
    c0 = _lib.launch_count()
    y = spmm_device(t, torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), mode="tf32")
    torch.cuda.synchronize()
    assert _lib.launch_count() > c0
    ref = oracle.spmm(g.node_pointer, g.edge_list, x, f=w)
    e = float(np.linalg.norm(y.cpu().numpy() - ref) / np.linalg.norm(ref))
    worst = max(worst, e)
print(worst)
"""


def test_tma_gather_engine_opt_in(tmp_path):
    """The opt-in TMA tile::gather4 SpMM (TCG_SPMM_ENGINE=tma; measured slower
    than the cp.async ring, kept as the A/B of DESIGN.md section 3) matches
    the oracle, including a 64-wide (two chunk) and a masked 40-wide operand."""
    import os
    import subprocess
    import sys

    from conftest import ROOT

    env = dict(os.environ, TCG_SPMM_ENGINE="tma")
    r = subprocess.run([sys.executable, "-c", _TMA_SCRIPT, str(ROOT)], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert float(r.stdout.strip().splitlines()[-1]) <= TF32_REL_L2


def test_ws_gather_engine_opt_in(tmp_path):
    """The opt-in warp-specialised TMA gather4 SpMM (TCG_SPMM_ENGINE=ws: one
    producer warp per CTA; measured slower, profiles/r02/spmm_engines_ab.txt)
    matches the oracle (32- and 64-wide operands; the masked 40-wide tail takes
    the ring)."""
    import os
    import subprocess
    import sys

    from conftest import ROOT

    env = dict(os.environ, TCG_SPMM_ENGINE="ws")
    r = subprocess.run([sys.executable, "-c", _TMA_SCRIPT, str(ROOT)], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert float(r.stdout.strip().splitlines()[-1]) <= TF32_REL_L2


@pytest.mark.parametrize("dim", [4, 8, 12, 16, 20, 32])
def test_stream_sddmm_wide_windows(env, oracle, dim):
    """Products-like windows (~480 edges, up to ~900 with the hub rows): the
    wide SDDMM (u16 slot map rebuilt per 16-block round) with each epilogue,
    against the oracle; the launch is sddmm_wide, not the window engine. D <= 16
    runs the 16-wide staged layout (masked below 16), 16 < D < 32 the 32-wide one
    masked."""
    tcg, kernels, _, torch = env
    from paper_2112_02052_b200 import _lib

    rng = np.random.default_rng(100 + dim)
    n = 2000
    src = np.concatenate([rng.integers(0, n, n * 30), np.repeat(np.arange(16), 25)])
    dst = np.concatenate([rng.integers(0, n, n * 30), rng.integers(0, n, 16 * 25)])
    g = tcg.CsrGraph.from_edges(src, dst, n)
    t = tcg.translate(g, tcg.BlockConfig())
    ptr, cols = g.node_pointer, g.edge_list
    wmax = int(np.diff(ptr[::16]).max())
    assert 255 < wmax <= 1024, wmax
    xa = rng.standard_normal((n, dim)).astype(np.float32)
    xb = rng.standard_normal((n, dim)).astype(np.float32)
    xat, xbt = torch.from_numpy(xa).cuda(), torch.from_numpy(xb).cuda()
    res = {}
    names = _kernel_names(torch, lambda: res.update(s=kernels.sddmm_device(t, xat, xbt)))
    assert any("sddmm_wide" in k for k in names), names
    s_ref = oracle.sddmm(ptr, cols, xa, xb)
    assert rel_l2(res["s"].cpu().numpy(), s_ref) <= TF32_REL_L2
    p = kernels.sddmm_device(t, xat, epilogue=_lib.EPI_SOFTMAX)
    p_ref = oracle.segment_softmax(oracle.sddmm(ptr, cols, xa), ptr)
    assert rel_l2(p.cpu().numpy(), p_ref) <= TF32_REL_L2
    ds = kernels.sddmm_device(t, xat, xbt, epilogue=_lib.EPI_SOFTMAX_BWD, aux=torch.from_numpy(p_ref).cuda())
    ds_ref = oracle.softmax_backward(p_ref, s_ref, ptr)
    assert rel_l2(ds.cpu().numpy(), ds_ref) <= TF32_REL_L2

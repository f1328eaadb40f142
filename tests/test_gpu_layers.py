"""GPU autograd layers: forward = reference layer semantics, backward = the
restated gradients (oracle.agnn_backward / spmm_transpose), CSR transpose =
the oracle's stable permutation, CUDA-graph replay = eager."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import TF32_REL_L2, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_2112_02052_b200 as tcg
    from paper_2112_02052_b200 import layers

    torch.backends.cuda.matmul.allow_tf32 = False
    return tcg, layers, torch


@pytest.mark.parametrize("n,deg,seed", [(300, 5, 7), (1000, 8, 3), (45, 3, 2), (2708, 4, 1)])
def test_csr_transpose_matches_oracle(env, oracle, n, deg, seed):
    tcg, _, _ = env
    g = tcg.synth.gen_uniform(n, deg, seed)
    t = tcg.translate(g, tcg.BlockConfig())
    tt = t.transpose()
    pt, ct, perm = oracle.csr_transpose(g.node_pointer, g.edge_list, n)
    assert np.array_equal(tt.tiled.graph.node_pointer, pt)
    assert np.array_equal(tt.tiled.graph.edge_list, ct)
    assert np.array_equal(tt.perm.cpu().numpy().view(np.uint32).astype(np.int64), perm)
    ref = oracle.translate(pt, ct, n, 16, 8)
    for k, v in zip(("win_partition", "edge_to_col", "col_offsets", "col_to_node"), ref):
        assert np.array_equal(getattr(tt.tiled, k), v), k


@pytest.mark.parametrize("mode,tol", [("f32", 2e-5), ("tf32", TF32_REL_L2)])
def test_agnn_backward_vs_oracle(env, oracle, mode, tol):
    tcg, layers, torch = env
    g = tcg.synth.gen_uniform(3000, 6, 11)
    t = tcg.translate(g, tcg.BlockConfig())
    rng = np.random.default_rng(0)
    z = rng.standard_normal((3000, 32)).astype(np.float32)
    gy = rng.standard_normal((3000, 32)).astype(np.float32)
    zt = torch.from_numpy(z).cuda().requires_grad_(True)
    y = layers.AgnnAggregate.apply(zt, t, mode)
    y.backward(torch.from_numpy(gy).cuda())
    ptr, cols = g.node_pointer, g.edge_list
    p = oracle.segment_softmax(oracle.sddmm(ptr, cols, z), ptr)
    y_ref = oracle.spmm(ptr, cols, z, f=p)
    dz_ref = oracle.agnn_backward(ptr, cols, z, p, gy)
    assert rel_l2(y.detach().cpu().numpy(), y_ref) <= tol
    assert rel_l2(zt.grad.cpu().numpy(), dz_ref) <= tol


@pytest.mark.parametrize("weighted", [False, True])
def test_gcn_backward_vs_oracle(env, oracle, weighted):
    tcg, layers, torch = env
    base = tcg.synth.gen_uniform(2000, 5, 4)
    vals = np.random.default_rng(5).random(base.num_edges).astype(np.float32) if weighted else None
    g = tcg.CsrGraph(2000, base.node_pointer, base.edge_list, vals)
    t = tcg.translate(g, tcg.BlockConfig())
    rng = np.random.default_rng(1)
    h = rng.standard_normal((2000, 16)).astype(np.float32)
    b = rng.standard_normal(16).astype(np.float32)
    gy = rng.standard_normal((2000, 16)).astype(np.float32)
    ht = torch.from_numpy(h).cuda().requires_grad_(True)
    bt = torch.from_numpy(b).cuda().requires_grad_(True)
    y = layers.GcnAggregate.apply(ht, bt, t, "f32", False)
    y.backward(torch.from_numpy(gy).cuda())
    ptr, cols = g.node_pointer, g.edge_list
    assert np.array_equal(y.detach().cpu().numpy(),
                          (oracle.spmm(ptr, cols, h, f=vals) + b).astype(np.float32))
    dh = oracle.spmm_transpose(ptr, cols, gy, f=vals)
    assert np.array_equal(ht.grad.cpu().numpy(), dh)  # exact mode: same fold order
    np.testing.assert_allclose(bt.grad.cpu().numpy(), gy.sum(0), rtol=1e-4, atol=1e-3)


@pytest.mark.parametrize("mode", ["tf32", "f32"])
@pytest.mark.parametrize("d", [16, 32])
def test_gcn_aggregate_fused_relu(env, mode, d):
    """relu=True (the ReLU in the SpMM epilogue, its backward fused with the bias
    gradient in tcg_colsum_gate; f32 mode takes the separate ReLU pass) is
    bitwise equal to F.relu of the plain layer, forward and backward."""
    tcg, layers, torch = env
    g = tcg.synth.gen_uniform(3000, 6, 9)
    t = tcg.translate(g, tcg.BlockConfig())
    gen = torch.Generator(device="cuda").manual_seed(d)
    h = torch.randn(3000, d, device="cuda", generator=gen)
    b = torch.randn(d, device="cuda", generator=gen)
    gy = torch.randn(3000, d, device="cuda", generator=gen)
    outs = []
    for fused in (True, False):
        ht, bt = h.clone().requires_grad_(True), b.clone().requires_grad_(True)
        y = (layers.GcnAggregate.apply(ht, bt, t, mode, True) if fused
             else torch.nn.functional.relu(layers.GcnAggregate.apply(ht, bt, t, mode, False)))
        y.backward(gy)
        outs.append((y.detach(), ht.grad, bt.grad))
    for a, b_ in zip(*outs):
        assert torch.equal(a, b_)
    assert (outs[0][0] == 0).any() and (outs[0][0] > 0).any()


@pytest.mark.parametrize("kind", ["uniform", "hub"])
def test_agnn_aggregate_next(env, kind):
    """AgnnAggregateNext (the next layer's Z = Y W in the AGNN forward kernel's
    epilogue) against AgnnAggregate followed by DenseFn: forward and gradients
    within fp32-class tolerance (both 3xTF32), and the fused kernel is what runs
    (on the hub graph the > 255-edge windows take the two-step form)."""
    tcg, layers, torch = env
    from torch.profiler import ProfilerActivity, profile

    if kind == "uniform":
        g = tcg.synth.gen_uniform(4000, 7, 11)
    else:
        rng = np.random.default_rng(3)
        n = 3000
        src = np.concatenate([rng.integers(0, n, n * 5), np.repeat(np.arange(3), 400)])
        dst = np.concatenate([rng.integers(0, n, n * 5), rng.integers(0, n, 1200)])
        g = tcg.CsrGraph.from_edges(src, dst, n)
    t = tcg.translate(g, tcg.BlockConfig())
    gen = torch.Generator(device="cuda").manual_seed(5)
    z = torch.randn(g.num_nodes, 32, device="cuda", generator=gen)
    w = torch.randn(32, 32, device="cuda", generator=gen) / 32 ** 0.5
    gz = torch.randn(g.num_nodes, 32, device="cuda", generator=gen)
    res = []
    for fused in (True, False):
        zt, wt = z.clone().requires_grad_(True), w.clone().requires_grad_(True)
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            if fused:
                zn = layers.AgnnAggregateNext.apply(zt, wt, t, "tf32")
            else:
                zn = layers.DenseFn.apply(layers.AgnnAggregate.apply(zt, t, "tf32"), wt, None, False)
            torch.cuda.synchronize()
        if fused and kind == "uniform":
            names = [e.name for e in prof.events()]
            # agnn_stream<KIND=0, PAIR, MASK=false, NEXT=true, ZR>
            assert any("agnn_stream<0, true, false, true" in nm or "agnn_stream<0, 1, 0, 1" in nm
                       for nm in names), names
        zn.backward(gz)
        res.append((zn.detach(), zt.grad, wt.grad))
    for a, b in zip(*res):
        assert rel_l2(a.cpu().numpy(), b.cpu().numpy()) < 2e-6


def test_agnn_model_next_layer_fusion(env, monkeypatch):
    """The AGNN model with the next layer's dense step fused into each AGNN
    forward (TCG_AGNN_NEXT=1) against the default: same loss and gradients
    within fp32-class tolerance."""
    tcg, layers, torch = env
    g = tcg.synth.gen_uniform(5000, 7, 13)
    t = tcg.translate(g, tcg.BlockConfig())
    x = torch.randn(5000, 64, device="cuda")
    lab = torch.randint(0, 7, (5000,), device="cuda")
    out = []
    for fused in (False, True):
        monkeypatch.setattr(layers, "_AGNN_NEXT", fused)
        torch.manual_seed(0)
        net = layers.AGNN(64, 32, 7, layers=3).cuda()
        loss = net.loss(x, t, lab)
        loss.backward()
        out.append([loss.detach()] + [p.grad.detach().clone() for p in net.parameters()])
    for a, b in zip(*out):
        assert rel_l2(a.reshape(-1).cpu().numpy(), b.reshape(-1).cpu().numpy()) < 1e-5


def test_models_train_and_graph_capture(env):
    tcg, layers, torch = env
    g = tcg.synth.gen_uniform(5000, 7, 2)
    t = tcg.translate(g, tcg.BlockConfig())
    t.transpose()
    x = torch.randn(5000, 64, device="cuda")
    labels = torch.randint(0, 10, (5000,), device="cuda")
    for Model in (lambda: layers.GCN(64, 16, 10), lambda: layers.AGNN(64, 32, 10, layers=2)):
        torch.manual_seed(0)
        m = Model().cuda()
        opt = torch.optim.Adam(m.parameters(), lr=0.01)
        losses = []
        for _ in range(20):
            opt.zero_grad(set_to_none=False)
            loss = layers.cross_entropy(m(x, t), labels)
            loss.backward()
            opt.step()
            losses.append(float(loss))
        assert losses[-1] < losses[0]
        # CUDA graph replay of one step equals eager
        m2 = Model().cuda()
        m2.load_state_dict(m.state_dict())

        def step(mod):
            mod.zero_grad(set_to_none=False)
            out = layers.cross_entropy(mod(x, t), labels)
            out.backward()
            return out

        eager = step(m2).detach().clone()
        grads = [p.grad.clone() for p in m2.parameters()]
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(2):
                step(m2)
        torch.cuda.current_stream().wait_stream(s)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            cap = step(m2)
        gr.replay()
        torch.cuda.synchronize()
        assert torch.equal(cap, eager)
        for p, q in zip(m2.parameters(), grads):
            assert torch.equal(p.grad, q)


def test_agnn_z_tf32_bitwise():
    """AGNNConv stores Z = X W on the tf32 grid (TCG_DENSE_OUT_TF32) and the
    fused forward / A-side backward / dual A^T SpMM skip its operand rounding
    (TCG_AGNN_Z_TF32, TCG_PREC_X2_TF32): the loss and every gradient are
    bitwise those of the unflagged path, which rounds Z inside the kernels."""
    import torch

    import paper_2112_02052_b200 as tcg
    from paper_2112_02052_b200 import layers

    g = tcg.synth.gen_uniform(4000, 7, seed=11)
    t = tcg.translate(g, tcg.BlockConfig(), device="cuda")
    t.transpose()
    gen = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(g.num_nodes, 48, device="cuda", generator=gen)
    lab = torch.randint(0, 9, (g.num_nodes,), device="cuda", generator=gen)
    res = {}
    saved = layers._Z_TF32
    try:
        for flag in (False, True):
            layers._Z_TF32 = flag
            net = layers.AGNN(48, 32, 9, layers=3).cuda()
            loss = net.loss(x, t, lab)
            loss.backward()
            res[flag] = (loss.detach().clone(), [p.grad.clone() for p in net.parameters()])
    finally:
        layers._Z_TF32 = saved
    assert torch.equal(res[False][0], res[True][0])
    for a, b in zip(res[False][1], res[True][1]):
        assert torch.equal(a, b)


def test_operand_tf32_flags():
    """TCG_DENSE_OUT_TF32 stores tcg_dense's output RN-rounded to tf32 (the
    32 x 32 kernel in its epilogue, other shapes by a rounding pass), and
    TCG_PREC_X2_TF32 on a dual SpMM of a pre-rounded x2 equals the unflagged
    call bitwise."""
    import torch

    import paper_2112_02052_b200 as tcg
    from paper_2112_02052_b200 import dense, kernels, tiles

    gen = torch.Generator(device="cuda").manual_seed(3)
    for n, ci, co in ((5000, 32, 32), (4500, 128, 16), (700, 20, 12)):
        x = torch.randn(n, ci, device="cuda", generator=gen)
        w = torch.randn(ci, co, device="cuda", generator=gen)
        y = dense.dense(dense.rows_ok(x), w)
        yr = dense.dense(dense.rows_ok(x), w, out_tf32=True)
        assert torch.equal(yr, tiles.quantize_tf32(y)), (n, ci, co)
    g = tcg.synth.gen_uniform(3000, 7, seed=4)
    t = tcg.translate(g, tcg.BlockConfig(), device="cuda")
    a = torch.randn(g.num_nodes, 32, device="cuda", generator=gen)
    b = dense.dense(dense.rows_ok(torch.randn(g.num_nodes, 32, device="cuda", generator=gen)),
                    torch.randn(32, 32, device="cuda", generator=gen), out_tf32=True)
    w1 = torch.rand(g.num_edges, device="cuda", generator=gen)
    w2 = torch.rand(g.num_edges, device="cuda", generator=gen)
    y0 = kernels.spmm_device(t, a, w1, x2=b, weights2=w2)
    y1 = kernels.spmm_device(t, a, w1, x2=b, weights2=w2, x2_tf32=True)
    assert torch.equal(y0, y1)

"""Dense companions (csrc/dense.cu) against float64 torch, and the whole AGNN /
GCN training step against the CPU oracle's restated epoch (same weights)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import TF32_REL_L2, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_2112_02052_b200 as tcg
    from paper_2112_02052_b200 import dense, layers

    return tcg, dense, layers, torch


@pytest.mark.parametrize("n,ci,co", [(1000, 128, 32), (777, 32, 40), (50, 1433, 16), (3, 7, 3),
                                     (4096, 32, 128), (20000, 32, 32), (5001, 40, 32),
                                     (3333, 64, 7), (999, 16, 8), (30000, 128, 40), (129, 32, 12),
                                     (20011, 100, 16), (7000, 96, 32), (5000, 96, 22),
                                     (3001, 100, 47), (169343, 128, 32), (4096, 100, 32)])
def test_dense_forward_backward_kernels(env, n, ci, co):
    _, dense, _, torch = env
    g = torch.Generator(device="cuda").manual_seed(n)
    x = torch.randn(n, ci, device="cuda", generator=g)
    w = torch.randn(ci, co, device="cuda", generator=g)
    b = torch.randn(co, device="cuda", generator=g)
    ref = (x.double() @ w.double() + b.double()).relu()
    y = dense.dense(x, w, bias=b, relu=True)
    # the wide input layers (33..128 -> 16 / 32, n >= 4096) run 3xTF32 on the tensor
    # cores (csrc/dense_mma.cu dense_in_mma): fp32-class, ~1e-6 against float64
    # instead of the FFMA kernel's ~2.5e-7
    tol = 2e-6 if (n >= 4096 and co in (16, 32) and 33 <= ci <= 128) else 1e-6
    assert rel_l2(y.cpu().numpy(), ref.cpu().numpy()) < tol
    gy = torch.randn(n, co, device="cuda", generator=g)
    m = (ref > 0).double()
    dx = dense.dense(gy, w, mask=y, transposed=True)  # mask: y [n x co] on the input gy
    assert rel_l2(dx.cpu().numpy(), ((gy.double() * m) @ w.double().T).cpu().numpy()) < 1e-6
    dw, db = dense.gemm_tn(x, gy, mask=y, colsum=True)
    assert rel_l2(dw.cpu().numpy(), (x.double().T @ (gy.double() * m)).cpu().numpy()) < 1e-6
    assert rel_l2(db.cpu().numpy(), (gy.double() * m).sum(0).cpu().numpy()) < 1e-6
    # deterministic
    dw2, _ = dense.gemm_tn(x, gy, mask=y, colsum=True)
    assert torch.equal(dw, dw2)


@pytest.mark.parametrize("n,ci,co", [(2708, 1433, 16), (19717, 500, 16), (5000, 300, 32), (3000, 132, 16),
                                     (300, 260, 32)])
def test_dense_wide_inputs(env, n, ci, co):
    """Inputs wider than 128 features (Cora 1433, Pubmed 500): the forward in
    128-feature K panels and the weight gradient over feature panels, both on
    the tensor cores (3xTF32), through DenseFn (which pads Cora's odd width to
    16-B rows) against float64."""
    _, dense, _, torch = env
    gen = torch.Generator(device="cuda").manual_seed(ci)
    x = torch.randn(n, ci, device="cuda", generator=gen)
    w = (torch.randn(ci, co, device="cuda", generator=gen) / ci ** 0.5).requires_grad_(True)
    b = torch.randn(co, device="cuda", generator=gen).requires_grad_(True)
    gy = torch.randn(n, co, device="cuda", generator=gen)
    y = dense.DenseFn.apply(x, w, b, True)
    y.backward(gy)
    xd, wd, bd = x.double(), w.detach().double().requires_grad_(True), b.detach().double().requires_grad_(True)
    ref = (xd @ wd + bd).relu()
    ref.backward(gy.double())
    assert rel_l2(y.detach().cpu().numpy(), ref.detach().cpu().numpy()) < 2e-6
    assert rel_l2(w.grad.cpu().numpy(), wd.grad.cpu().numpy()) < 2e-6
    assert rel_l2(b.grad.cpu().numpy(), bd.grad.cpu().numpy()) < 1e-6
    y2 = dense.DenseFn.apply(x, w, b, True)
    assert torch.equal(y, y2)


@pytest.mark.parametrize("ci,co", [(47, 16), (22, 32), (45, 40), (13, 8)])
def test_dense_padded_stride_inputs(env, ci, co):
    """Odd widths in padded-stride buffers (rows_empty) run the next tile width
    up; the padding columns hold NaN here and must not leak into the result."""
    _, dense, _, torch = env
    n = 3001
    gen = torch.Generator(device="cuda").manual_seed(ci)
    ld = (ci + 3) // 4 * 4
    buf = torch.full((n, ld), float("nan"), device="cuda")
    x = buf[:, :ci]
    x.copy_(torch.randn(n, ci, device="cuda", generator=gen))
    w = torch.randn(ci, co, device="cuda", generator=gen)
    y = dense.dense(x, w)
    assert rel_l2(y.cpu().numpy(), (x.double() @ w.double()).cpu().numpy()) < 1e-6
    wt = torch.randn(co, ci, device="cuda", generator=gen)  # dense(x, wt, transposed) = x wt^T
    yt = dense.dense(x, wt, transposed=True)
    assert rel_l2(yt.cpu().numpy(), (x.double() @ wt.double().T).cpu().numpy()) < 1e-6


@pytest.mark.parametrize("n,ci,co", [(169343, 32, 32), (1000, 32, 32), (77, 32, 32), (0, 32, 32),
                                     (5000, 32, 40), (3000, 16, 8)])
def test_dense_backward(env, n, ci, co):
    _, dense, _, torch = env
    gen = torch.Generator(device="cuda").manual_seed(n + ci)
    x = torch.randn(n, ci, device="cuda", generator=gen)
    g = torch.randn(n, co, device="cuda", generator=gen)
    w = torch.randn(ci, co, device="cuda", generator=gen)
    dx, dw = dense.dense_backward(x, g, w)
    if n:
        assert rel_l2(dx.cpu().numpy(), (g.double() @ w.double().T).cpu().numpy()) < 1e-6
        assert rel_l2(dw.cpu().numpy(), (x.double().T @ g.double()).cpu().numpy()) < 1e-6
        # the dx fold order is dense_tile's: bitwise equal to the unfused product
        assert torch.equal(dx, dense.dense(g, w, transposed=True))
    else:
        assert torch.equal(dw, torch.zeros_like(dw))
    dx2, dw2 = dense.dense_backward(x, g, w)
    assert torch.equal(dx, dx2) and torch.equal(dw, dw2)


@pytest.mark.parametrize("n,c,ld", [(169343, 16, 16), (5000, 47, 48), (1000, 300, 300),
                                    (7, 3, 3), (0, 5, 5), (100000, 40, 40)])
def test_colsum(env, n, c, ld):
    _, dense, _, torch = env
    buf = torch.randn(max(n, 1), ld, device="cuda")[:n]
    x = buf[:, :c]
    got = dense.colsum(x)
    ref = x.double().sum(0)
    assert got.shape == (c,)
    if n:
        assert rel_l2(got.cpu().numpy(), ref.cpu().numpy()) < 1e-6
    else:
        assert torch.equal(got, torch.zeros(c, device="cuda"))
    assert torch.equal(got, dense.colsum(x))  # deterministic


def test_softmax_xent(env):
    _, dense, _, torch = env
    logits = torch.randn(5000, 40, device="cuda") * 3
    labels = torch.randint(0, 40, (5000,), device="cuda")
    loss, dl = dense.softmax_xent(logits, labels)
    lg = logits.double().requires_grad_(True)
    ref = torch.nn.functional.cross_entropy(lg, labels)
    ref.backward()
    assert abs(float(loss) - float(ref)) < 1e-5 * max(1.0, abs(float(ref)))
    assert rel_l2(dl.cpu().numpy(), lg.grad.cpu().numpy()) < 1e-5
    # loss-only forward, backward recomputed from the logits with a device grad scale
    loss2, none = dense.softmax_xent(logits, labels, grad=False)
    assert none is None and torch.equal(loss, loss2)
    g = torch.tensor(2.5, device="cuda")
    dl2 = dense.softmax_xent_backward(logits, labels, g)
    assert torch.equal(dl2, dense.softmax_xent_backward(logits, labels, g))
    assert rel_l2(dl2.cpu().numpy(), 2.5 * lg.grad.cpu().numpy()) < 1e-5
    # autograd: a scaled loss scales the logits gradient
    lt = logits.clone().requires_grad_(True)
    (3.0 * dense.cross_entropy(lt, labels)).backward()
    assert rel_l2(lt.grad.cpu().numpy(), 3.0 * lg.grad.cpu().numpy()) < 1e-5


@pytest.mark.parametrize("n,kin,c", [(169343, 32, 40), (1000, 16, 47), (37, 32, 1), (50, 20, 9),
                                     (5003, 32, 48), (100, 12, 7), (16, 4, 2), (1, 32, 40),
                                     (700, 64, 40), (300, 32, 64), (200, 30, 10)])
def test_linear_xent(env, n, kin, c):
    """Output layer fused with the loss (and the two-kernel form for the shapes
    the fused kernel declines: kin 64, c 64, kin not a multiple of 4) against
    float64 torch: loss, dx, dW, db; bitwise deterministic."""
    _, dense, _, torch = env
    gen = torch.Generator(device="cuda").manual_seed(n + kin + c)
    x = torch.randn(n, kin, device="cuda", generator=gen)
    w = torch.randn(kin, c, device="cuda", generator=gen) / kin ** 0.5 * 3
    b = torch.randn(c, device="cuda", generator=gen)
    labels = torch.randint(0, c, (n,), device="cuda", generator=gen)
    fused = dense.linear_xent(x, w, b, labels)
    assert (fused is None) == (kin > 32 or kin % 4 != 0 or c > 48)
    xd, wd, bd = (v.double().requires_grad_(True) for v in (x, w, b))
    ref = torch.nn.functional.cross_entropy(xd @ wd + bd, labels)
    ref.backward()
    tol = 2e-6
    for div in (None, 3 * n):
        xs, ws, bs = (v.clone().requires_grad_(True) for v in (x, w, b))
        loss = dense.linear_cross_entropy(xs, ws, bs, labels, div)
        (2.0 * loss).backward()
        sc = 1.0 if div is None else n / div
        assert abs(float(loss) - sc * float(ref)) <= tol * max(1.0, abs(float(ref)))
        for got, want in ((xs.grad, xd.grad), (ws.grad, wd.grad), (bs.grad, bd.grad)):
            assert rel_l2(got.cpu().numpy(), 2.0 * sc * want.cpu().numpy()) < tol
    if fused is not None:
        loss, dl = fused
        again = dense.linear_xent(x, w, b, labels)
        assert torch.equal(loss, again[0]) and torch.equal(dl, again[1])
        lg = (xd @ wd + bd).detach().requires_grad_(True)
        torch.nn.functional.cross_entropy(lg, labels).backward()
        assert rel_l2(dl.cpu().numpy(), lg.grad.cpu().numpy()) < tol
        # a label outside [0, c) poisons the loss and its row
        bad = labels.clone()
        bad[n // 2] = c
        lb, db_ = dense.linear_xent(x, w, b, bad)
        assert torch.isnan(lb) and torch.isnan(db_[n // 2]).all()
        assert not torch.isnan(db_[:n // 2]).any()
        # the backward alone: no bias, no dx, a device grad scale; deterministic
        gsc = torch.tensor(0.5, device="cuda")
        dx0, dw0, db0 = dense.linear_xent_backward(x, w, None, labels, None, gsc, need_dx=False)
        assert dx0 is None and db0 is None
        wd2 = w.double().requires_grad_(True)
        torch.nn.functional.cross_entropy(x.double() @ wd2, labels).backward()
        assert rel_l2(dw0.cpu().numpy(), 0.5 * wd2.grad.cpu().numpy()) < tol
        assert torch.equal(dw0, dense.linear_xent_backward(x, w, None, labels, None, gsc, False)[1])


def _copy_weights_agnn(net, cpu):
    cpu.w_in[...] = net.lin_in.weight.detach().cpu().numpy()
    cpu.b_in[...] = net.lin_in.bias.detach().cpu().numpy()
    for wc, conv in zip(cpu.ws, net.convs):
        wc[...] = conv.weight.detach().cpu().numpy()
    cpu.w_out[...] = net.lin_out.weight.detach().cpu().numpy()
    cpu.b_out[...] = net.lin_out.bias.detach().cpu().numpy()


@pytest.mark.parametrize("fused", [False, True])
def test_agnn_train_step_vs_oracle(env, oracle, fused):
    tcg, _, layers, torch = env
    n, f, h, c = 3000, 64, 32, 10
    g = tcg.synth.gen_uniform(n, 6, 5)
    t = tcg.translate(g, tcg.BlockConfig())
    x = tcg.synth.random_embeddings(n, f, 2)
    lab = np.random.default_rng(4).integers(0, c, n)
    net = layers.AGNN(f, h, c, layers=2).cuda()
    cpu = oracle.AgnnModelCPU(f, h, c, layers=2)
    _copy_weights_agnn(net, cpu)
    params0 = [p.copy() for p in cpu.params]
    xg, lg = torch.from_numpy(x).cuda(), torch.from_numpy(lab).cuda()
    loss = net.loss(xg, t, lg) if fused else layers.cross_entropy(net(xg, t), lg)
    loss.backward()
    cpu_loss = cpu.epoch(g.node_pointer, g.edge_list, x, lab, mode="tf32")
    assert abs(float(loss) - cpu_loss) <= TF32_REL_L2 * abs(cpu_loss)
    # the CPU epoch took one Adam step: recover its gradients from m = (1-b1) g
    grads_cpu = [m / (1 - cpu.opt.b1) for m in cpu.opt.m]
    grads_gpu = [net.lin_in.weight.grad, net.lin_in.bias.grad,
                 *[cv.weight.grad for cv in net.convs], net.lin_out.weight.grad,
                 net.lin_out.bias.grad]
    for gg, gc in zip(grads_gpu, grads_cpu):
        assert rel_l2(gg.cpu().numpy(), gc) <= TF32_REL_L2
    # the Adam step moved every parameter
    assert all(not np.array_equal(a, b) for a, b in zip(params0, cpu.params))


@pytest.mark.parametrize("fused", [False, True])
def test_gcn_train_step_vs_oracle(env, oracle, fused):
    tcg, _, layers, torch = env
    n, f, h, c = 2000, 100, 16, 7
    g = tcg.synth.gen_uniform(n, 5, 8)
    t = tcg.translate(g, tcg.BlockConfig())
    x = tcg.synth.random_embeddings(n, f, 2)
    lab = np.random.default_rng(4).integers(0, c, n)
    net = layers.GCN(f, h, c).cuda()
    cpu = oracle.GcnModelCPU(f, h, c)
    cpu.w1[...] = net.c1.weight.detach().cpu().numpy()
    cpu.w2[...] = net.c2.weight.detach().cpu().numpy()
    xg, lg = torch.from_numpy(x).cuda(), torch.from_numpy(lab).cuda()
    loss = net.loss(xg, t, lg) if fused else layers.cross_entropy(net(xg, t), lg)
    loss.backward()
    cpu_loss = cpu.epoch(g.node_pointer, g.edge_list, x, lab, mode="tf32")
    assert abs(float(loss) - cpu_loss) <= TF32_REL_L2 * abs(cpu_loss)
    grads_cpu = [m / (1 - cpu.opt.b1) for m in cpu.opt.m]
    grads_gpu = [net.c1.weight.grad, net.c1.bias.grad, net.c2.weight.grad, net.c2.bias.grad]
    for gg, gc in zip(grads_gpu, grads_cpu):
        assert rel_l2(gg.cpu().numpy(), gc) <= TF32_REL_L2


_TC_SCRIPT = r"""
import sys
sys.path.insert(0, sys.argv[1])
import torch
from paper_2112_02052_b200 import _lib, dense
n0 = _lib.launch_count()
worst = 0.0
for n, ci, co in ((169343, 128, 32), (4096, 100, 32), (7000, 96, 32)):
    g = torch.Generator(device="cuda").manual_seed(n)
    x = torch.randn(n, ci, device="cuda", generator=g)
    w = torch.randn(ci, co, device="cuda", generator=g)
    b = torch.randn(co, device="cuda", generator=g)
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        y = dense.dense(x, w, bias=b, relu=True)
        torch.cuda.synchronize()
    assert any("dense_tc" in e.name for e in prof.events()), [e.name for e in prof.events()]
    ref = (x.double() @ w.double() + b.double()).relu()
    worst = max(worst, float((y.double() - ref).norm() / ref.norm()))
print(worst)
"""


def test_tcgen05_dense_opt_in():
    """The tcgen05 3xTF32 input-layer GEMM (csrc/dense_tc.cu; TCG_DENSE_TC=1,
    measured slower than the mma.sync kernel on these memory-bound shapes and
    kept as the A/B of DESIGN.md) against float64."""
    import os
    import subprocess
    import sys

    from conftest import ROOT

    env = dict(os.environ, TCG_DENSE_TC="1")
    r = subprocess.run([sys.executable, "-c", _TC_SCRIPT, str(ROOT)], env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert float(r.stdout.strip().splitlines()[-1]) < 2e-6


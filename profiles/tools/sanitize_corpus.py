"""Small-case corpus for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family once or more on small graphs, incl. hub windows, empty
windows, ragged N, several widths. Exits non-zero on a parity failure.
usage: compute-sanitizer --tool memcheck python sanitize_corpus.py"""
import sys

sys.path.insert(0, "/root/repo")
import numpy as np
import torch

import paper_2112_02052_b200 as tcg
from oracle import tcg_oracle as o
from paper_2112_02052_b200 import layers
from paper_2112_02052_b200.kernels import agnn_backward_device, agnn_forward_device, sddmm_device, spmm_device
from paper_2112_02052_b200.sgt import ShardSgt

torch.backends.cuda.matmul.allow_tf32 = False


def hub(n, seed):
    rng = np.random.default_rng(seed)
    src = np.concatenate([rng.integers(0, n, n * 5), np.repeat(np.arange(3), 600)])
    dst = np.concatenate([rng.integers(0, n, n * 5), rng.integers(0, n, 1800)])
    keep = (src < 32) | (src >= 64)
    return tcg.CsrGraph.from_edges(src[keep], dst[keep], n)


graphs = [tcg.synth.gen_uniform(333, 4, 1), tcg.synth.gen_uniform(1001, 9, 2), hub(1200, 3),
          tcg.synth.gen_powerlaw(900, 6, 4),
          tcg.synth.gen_uniform(1500, 30, 5)]  # products-like windows (~480 edges): sddmm_wide, BIG SpMM
worst = 0.0
for g in graphs:
    n = g.num_nodes
    t = tcg.translate(g, tcg.BlockConfig())
    ref = o.translate(g.node_pointer, g.edge_list, n, 16, 8)
    assert np.array_equal(t.edge_to_col, ref[1]) and np.array_equal(t.col_to_node, ref[3])
    W = t.num_row_windows
    ShardSgt(g, tcg.BlockConfig(), (W // 3, W)).count().fill(0)
    for d in (8, 16, 32, 40, 64):
        x = torch.randn(n, d, device="cuda")
        w = torch.rand(g.num_edges, device="cuda")
        y = spmm_device(t, x, w)
        yr = o.spmm(g.node_pointer, g.edge_list, x.cpu().numpy(), f=w.cpu().numpy())
        worst = max(worst, float(np.linalg.norm(y.cpu().numpy() - yr) / np.linalg.norm(yr)))
        spmm_device(t, x, w, mode="f32")
        sddmm_device(t, x, mode="tf32")
    for d in (32, 16, 12):  # masked D < 32 on the fused AGNN kernels (round 2)
        z = torch.randn(n, d, device="cuda")
        y, p = agnn_forward_device(t, z)
        agnn_backward_device(t, z, torch.randn_like(z), p, y_fwd=y)
        from paper_2112_02052_b200 import _lib
        sddmm_device(t, z, epilogue=_lib.EPI_SOFTMAX)
        sddmm_device(t, z, torch.randn_like(z), epilogue=_lib.EPI_SOFTMAX_BWD, aux=p)
    z = torch.randn(n, 32, device="cuda")
    net = layers.AGNN(32, 32, 5, layers=2).cuda()
    lab = torch.randint(0, 5, (n,), device="cuda")
    layers.cross_entropy(net(z, t), lab).backward()
    net.loss(z, t, lab).backward()  # fused output layer + loss (linear_xent, _bwd)
    gnet = layers.GCN(32, 16, 5).cuda()
    layers.cross_entropy(gnet(z, t), lab).backward()
    gnet.loss(z, t, lab).backward()  # fused ReLU epilogue, tcg_colsum_gate, linear_xent
# the round-2 dense tensor-core kernels at shapes that take them (n >= 4096 / wide inputs)
from paper_2112_02052_b200 import dense  # noqa: E402
for n, ci, co in ((4100, 128, 32), (4100, 100, 16), (1500, 300, 16), (1300, 1433, 32)):
    x = dense.rows16(torch.randn(n, ci, device="cuda"))
    wt = torch.randn(ci, co, device="cuda", requires_grad=True)
    b = torch.randn(co, device="cuda", requires_grad=True)
    dense.DenseFn.apply(x, wt, b, True).sum().backward()
for n, kin, c in ((5000, 32, 47), (4097, 16, 40), (33, 12, 3)):
    x = torch.randn(n, kin, device="cuda", requires_grad=True)
    wt = torch.randn(kin, c, device="cuda", requires_grad=True)
    b = torch.randn(c, device="cuda", requires_grad=True)
    lab = torch.randint(0, c, (n,), device="cuda")
    dense.linear_cross_entropy(x, wt, b, lab).backward()
torch.cuda.synchronize()
print(f"corpus ok, worst tf32 rel-L2 {worst:.2e}")
assert worst <= 5e-3

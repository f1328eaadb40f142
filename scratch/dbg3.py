import sys; sys.path.insert(0,'.')
import torch, paper_2112_02052_b200 as tcg
from paper_2112_02052_b200 import layers, _lib
from paper_2112_02052_b200.kernels import agnn_forward_device, sddmm_device, spmm_device
g = tcg.synth.shaped_graph("arxiv")
t = tcg.translate(g, tcg.BlockConfig(16, 8, "tf32"))
lin = layers.Linear(128, 32, relu=True).cuda()
x = torch.randn(g.num_nodes, 128, device='cuda')
for it in range(6):
    h = lin(x).detach() if it % 2 else torch.randn(g.num_nodes, 32, device='cuda')
    z = layers.DenseFn.apply(h, torch.randn(32, 32, device='cuda'), None, False).detach()
    y, p = agnn_forward_device(t, z)
    torch.cuda.synchronize()
    p2 = sddmm_device(t, z, epilogue=_lib.EPI_SOFTMAX)
    y2 = spmm_device(t, z, p2)
    torch.cuda.synchronize()
    print(it, float((y - y2).abs().max()), float((p[:g.num_edges]-p2).abs().max()), flush=True)

import sys; sys.path.insert(0, '/root/repo')
import torch
import paper_2112_02052_b200 as tcg
from paper_2112_02052_b200.kernels import spmm_device
g = tcg.synth.shaped_graph("products"); t = tcg.translate(g, tcg.BlockConfig(), device="cuda")
z = torch.randn(g.num_nodes, 16, device='cuda'); w = torch.rand(g.num_edges, device='cuda')
out = torch.empty_like(z)
for _ in range(3): spmm_device(t, z, w, out=out)
torch.cuda.synchronize()

import sys; sys.path.insert(0,'.')
import torch, paper_2112_02052_b200 as tcg
from paper_2112_02052_b200 import layers
g = tcg.synth.shaped_graph("arxiv")
t = tcg.translate(g, tcg.BlockConfig()); torch.cuda.synchronize(); print("sgt ok", t.window_maxima())
tt = t.transpose(); torch.cuda.synchronize(); print("transpose ok", tt.tiled.window_maxima())
t.abi(); tt.tiled.abi(); torch.cuda.synchronize(); print("abi ok")
z = torch.randn(g.num_nodes, 32, device='cuda', requires_grad=True)
y = layers.AgnnAggregate.apply(z, t, "tf32", None); torch.cuda.synchronize(); print("fwd ok")
y.sum().backward(); torch.cuda.synchronize(); print("bwd ok")

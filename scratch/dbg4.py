import sys; sys.path.insert(0,'.')
import torch, numpy as np, paper_2112_02052_b200 as tcg
from paper_2112_02052_b200 import layers, _lib
dev = torch.device("cuda", 0)
g = tcg.synth.shaped_graph("arxiv")
x_np = tcg.synth.random_embeddings(g.num_nodes, 128, seed=2)
lab = np.random.default_rng(4).integers(0, 40, g.num_nodes)
cfg = tcg.BlockConfig(16, 8, "tf32")
flush = torch.empty(64 << 20, device=dev)
for i in range(4):
    flush.fill_(1.0); t = tcg.translate(g, cfg, device=dev); torch.cuda.synchronize()
print("maxima", t.window_maxima(), flush=True)
tt = t.transpose(); torch.cuda.synchronize(); print("T maxima", tt.tiled.window_maxima(), flush=True)
torch.manual_seed(0)
net = layers.AGNN(128, 32, 40, layers=4).to(dev)
x = torch.from_numpy(x_np).to(dev); y = torch.from_numpy(lab).to(dev)
h = net.lin_in(x); torch.cuda.synchronize(); print("lin ok", flush=True)
for k, c in enumerate(net.convs):
    h = c(h, t); torch.cuda.synchronize(); print("conv", k, "ok", float(h.abs().max()), flush=True)
loss = layers.cross_entropy(net.lin_out(h), y); loss.backward(); torch.cuda.synchronize(); print("bwd ok", float(loss))

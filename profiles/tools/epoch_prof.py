"""One AGNN-4 arxiv epoch between cudaProfilerStart/Stop for ncu launch lists:
ncu --profile-from-start off --metrics gpu__time_duration.sum --csv python scratch/epoch_prof.py [agnn|gcn]"""
import sys; sys.path.insert(0, '.')
import torch
import bench
import paper_2112_02052_b200 as tcg
from paper_2112_02052_b200 import layers
kind = sys.argv[1] if len(sys.argv) > 1 else "agnn"
shape = sys.argv[2] if len(sys.argv) > 2 else "arxiv"
feats, classes = {"arxiv": (128, 40), "products": (100, 47), "amazon0601": (96, 22), "cora": (1433, 7),
                  "pubmed": (500, 3)}[shape]
g, x_np, lab_np = bench.make_inputs(shape, feats, classes)
t = tcg.translate(g, tcg.BlockConfig(), device="cuda")
t.transpose()
x = torch.from_numpy(x_np).cuda(); y = torch.from_numpy(lab_np).cuda()
net = (layers.AGNN(feats, 32, classes, layers=4) if kind == "agnn" else layers.GCN(feats, 16, classes)).cuda()
opt = torch.optim.Adam(net.parameters(), lr=0.01, capturable=True, fused=True)
def step():
    opt.zero_grad(set_to_none=True)
    lo = net.loss(x, t, y); lo.backward(); opt.step()
for _ in range(3): step()
torch.cuda.synchronize()
torch.cuda.profiler.start(); step(); torch.cuda.synchronize(); torch.cuda.profiler.stop()

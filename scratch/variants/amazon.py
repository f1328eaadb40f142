import sys, os; sys.path.insert(0, '/root/repo'); os.chdir('/root/repo')
import torch, time
import bench
import paper_2112_02052_b200 as tcg
from paper_2112_02052_b200 import layers
g, x_np, lab_np = bench.make_inputs("amazon0601", 96, 22)
t = tcg.translate(g, tcg.BlockConfig(), device="cuda"); t.transpose()
x = torch.from_numpy(x_np).cuda(); y = torch.from_numpy(lab_np).cuda()
out = []
for kind in ("gcn", "agnn"):
    net = (layers.AGNN(96, 32, 22, layers=4) if kind == "agnn" else layers.GCN(96, 16, 22)).cuda()
    opt = torch.optim.Adam(net.parameters(), lr=0.01, capturable=True, fused=True)
    def step():
        opt.zero_grad(set_to_none=True)
        lo = layers.cross_entropy(net(x, t), y); lo.backward(); opt.step()
    for _ in range(3): step()
    torch.cuda.synchronize(); s = time.perf_counter()
    for _ in range(10): step()
    torch.cuda.synchronize(); out.append(f"{kind} {(time.perf_counter() - s) / 10 * 1e3:.3f} ms")
print(" | ".join(out))

import sys; sys.path.insert(0, '/root/repo')
import torch, statistics
import paper_2112_02052_b200 as tcg
from paper_2112_02052_b200.kernels import spmm_device
flush = torch.empty(64 << 20, device='cuda')
def tm(fn, reps=15):
    ts=[]
    for _ in range(reps):
        flush.fill_(1.0)
        s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e)*1e3)
    return statistics.median(ts)
res = []
for shape in ("arxiv", "products"):
    g = tcg.synth.shaped_graph(shape); t = tcg.translate(g, tcg.BlockConfig(), device="cuda")
    for d in (16, 24):
        z = torch.randn(g.num_nodes, d, device='cuda'); w = torch.rand(g.num_edges, device='cuda')
        out = torch.empty_like(z)
        f = lambda: spmm_device(t, z, w, out=out)
        res.append(f"{shape} D={d} {tm(f):.1f}us")
    del t, g
print(" | ".join(res))

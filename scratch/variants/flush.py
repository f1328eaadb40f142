import sys; sys.path.insert(0, '/root/repo')
import torch, statistics
import paper_2112_02052_b200 as tcg
from paper_2112_02052_b200 import _lib
from paper_2112_02052_b200.kernels import spmm_device, sddmm_device
g = tcg.synth.shaped_graph("arxiv"); t = tcg.translate(g, tcg.BlockConfig())
z = torch.randn(g.num_nodes, 32, device='cuda')
p = sddmm_device(t, z, epilogue=_lib.EPI_SOFTMAX); out = torch.empty_like(z)
flush = torch.empty(64 << 20, device='cuda'); flush2 = torch.ones(64 << 20, device='cuda')
sink = torch.empty(1, device='cuda')
def tm(fn, mode):
    ts=[]
    for _ in range(40):
        if mode == 'write': flush.fill_(1.0)
        elif mode == 'writeread': flush.fill_(1.0); torch.sum(flush2, dim=0, out=sink)
        elif mode == 'read': torch.sum(flush2, dim=0, out=sink)
        s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e)*1e3)
    return statistics.median(ts)
f = lambda: spmm_device(t, z, p, out=out)
for m in ('write', 'writeread', 'read', 'none', 'write'):
    print(m, f"{tm(f, m):.1f}")

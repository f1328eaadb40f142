import sys; sys.path.insert(0, '/root/repo')
import torch, statistics
import paper_2112_02052_b200 as tcg
from paper_2112_02052_b200 import _lib
from paper_2112_02052_b200.kernels import agnn_forward_device, agnn_backward_device, sddmm_device
g = tcg.synth.shaped_graph("arxiv"); t = tcg.translate(g, tcg.BlockConfig())
z = torch.randn(g.num_nodes, 32, device='cuda'); gy = torch.randn_like(z)
y, p = agnn_forward_device(t, z)
flush = torch.empty(64 << 20, device='cuda')
def tm(fn):
    ts=[]
    for _ in range(30):
        flush.fill_(1.0)
        s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e)*1e3)
    return statistics.median(ts)
out = torch.empty_like(z); ds = torch.empty_like(p)
f = lambda: agnn_forward_device(t, z, p=p, out=out)
b = lambda: agnn_backward_device(t, z, gy, p, ds=ds, out=out, y_fwd=y)
sd = lambda: sddmm_device(t, z, epilogue=_lib.EPI_SOFTMAX, out=ds)
print(f"fwd {tm(f):.1f} bwd {tm(b):.1f} sddmm {tm(sd):.1f}")

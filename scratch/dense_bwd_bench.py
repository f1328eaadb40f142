import sys; sys.path.insert(0, '/root/repo')
import torch, statistics
from paper_2112_02052_b200 import dense
n = 169343
x = torch.randn(n, 32, device='cuda'); g = torch.randn(n, 32, device='cuda'); w = torch.randn(32, 32, device='cuda')
flush = torch.empty(64 << 20, device='cuda')
def tm(fn):
    ts = []
    for _ in range(30):
        flush.fill_(1.0)
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
    return statistics.median(ts)
split = lambda: (dense.dense(g, w, transposed=True), dense.gemm_tn(x, g))
fused = lambda: dense.dense_backward(x, g, w)
for _ in range(2):
    print(f"split {tm(split):.1f} us  fused {tm(fused):.1f} us")

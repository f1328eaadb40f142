import sys; sys.path.insert(0,'scratch')
import torch, statistics
from tmutil import tm
for mb in (4, 21.7, 86, 340, 1360):
    n = int(mb * 1e6 / 4)
    x = torch.randn(n, device='cuda'); y = torch.empty_like(x)
    t = tm(lambda: y.copy_(x)); t2 = tm(lambda: torch.add(x, 1.0, out=y))
    print(f"{mb:7.1f} MB copy {t:8.1f} us {2*n*4/t/1e3:7.0f} GB/s | add {t2:8.1f} us {2*n*4/t2/1e3:7.0f} GB/s")
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record(); e.record(); e.synchronize(); print("empty event pair", s.elapsed_time(e)*1e3, "us")
k = torch.empty(1, device='cuda')
print("tiny kernel", tm(lambda: k.add_(1.0)), "us")

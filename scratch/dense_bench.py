import sys; sys.path.insert(0,'.'); sys.path.insert(0,'scratch')
import torch, statistics
from paper_2112_02052_b200 import dense
torch.backends.cuda.matmul.allow_tf32 = False
from tmutil import tm
n = 169343
for ci, co in ((32, 32), (128, 32), (32, 40)):
    x = torch.randn(n, ci, device='cuda'); w = torch.randn(ci, co, device='cuda'); g = torch.randn(n, co, device='cuda')
    print(f"ci={ci} co={co}: dense {tm(lambda: dense.dense(x, w)):.1f}us  torch mm {tm(lambda: x @ w):.1f}us | "
          f"dX {tm(lambda: dense.dense(g, w, transposed=True)):.1f}us torch {tm(lambda: g @ w.t()):.1f} | "
          f"dW {tm(lambda: dense.gemm_tn(x, g)):.1f}us torch {tm(lambda: x.t() @ g):.1f}")
l = torch.randn(n, 40, device='cuda'); lab = torch.randint(0, 40, (n,), device='cuda')
print(f"xent {tm(lambda: dense.softmax_xent(l, lab)):.1f}us")

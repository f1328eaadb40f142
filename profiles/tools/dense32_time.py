"""32 x 32 dense forward / fused backward at the arxiv row count: cold times and accuracy."""
import statistics
import sys

sys.path.insert(0, "/root/repo")
import torch

from paper_2112_02052_b200 import dense

buf = torch.empty(512 << 18, device="cuda")
rd = torch.ones(512 << 18, device="cuda")


def cold(fn, reps=20):
    ts = []
    for _ in range(reps):
        buf.fill_(1.0)
        rd.sum()
        torch.cuda._sleep(200000)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return statistics.median(ts)


n = 169343
x = torch.randn(n, 32, device="cuda")
g = torch.randn(n, 32, device="cuda")
w = torch.randn(32, 32, device="cuda")
y = torch.empty(n, 32, device="cuda")
print(f"dense 32x32 fwd: {cold(lambda: dense.dense(x, w, out=y)):.1f} us")
print(f"dense 32x32 bwd (dx + dW): {cold(lambda: dense.dense_backward(x, g, w)):.1f} us")
yy = dense.dense(x, w)
dx, dw = dense.dense_backward(x, g, w)
r = lambda a, b: float((a.double() - b).norm() / b.norm())
print("y err", r(yy, x.double() @ w.double()), "dx err", r(dx, g.double() @ w.double().T),
      "dw err", r(dw, x.double().T @ g.double()))

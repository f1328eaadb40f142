"""tcgen05 3xTF32 dense GEMM (csrc/dense_tc.cu) vs float64 and vs the FFMA kernel:
accuracy and cold time for the BASELINE input layers."""
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


for n, ci, co in ((169343, 128, 32), (169343, 128, 16), (403394, 96, 16), (2449029, 100, 16), (5000, 40, 32),
                  (100001, 33, 32)):
    x = torch.randn(n, ci, device="cuda")
    w = torch.randn(ci, co, device="cuda") / ci ** 0.5
    b = torch.randn(co, device="cuda")
    y = dense.dense(x, w, bias=b, relu=True)
    ref = torch.relu(x.double() @ w.double() + b.double())
    err = float((y.double() - ref).norm() / ref.norm())
    us = cold(lambda: dense.dense(x, w, bias=b, relu=True, out=y))
    gb = (n * ci * 4 + n * co * 4) / (us * 1e-6) / 1e9
    print(f"n={n} ci={ci} co={co}: rel-L2 vs f64 {err:.2e}, {us:.1f} us cold ({gb:.0f} GB/s)", flush=True)

"""The fused output layer + loss kernels (dense_mma.cu linear_xent / linear_xent_bwd)
at the arxiv shapes: GCN (kin 16) and AGNN (kin 32), 40 classes. Prints CUDA-event
times (L2 warm) and serves as the ncu target:
ncu --set full -k regex:linear_xent python profiles/tools/xent_prof.py"""
import sys
sys.path.insert(0, ".")
import torch
from paper_2112_02052_b200 import dense

shapes = [(169343, 40, 16), (169343, 40, 32), (2449029, 47, 16)]
for n, c, kin in shapes:
    gen = torch.Generator(device="cuda").manual_seed(kin)
    x = torch.randn(n, kin, device="cuda", generator=gen)
    w = torch.randn(kin, c, device="cuda", generator=gen) / kin ** 0.5
    b = torch.randn(c, device="cuda", generator=gen)
    y = torch.randint(0, c, (n,), device="cuda", generator=gen)
    g = torch.ones((), device="cuda")
    for name, fn in (("fwd", lambda: dense.linear_xent(x, w, b, y, grad=False)),
                     ("bwd", lambda: dense.linear_xent_backward(x, w, b, y, None, g))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        torch.cuda.synchronize()
        print(f"n {n} c {c} kin {kin} {name}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us/call (incl. final_loss / sum_slabs)")

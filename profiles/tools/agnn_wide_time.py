"""AGNN layer forward / backward on products-shaped windows (~400 edges, past the
fused stream kernels' slot map), D = 32: CUDA events, median of 10, warm.
TCG_AGNN_WIN_FUSED=1 keeps the window engine's fused kernels (the pre-sddmm_wide path)."""
import os
import statistics
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch

import paper_2112_02052_b200 as tcg
from paper_2112_02052_b200 import layers

name = sys.argv[1] if len(sys.argv) > 1 else "products"
D = int(sys.argv[2]) if len(sys.argv) > 2 else 32
g = tcg.synth.shaped_graph(name)
t = tcg.translate(g, tcg.BlockConfig(), device="cuda")
t.transpose()
torch.manual_seed(0)
z = torch.randn(g.num_nodes, D, device="cuda", requires_grad=True)
gy = torch.randn(g.num_nodes, D, device="cuda")


def timed(fn, reps=10):
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


out = {}
fwd = lambda: out.update(y=layers.AgnnAggregate.apply(z, t, "tf32"))
fwd()
bwd = lambda: out["y"].backward(gy, retain_graph=True)
tf = timed(fwd)
tb = timed(bwd)
mode = "window-fused" if os.environ.get("TCG_AGNN_WIN_FUSED") else "two-step stream"
print(f"{name} AGNN D={D} {mode}: forward {tf:.3f} ms, backward {tb:.3f} ms")

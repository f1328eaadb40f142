"""Cold-L2 protocol check for the roofline SpMM (arxiv, weighted, D=32).

dirty: the round-1 flush (256+ MB write; ~126 MB of dirty lines are left in
       L2 and the timed kernel pays their write-back);
clean: the same write followed by a 512 MB read (write-back happens inside the
       flush, before the timed region);
warm : back-to-back launches.
"""
import statistics
import sys

sys.path.insert(0, "/root/repo")
import torch

import paper_2112_02052_b200 as tcg
from paper_2112_02052_b200 import _lib
from paper_2112_02052_b200.kernels import sddmm_device, spmm_device

g = tcg.synth.shaped_graph("arxiv")
t = tcg.translate(g, tcg.BlockConfig(), device="cuda")
n = g.num_nodes
D = int(sys.argv[1]) if len(sys.argv) > 1 else 32
z = torch.randn(n, D, device="cuda")
p = sddmm_device(t, z, mode="tf32", epilogue=_lib.EPI_SOFTMAX)
out = torch.empty(n, D, device="cuda")
buf = torch.empty(512 << 18, device="cuda")
rd = torch.empty(512 << 18, device="cuda")


def run():
    spmm_device(t, z, p, mode="tf32", out=out)


def timeit(mode, reps=50):
    ts = []
    for _ in range(reps):
        if mode != "warm":
            buf.fill_(1.0)
        if mode == "clean":
            rd.sum()
        torch.cuda._sleep(200000)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        run()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return statistics.median(ts)


for _ in range(5):
    run()
for mode in ("warm", "dirty", "clean"):
    print(f"spmm D={D} {mode}: {timeit(mode):.2f} us")

"""A/B of the SpMM engines at arxiv D=32 (weighted), cold clean L2 + warm.

Run once with the default engine (writes the reference output), then with
TCG_SPMM_ENGINE=ws TCG_WS_CFG=k: checks the output bitwise against the
default engine's and prints the cold / warm times (CUDA events, median of 50).
    python profiles/tools/ws_ab.py [graph] [D]
"""
import os
import statistics
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch

import paper_2112_02052_b200 as tcg
from paper_2112_02052_b200 import _lib
from paper_2112_02052_b200.kernels import sddmm_device, spmm_device

name = sys.argv[1] if len(sys.argv) > 1 else "arxiv"
D = int(sys.argv[2]) if len(sys.argv) > 2 else 32
g = tcg.synth.shaped_graph(name)
t = tcg.translate(g, tcg.BlockConfig(), device="cuda")
n = g.num_nodes
torch.manual_seed(0)
z = torch.randn(n, D, device="cuda")
zs = torch.randn(n, 32, device="cuda")
p = sddmm_device(t, zs, mode="tf32", epilogue=_lib.EPI_SOFTMAX)
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
torch.cuda.synchronize()
eng = os.environ.get("TCG_SPMM_ENGINE", "default") + os.environ.get("TCG_WS_CFG", "")
for k in sorted(os.environ):
    if k.startswith("TCG_") and k not in ("TCG_SPMM_ENGINE", "TCG_WS_CFG"):
        eng += f"+{k[4:].lower()}={os.environ[k]}"
refp = f"gpurun_out/ws_ref_{name}_{D}.pt"
if eng == "default":
    torch.save(out.cpu(), refp)
    same = "ref"
else:
    ref = torch.load(refp)
    o = out.cpu()
    same = "bitwise" if torch.equal(o, ref) else f"DIFF max {float((o - ref).abs().max()):.3e}"
print(f"{name} D={D} {eng:10s} cold {timeit('clean'):.2f} us  warm {timeit('warm'):.2f} us  [{same}]", flush=True)

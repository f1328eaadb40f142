"""Is the products-scale D=16 SpMM bound by X spilling out of L2 (157 MB X,
126 MB L2)? Same tiling, same instruction stream, but the column stream's node
ids folded into the first N/4 rows (a 39 MB, L2-resident X range): if DRAM
were the bound this version would be much faster. Also times the exact-f32
CSR kernel beside the TF32 one at D = 16 for the shapes of BASELINE."""
import statistics
import sys

sys.path.insert(0, "/root/repo")
import torch

import paper_2112_02052_b200 as tcg
from paper_2112_02052_b200.kernels import spmm_device

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


for shape in sys.argv[1:] or ["amazon0601", "products"]:
    g = tcg.synth.shaped_graph(shape)
    t = tcg.translate(g, tcg.BlockConfig(), device="cuda")
    t.abi()
    n = g.num_nodes
    for d in (16,):
        z = torch.randn(n, d, device="cuda")
        w = torch.rand(g.num_edges, device="cuda")
        out = torch.empty(n, d, device="cuda")
        tc = cold(lambda: spmm_device(t, z, w, out=out))
        ex = cold(lambda: spmm_device(t, z, w, mode="f32", out=out))
        line = f"{shape} D={d}: tf32 TC {tc:.1f} us, exact f32 CSR {ex:.1f} us"
        if shape == "products":
            cs = t.dev["col_stream"]
            saved = cs.clone()
            cs.remainder_(n // 4)
            folded = cold(lambda: spmm_device(t, z, w, out=out))
            cs.copy_(saved)
            line += f", TC with X folded into N/4 rows (L2-resident) {folded:.1f} us"
        print(line, flush=True)

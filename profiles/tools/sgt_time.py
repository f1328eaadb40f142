"""GPU SGT time (translate, CUDA events, median of 10) on the BASELINE shapes.
usage: python sgt_time.py [shape ...]"""
import statistics
import sys

sys.path.insert(0, "/root/repo")
import torch

import paper_2112_02052_b200 as tcg

for shape in sys.argv[1:] or ["arxiv", "products"]:
    g = tcg.synth.shaped_graph(shape)
    g.device_arrays("cuda")
    cfg = tcg.BlockConfig()
    ts = []
    for i in range(11):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        t = tcg.translate(g, cfg, device="cuda")
        e.record()
        e.synchronize()
        if i:
            ts.append(s.elapsed_time(e))
    n, m, u, W = g.num_nodes, g.num_edges, t.num_unique, t.num_row_windows
    b = 8 * (n + 1) + 8 * m + 4 * u + 8 * (W + 1) + 4 * W
    ms = statistics.median(ts)
    print(f"{shape}: SGT {ms * 1e3:.1f} us  ({b / (ms * 1e-3) / 1e9:.0f} GB/s algorithmic, B_SGT {b / 1e6:.1f} MB)")

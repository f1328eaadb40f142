import sys; sys.path.insert(0,'.')
import numpy as np, torch
import paper_2112_02052_b200 as tcg
from oracle import tcg_oracle as o
g = tcg.synth.gen_uniform(300, 4, 11)
t = tcg.translate(g, tcg.BlockConfig())
for d in (16, 17, 18, 20, 24, 32, 40, 64, 7, 3):
    x = np.random.default_rng(0).standard_normal((300, d)).astype(np.float32)
    got = tcg.spmm(t, x, mode="tf32")
    ref = o.spmm(g.node_pointer, g.edge_list, x, mode="tf32")
    err = np.abs(got - ref) > 1e-3 * (1 + np.abs(ref))
    rows = np.nonzero(err.any(1))[0]; cols = np.nonzero(err.any(0))[0]
    print(d, "bad rows", len(rows), rows[:10], "bad cols", cols[:40])
    gs = tcg.sddmm(t, x, mode="tf32"); rs = o.sddmm(g.node_pointer, g.edge_list, x, mode="tf32")
    print("  sddmm rel", np.linalg.norm(gs-rs)/np.linalg.norm(rs))

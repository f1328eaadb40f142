import sys; sys.path.insert(0, '/root/repo')
import torch, time
import paper_2112_02052_b200 as tcg
res = []
for shape in ("arxiv", "products"):
    g = tcg.synth.shaped_graph(shape)
    g.device_arrays(None)
    for _ in range(2): tcg.translate(g, tcg.BlockConfig())
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        s = time.perf_counter(); t = tcg.translate(g, tcg.BlockConfig()); torch.cuda.synchronize(); ts.append(time.perf_counter() - s)
    res.append(f"{shape} {min(ts)*1e3:.3f} ms")
print(" | ".join(res))

import sys; sys.path.insert(0, '/root/repo')
import torch
import paper_2112_02052_b200 as tcg
g = tcg.synth.shaped_graph(sys.argv[1] if len(sys.argv) > 1 else "products")
g.device_arrays(None)
tcg.translate(g, tcg.BlockConfig()); torch.cuda.synchronize()
torch.cuda.profiler.start(); tcg.translate(g, tcg.BlockConfig()); torch.cuda.synchronize(); torch.cuda.profiler.stop()

"""ncu target: the wide SDDMM (+ softmax) at products D=16 (sddmm_wide<16-wide>),
one launch after a warm-up, between cudaProfilerStart/Stop."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2112_02052_b200 as tcg
from paper_2112_02052_b200 import _lib
from paper_2112_02052_b200.kernels import sddmm_device

g = tcg.synth.shaped_graph("products")
t = tcg.translate(g, tcg.BlockConfig(), device="cuda")
z = torch.randn(g.num_nodes, 16, device="cuda")
sddmm_device(t, z, epilogue=_lib.EPI_SOFTMAX)
torch.cuda.synchronize()
torch.cuda.profiler.start()
sddmm_device(t, z, epilogue=_lib.EPI_SOFTMAX)
torch.cuda.synchronize()
torch.cuda.profiler.stop()

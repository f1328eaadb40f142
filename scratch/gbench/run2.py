import sys, ctypes, torch
sys.path.insert(0, '/root/repo')
import paper_2112_02052_b200 as tcg
lib = ctypes.CDLL('/root/repo/scratch/gbench/libgather.so')
lib.run_gather.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
g = tcg.synth.shaped_graph("arxiv"); t = tcg.translate(g, tcg.BlockConfig())
x = torch.randn(g.num_nodes, 32, device='cuda'); idx = t.dev["col_to_node"]
out = torch.empty(148*64*256, device='cuda')
for bps in (1, 2, 4, 8):
  for thr in (128, 256):
    blocks = 148 * bps
    ts = []
    for rep in range(20):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); lib.run_gather(x.data_ptr(), idx.data_ptr(), idx.numel(), 32, out.data_ptr(), blocks, thr, torch.cuda.current_stream().cuda_stream); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    ms = sorted(ts)[10]
    print(f"warps/SM {bps*thr//32:3d}: {ms*1e3:6.1f} us  {idx.numel()*128/ms/1e6:6.0f} GB/s")

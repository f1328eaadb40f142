import sys, ctypes, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2112_02052_b200 as tcg
lib = ctypes.CDLL('/root/repo/scratch/gbench/libgather.so')
lib.run_gather.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
g = tcg.synth.shaped_graph("arxiv")
t = tcg.translate(g, tcg.BlockConfig())
n = g.num_nodes
x = torch.randn(n, 32, device='cuda')
flush = torch.empty(64 << 20, device='cuda')
c2n = t.dev["col_to_node"]
cols = t.dev["edge_list"]
idx_sets = {"c2n(window order)": c2n, "edge_list": cols,
            "sequential": torch.arange(c2n.numel(), device='cuda', dtype=torch.int32) % n,
            "random": torch.randint(0, n, (c2n.numel(),), device='cuda', dtype=torch.int32)}
out = torch.empty(148*64*256, device='cuda')
for name, idx in idx_sets.items():
    for blocks, threads in ((148*8, 256), (148*16, 256), (148*32, 256)):
        res = []
        for cold in (True, False):
            ts = []
            for rep in range(20):
                if cold: flush.fill_(1.0)
                s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
                s.record()
                lib.run_gather(x.data_ptr(), idx.data_ptr(), idx.numel(), 32, out.data_ptr(), blocks, threads, torch.cuda.current_stream().cuda_stream)
                e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
            ms = sorted(ts)[len(ts)//2]
            res.append(f"{'cold' if cold else 'warm'} {ms*1e3:7.1f}us {idx.numel()*128/ms/1e6:7.0f}GB/s")
        print(f"{name:20s} grid {blocks:5d}: " + " | ".join(res))

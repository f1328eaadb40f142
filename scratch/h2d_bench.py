import torch, time
n = 169343 * 128
h = torch.randn(n).pin_memory()
d = torch.empty(n, device='cuda')
streams = [torch.cuda.Stream() for _ in range(4)]
def copy(k):
    chunk = (n + k - 1) // k
    ev = []
    for i in range(k):
        s = streams[i]
        with torch.cuda.stream(s):
            d[i*chunk:(i+1)*chunk].copy_(h[i*chunk:(i+1)*chunk], non_blocking=True)
    for s in streams[:k]: torch.cuda.current_stream().wait_stream(s)
for k in (1, 2, 4, 1, 2, 4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10): copy(k)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 10
    print(f"{k} streams: {dt*1e3:.3f} ms  {n*4/dt/1e9:.1f} GB/s")

"""Pinned H2D copy throughput for the per-step feature copy of the e2e leg
(arxiv: 86.7 MB), one copy vs chunks spread over several streams."""
import sys
import time

import torch

nbytes = int(float(sys.argv[1])) if len(sys.argv) > 1 else 169343 * 128 * 4
h = torch.empty(nbytes // 4, dtype=torch.float32).pin_memory()
d = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
for nst in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(nst)]
    chunks = list(zip(h.chunk(nst), d.chunk(nst)))
    for rep in range(6):
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        for st, (hc, dc) in zip(streams, chunks):
            st.wait_event(s)
            with torch.cuda.stream(st):
                dc.copy_(hc, non_blocking=True)
        for st in streams:
            torch.cuda.current_stream().wait_stream(st)
        e.record()
        e.synchronize()
        if rep == 5:
            ms = s.elapsed_time(e)
            print(f"{nst} stream(s): {ms:.3f} ms, {nbytes / ms / 1e6:.1f} GB/s", flush=True)

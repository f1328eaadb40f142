import torch, statistics
def tm(fn, reps=30, flush=None):
    """device time of fn(): GPU kept busy (spin) while the host enqueues, so no host gap is timed"""
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        if flush is not None: flush()
        torch.cuda._sleep(300000)
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
    return statistics.median(ts)

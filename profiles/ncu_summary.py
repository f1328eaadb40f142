import csv, sys, collections, subprocess
rep = sys.argv[1]
raw = subprocess.run(["ncu","-i",rep,"--page","raw","--csv"],capture_output=True,text=True).stdout.splitlines()
r = list(csv.reader(raw)); hdr = r[0]
keys = ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','lts__t_bytes.sum','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','launch__grid_size','launch__registers_per_thread','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','lts__throughput.avg.pct_of_peak_sustained_elapsed','sm__throughput.avg.pct_of_peak_sustained_elapsed','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']
stalls = [h for h in hdr if h.startswith('smsp__pcsamp_warps_issue_stalled') and not h.endswith('not_issued')]
for row in r[2:]:
    print(row[hdr.index('Kernel Name')][:70])
    for k in keys:
        if k in hdr: print(f"   {k:70s} {row[hdr.index(k)]}")
    st = sorted(((float(row[hdr.index(s)] or 0), s) for s in stalls), reverse=True)[:6]
    print("   stalls:", ", ".join(f"{s.split('stalled_')[1]}={v:.0f}" for v,s in st))

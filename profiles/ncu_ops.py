import csv, sys, collections, subprocess
rep, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu","-i",rep,"--page","source","--csv"],capture_output=True,text=True).stdout.splitlines()
rows=list(csv.reader(out)); cur=None; hdr=None; data={}
for r in rows:
    if not r: continue
    if r[0]=="Kernel Name": cur=r[1]; continue
    if r[0]=="Address": hdr=r; continue
    if hdr and cur: data.setdefault(cur,[]).append(r)
for k,v in data.items():
    if pat not in k: continue
    ie=hdr.index("Instructions Executed"); ss=hdr.index("Warp Stall Sampling (All Samples)")
    tot=sum(float(x[ie] or 0) for x in v)
    print(k, "total", tot)
    ops=collections.Counter(); st=collections.Counter()
    for x in v:
        toks=x[1].split()
        if not toks: continue
        op=toks[1] if toks[0].startswith('@') else toks[0]
        op=op.split('.')[0]
        ops[op]+=float(x[ie] or 0); st[op]+=float(x[ss] or 0)
    for op,c in ops.most_common(22): print(f"  {op:10s} {c/1e6:7.2f}M  stall_samples {st[op]:.0f}")
    if len(sys.argv) > 3:
        top=sorted(v,key=lambda x:-float(x[ss] or 0))[:40]
        for x in top: print("   ", x[0][-5:], x[ie], x[ss], x[1][:80])
    break

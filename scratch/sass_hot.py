import csv, subprocess, sys
rep, pat, scale = sys.argv[1], sys.argv[2], float(sys.argv[3])
out = subprocess.run(["ncu","-i",rep,"--page","source","--csv"],capture_output=True,text=True).stdout.splitlines()
rows=list(csv.reader(out)); cur=None; hdr=None; data={}
for r in rows:
    if not r: continue
    if r[0]=="Kernel Name": cur=r[1]; continue
    if r[0]=="Address": hdr=r; continue
    if hdr and cur: data.setdefault(cur,[]).append(r)
k=[k for k in data if pat in k][0]; v=data[k]
ie=hdr.index("Instructions Executed"); ss=hdr.index("Warp Stall Sampling (All Samples)")
tot=0
for i,x in enumerate(v):
    c=float(x[ie] or 0)/scale; tot+=c
    print(f"{i:5d} {c:7.2f} {x[ss]:>5s} {x[1][:110]}")
print("total per window", tot)

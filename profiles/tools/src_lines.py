"""Per CUDA source line instruction counts (and stall samples) of the first
kernel in an ncu report whose name contains a substring.
usage: python src_lines.py report.ncu-rep kernel-substring [top]"""
import csv
import subprocess
import sys

rep, ksub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows, fpath, fn, seen, hdr = [], None, None, None, None
for line in out:
    r = next(csv.reader([line]))
    if r[0] == "File Path":
        fpath = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        if seen is None and ksub in fn:
            seen = fn
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if fn != seen or not hdr or not r[0]:
        continue
    try:
        ie = float(r[hdr.index("Instructions Executed")])
        st = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except (ValueError, IndexError):
        continue
    rows.append((ie, st, f"{fpath}:{r[0]}", r[1][:80]))
tot = sum(x[0] for x in rows) or 1
stt = sum(x[1] for x in rows) or 1
print(seen)
for ie, st, where, src in sorted(rows, reverse=True)[:top]:
    print(f"{ie / tot * 100:5.1f}% inst {st / stt * 100:5.1f}% stall  {where:22s} {src}")

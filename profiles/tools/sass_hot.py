"""Hot SASS of one kernel in an ncu report: instruction mix weighted by
executions, and the lines with the most stall samples.
usage: python sass_hot.py report.ncu-rep [kernel-substring] [top]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
ksub = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout.splitlines()
blocks, cur = [], None
for line in out:
    if line.startswith('"Kernel Name"'):
        cur = [line.split(",")[1], []]
        blocks.append(cur)
    elif cur is not None:
        cur[1].append(line)
for name, lines in blocks:
    if ksub not in name:
        continue
    rows = list(csv.reader(lines))
    h = rows[0]
    ix = {k: h.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                  "Instructions Executed")}
    data = []
    for r in rows[1:]:
        try:
            data.append((r[ix["Source"]].strip(), int(r[ix["Instructions Executed"]] or 0),
                         int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)))
        except (ValueError, IndexError):
            pass
    tot = sum(d[1] for d in data)
    samp = sum(d[2] for d in data)
    print(f"== {name}  warp-instructions {tot}  stall samples {samp}")
    mix = collections.Counter()
    for s, n, _ in data:
        op = s.split()[0] if s else "?"
        if op.startswith("@"):
            op = s.split()[1]
        mix[op.split(".")[0]] += n
    print("   mix:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in mix.most_common(18)))
    print("   top stall lines:")
    for s, n, st in sorted(data, key=lambda d: -d[2])[:top]:
        print(f"   {st:6d} {n:9d}  {s[:90]}")

"""Split a kernel's executed warp-instructions (ncu source page, SASS) into
per-block / per-window / setup classes by execution count, and list the
per-block loop body. usage: python sass_split.py rep kernel-substring nblocks nwindows"""
import csv
import subprocess
import sys

rep, ksub, nblk, nwin = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout.splitlines()
blocks, cur = [], None
for line in out:
    if line.startswith('"Kernel Name"'):
        cur = [line, []]
        blocks.append(cur)
    elif cur is not None:
        cur[1].append(line)
for name, lines in blocks:
    if ksub not in name:
        continue
    rows = list(csv.reader(lines))
    h = rows[0]
    iS, iN, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    cls = {"block": [0, 0], "window": [0, 0], "setup": [0, 0]}
    body = []
    for r in rows[1:]:
        try:
            c, w = int(r[iN] or 0), int(r[iW] or 0)
        except (ValueError, IndexError):
            continue
        k = "block" if c >= 0.9 * nblk else "window" if c >= 0.7 * nwin else "setup"
        cls[k][0] += c
        cls[k][1] += w
        if k == "block":
            body.append((c, w, r[iS].strip()))
    print(name[:90])
    for k, (c, w) in cls.items():
        print(f"  {k:7s} {c:10d} warp-instr ({c / max(1, nblk if k == 'block' else nwin if k == 'window' else 1):.0f} per unit), {w} stall samples")
    if "--body" in sys.argv:
        for c, w, src in body:
            print(f"   {c:8d} {w:5d}  {src[:80]}")

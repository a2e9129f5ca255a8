"""Instruction-count / stall hot spots of one kernel in an ncu report (the
`--page source` SASS view): runs of consecutive instructions with the same
execution count (= one basic block), largest first.
usage: python tools/ncu_hot.py REPORT.ncu-rep [min_instructions]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
lim = float(sys.argv[2]) if len(sys.argv) > 2 else 2e5
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
data = rows[2:]
iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
blocks = []
for r in data:
    e = float(r[iE] or 0)
    w = float(r[iW] or 0)
    if blocks and blocks[-1][1] == e:
        blocks[-1][2] += 1
        blocks[-1][3] += w
        blocks[-1][5] = r[iS].strip()[:48]
    else:
        blocks.append([r[0][-5:], e, 1, w, r[iS].strip()[:48], r[iS].strip()[:48]])
tot = sum(b[1] * b[2] for b in blocks)
stall = sum(b[3] for b in blocks)
print(f"warp instructions {tot:.3e}, stall samples {stall:.0f}")
for b in sorted(blocks, key=lambda b: -b[1] * b[2]):
    if b[1] * b[2] < lim:
        break
    print(f"{b[0]} exec {int(b[1]):>8} x {b[2]:>3} = {int(b[1] * b[2]):>9} ({100 * b[1] * b[2] / tot:4.1f}%)  stall {100 * b[3] / max(stall, 1):4.1f}%  {b[4]} .. {b[5]}")

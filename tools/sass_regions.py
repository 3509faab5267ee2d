"""Stall / instruction share per code region of one kernel from an ncu source page (SASS).

    ncu -i rep --page source --csv --print-source sass -k regex:NAME > x.csv
    python tools/sass_regions.py x.csv
Region boundaries: barriers, EXIT and every 150 instructions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [r for r in rows[2:] if len(r) > 5 and r[0].startswith('0x')]
# keep the first kernel's listing
seen, first = set(), []
for r in data:
    if r[0] in seen:
        break
    seen.add(r[0])
    first.append(r)
iE, iS, iSrc = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
f = lambda x: float(x) if x.replace('.', '', 1).isdigit() else 0.0
tot_e = sum(f(r[iE]) for r in first) or 1
tot_s = sum(f(r[iS]) for r in first) or 1
print(f"instructions {tot_e:.0f} warp-level, stall samples {tot_s:.0f}")
acc_e = acc_s = 0.0
start = 0
for i, r in enumerate(first):
    acc_e += f(r[iE]); acc_s += f(r[iS])
    src = r[iSrc]
    if 'BAR.SYNC' in src or 'EXIT' in src or i - start >= 150 or i == len(first) - 1:
        print(f"[{start:4d},{i:4d}] instr {acc_e / tot_e * 100:5.1f}%  stall {acc_s / tot_s * 100:5.1f}%   end: {src.strip()[:60]}")
        acc_e = acc_s = 0.0
        start = i + 1

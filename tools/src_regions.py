"""Per barrier-delimited region of one kernel from an ncu source page: executed instructions,
stall samples (with reasons) and shared-memory wavefronts (actual / ideal).

    ncu -i rep --page source --csv --print-source sass -k regex:NAME --launch-count 1 > x.csv
    python tools/src_regions.py x.csv [--top N]
"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 12
h = rows[1]
f = lambda x: float(x) if x.replace('.', '', 1).isdigit() else 0.0
iE, iS, iSrc = h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)'), h.index('Source')
iW, iI = h.index('L1 Wavefronts Shared'), h.index('L1 Wavefronts Shared Ideal')
stall_cols = [(i, c[6:]) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
data, seen = [], set()
for r in rows[2:]:
    if len(r) > 5 and r[0].startswith('0x'):
        if r[0] in seen:
            break
        seen.add(r[0])
        data.append(r)
tE = sum(f(r[iE]) for r in data) or 1
tS = sum(f(r[iS]) for r in data) or 1
tW = sum(f(r[iW]) for r in data) or 1
print(f"{tE:.0f} warp instructions, {tS:.0f} stall samples, {tW / 1e6:.2f}M shared wavefronts ({sum(f(r[iI]) for r in data) / 1e6:.2f}M ideal)")
start = 0
aE = aS = aW = aI = 0.0
st = Counter()
for i, r in enumerate(data):
    aE += f(r[iE]); aS += f(r[iS]); aW += f(r[iW]); aI += f(r[iI])
    for j, n in stall_cols:
        st[n] += f(r[j])
    if 'BAR.SYNC' in r[iSrc] or 'EXIT' in r[iSrc] or i == len(data) - 1:
        if aE > 0.002 * tE or aS > 0.005 * tS:
            reasons = ", ".join(f"{k} {v / tS * 100:.1f}" for k, v in st.most_common(5) if v > 0)
            print(f"[{start:4d},{i:4d}] instr {aE / tE * 100:5.1f}%  time {aS / tS * 100:5.1f}%  smem wavefronts {aW / 1e6:5.2f}M (ideal {aI / 1e6:5.2f}M)  ({reasons})")
        start, aE, aS, aW, aI, st = i + 1, 0.0, 0.0, 0.0, 0.0, Counter()
print(f"top {top} by stall samples")
for i, r in sorted(enumerate(data), key=lambda x: -f(x[1][iS]))[:top]:
    reasons = ", ".join(f"{n} {f(r[j]):.0f}" for j, n in sorted(stall_cols, key=lambda c: -f(r[c[0]]))[:3] if f(r[j]) > 0)
    print(f"{i:5d} {f(r[iS]) / tS * 100:5.1f}%  x{f(r[iE]):9.0f}  {r[iSrc].strip()[:56]:56s} {reasons}")
print(f"top {top} by shared wavefronts")
for i, r in sorted(enumerate(data), key=lambda x: -f(x[1][iW]))[:top]:
    print(f"{i:5d} x{f(r[iE]):9.0f}  w={f(r[iW]):9.0f} ideal={f(r[iI]):9.0f}  {r[iSrc].strip()[:56]}")

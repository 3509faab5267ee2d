"""Executed-instruction and stall breakdown of one kernel from an ncu source page (SASS).

    ncu -i rep --page source --csv --print-source sass -k regex:NAME --launch-count 1 > x.csv
    python tools/sass_breakdown.py x.csv [--top N]
Prints executed warp instructions per opcode class, per barrier-delimited region (with the
dominant stall reasons), and the top instructions by stall samples."""
import csv
import sys
from collections import Counter, defaultdict

path = sys.argv[1]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
rows = list(csv.reader(open(path)))
h = rows[1]
data, seen = [], set()
for r in rows[2:]:
    if len(r) > 5 and r[0].startswith("0x"):
        if r[0] in seen:
            break
        seen.add(r[0])
        data.append(r)
f = lambda x: float(x) if x.replace(".", "", 1).isdigit() else 0.0
iE, iS, iSrc = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
stall_cols = [(i, c[6:]) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot_e = sum(f(r[iE]) for r in data) or 1
tot_s = sum(f(r[iS]) for r in data) or 1
print(f"{tot_e:.0f} warp instructions, {tot_s:.0f} stall samples, {len(data)} SASS lines")
op = Counter()
for r in data:
    toks = r[iSrc].split()
    toks = [t for t in toks if not t.startswith("@")]
    op[toks[0].split(".")[0] if toks else "?"] += f(r[iE])
print("opcode share of executed:", ", ".join(f"{k} {v / tot_e * 100:.1f}%" for k, v in op.most_common(22)))
start, acc_e, acc_s, st = 0, 0.0, 0.0, Counter()
for i, r in enumerate(data):
    acc_e += f(r[iE]); acc_s += f(r[iS])
    for j, n in stall_cols:
        st[n] += f(r[j])
    src = r[iSrc]
    if "BAR.SYNC" in src or "EXIT" in src or i == len(data) - 1:
        if acc_e > 0.002 * tot_e or acc_s > 0.005 * tot_s:
            reasons = ", ".join(f"{k} {v / tot_s * 100:.1f}" for k, v in st.most_common(4) if v > 0)
            print(f"[{start:4d},{i:4d}] instr {acc_e / tot_e * 100:5.1f}%  stall {acc_s / tot_s * 100:5.1f}%  ({reasons})  end: {src.strip()[:50]}")
        start, acc_e, acc_s, st = i + 1, 0.0, 0.0, Counter()
print(f"top {top} instructions by stall samples:")
for i, r in sorted(enumerate(data), key=lambda x: -f(x[1][iS]))[:top]:
    reasons = ", ".join(f"{n} {f(r[j]):.0f}" for j, n in sorted(stall_cols, key=lambda c: -f(r[c[0]]))[:3] if f(r[j]) > 0)
    print(f"{i:5d} {f(r[iS]) / tot_s * 100:5.1f}%  x{f(r[iE]):9.0f}  {r[iSrc].strip()[:60]:60s} {reasons}")

"""Print per-kernel stall summary and barrier-delimited SASS segments of an ncu report."""
import collections, csv, subprocess, sys
rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else "k_assemble"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
hdr = r[0]
for row in r[2:]:
    d = dict(zip(hdr, row))
    items = [(k, v) for k, v in d.items() if 'smsp__pcsamp_warps_issue_stalled' in k and not k.endswith('not_issued')]
    tot = sum(float(v.replace(',', '')) for k, v in items if v) or 1
    print(d['Kernel Name'][:70], d['gpu__time_duration.sum'])
    print('  ', ', '.join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_','')}={float(v.replace(',',''))/tot*100:.1f}%" for k, v in sorted(items, key=lambda x: -float(x[1].replace(',', '') or 0))[:7]))
    print('  ', ' '.join(f"{k.split('.')[0].split('__')[-1]}={d.get(k)}" for k in ['smsp__inst_executed.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers', 'launch__registers_per_thread']))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name", f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]; idx = {h: i for i, h in enumerate(hdr)}
data = [x for x in rows[2:] if len(x) >= len(hdr)]
half = len(data) // 2
if half and data[0][idx['Address']] == data[half][idx['Address']]:
    data = data[:half]
def f(x):
    try: return float(x.replace(',', ''))
    except Exception: return 0.0
tot = sum(f(x[idx['Instructions Executed']]) for x in data) or 1
totst = sum(f(x[idx['Warp Stall Sampling (All Samples)']]) for x in data) or 1
seg_ex = seg_st = 0; start = 0; ops = collections.Counter()
for i, x in enumerate(data):
    ex = f(x[idx['Instructions Executed']]); seg_ex += ex; seg_st += f(x[idx['Warp Stall Sampling (All Samples)']])
    s = x[idx['Source']].strip(); toks = s.split()
    op = (toks[1] if toks and toks[0].startswith('@') else toks[0]).split('.')[0] if toks else ''
    ops[op] += ex
    if 'BAR.' in s or 'SYNCS' in s or 'DEPBAR' in s or i == len(data) - 1:
        if seg_ex / tot > 0.003 or seg_st / totst > 0.01:
            print(f"seg {start:5d}-{i:5d}: instr {seg_ex/tot*100:5.1f}%  stall {seg_st/totst*100:5.1f}%  end {s[:30]:30s}", ', '.join(f"{k}:{v/max(seg_ex,1)*100:.0f}%" for k, v in ops.most_common(5)))
        seg_ex = seg_st = 0; start = i + 1; ops = collections.Counter()

"""Key ncu counters + top stalls per kernel of a report: python tools/ncu_brief.py rep.ncu-rep"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active"]
for r in rows[2:]:
    d = dict(zip(h, r))
    print(d["Kernel Name"][:90])
    for k in keys:
        if k in d:
            print(f"   {k:60s} {d[k]} {u[h.index(k)]}")
    st = []
    for k, v in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st.append((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v.replace(",", ""))))
            except ValueError:
                pass
    tot = sum(v for _, v in st) or 1
    print("   stalls:", ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in sorted(st, key=lambda x: -x[1])[:8]))

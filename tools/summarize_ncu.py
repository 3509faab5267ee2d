"""Summarise ncu captures (gpurun_out/*.ncu-rep, launches.csv) into profiles/.

    python tools/summarize_ncu.py <tag> <prof.ncu-rep> [launches.csv]

Writes profiles/<tag>_ncu.md (per-kernel SOL / stall / dram table), profiles/<tag>_launches.csv
(copy of the launch list) and updates profiles/traffic.json with the dram bytes per launch
of the bench kernels (read by bench.py's roofline.traffic).
"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size"]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def main():
    tag, rep = sys.argv[1], sys.argv[2]
    launches = sys.argv[3] if len(sys.argv) > 3 else None
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    rows, units = raw_rows(rep)
    lines = [f"# ncu summary `{tag}` ({os.path.basename(rep)})", "",
             "`ncu --set full --clock-control none`, one launch per row (replayed; not a bench timing).", "",
             "| kernel | " + " | ".join(k.split('.')[0] for k in KEYS) + " | top stalls |",
             "|---|" + "---|" * (len(KEYS) + 1)]
    traffic = {}
    for d in rows:
        name = d.get("Kernel Name", "")[:80]
        stalls = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), num(v)) for k, v in d.items()
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and num(v)]
        tot = sum(v for _, v in stalls) or 1.0
        top = ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in sorted(stalls, key=lambda x: -x[1])[:4])
        vals = []
        for k in KEYS:
            v = d.get(k, "")
            u = units.get(k, "")
            vals.append(f"{v} {u}".strip())
        lines.append(f"| `{name}` | " + " | ".join(vals) + f" | {top} |")
        r, w = num(d.get("dram__bytes_read.sum")), num(d.get("dram__bytes_write.sum"))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        if r is not None and w is not None:
            tb = r * scale.get(units.get("dram__bytes_read.sum", "byte"), 1) + \
                 w * scale.get(units.get("dram__bytes_write.sum", "byte"), 1)
            traffic.setdefault(name, []).append(tb)
    if launches:
        shutil.copy(launches, os.path.join(ROOT, "profiles", f"{tag}_launches.csv"))
        rows2 = list(csv.reader(open(launches)))
        start = next(i for i, r in enumerate(rows2) if r and r[0] == "ID")
        hdr = rows2[start]
        idx = {h: i for i, h in enumerate(hdr)}
        agg = collections.defaultdict(list)
        for r in rows2[start + 1:]:
            if len(r) == len(hdr):
                agg[r[idx["Kernel Name"]][:80]].append(num(r[idx["Metric Value"]]))
        lines += ["", "## Launch list (gpu__time_duration, cold-cache, serialised)", "",
                  "| kernel | launches | median us | share of listed time |", "|---|---|---|---|"]
        total = sum(sum(v) for v in agg.values())
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            v = sorted(v)
            lines.append(f"| `{k}` | {len(v)} | {v[len(v) // 2] / 1000:.1f} | {sum(v) / total * 100:.1f}% |")
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    tj = json.load(open(tp)) if os.path.exists(tp) else {}
    er = [v for k, v in traffic.items() if "k_assemble<3, 1, float, 1, 4" in k]
    fin = [v for k, v in traffic.items() if "k_node_finish<3, float, 4" in k]
    if er:
        a = sum(er[0]) / len(er[0])
        b = (sum(fin[0]) / len(fin[0])) if fin else 0.0
        tj["config3_energy_residual"] = {"dram_bytes_per_launch": a + b, "kernel_a": a, "kernel_b": b,
                                         "source": f"profiles/{tag}_ncu.md (ncu --set full)"}
    with open(tp, "w") as f:
        json.dump(tj, f, indent=1)
    print("\n".join(lines[:12]))


if __name__ == "__main__":
    main()

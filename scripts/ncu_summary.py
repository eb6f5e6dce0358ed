"""Summarise ncu reports / launch lists into profiles/ (run in the build container).

    python scripts/ncu_summary.py gpurun_out/x.ncu-rep [more.ncu-rep ...] > profiles/rNN_x.md
    python scripts/ncu_summary.py --launches gpurun_out/launches.csv
"""
import csv
import io
import subprocess
import sys
from collections import OrderedDict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "CTA limit (regs)"),
    ("launch__occupancy_limit_shared_mem", "CTA limit (smem)"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("launch__grid_size", "grid"),
    ("smsp__inst_executed.sum", "instructions"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = OrderedDict()
        for i, h in enumerate(hdr):
            d[h] = (r[i], units[i] if i < len(units) else "")
        res.append(d)
    return res


def summarize(rep):
    lines = [f"### {rep}", ""]
    for d in raw(rep):
        name = d.get("Kernel Name", ("?", ""))[0]
        lines.append(f"**{name[:110]}**")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for key, label in METRICS:
            if key in d:
                v, u = d[key]
                lines.append(f"| {label} | {v} {u} |")
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v[0].replace(",", "") or 0)
                  for k, v in d.items()
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
        tot = sum(stalls.values()) or 1.0
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:5]
        lines.append("| top stalls | " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top) + " |")
        lines.append("")
    return "\n".join(lines)


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            k = d["Kernel Name"][:80]
            agg.setdefault(k, []).append(float(d["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in agg.values()) or 1.0
    out = ["| kernel | launches | mean (us) | share |", "|---|---|---|---|"]
    for k, v in agg.items():
        out.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {100 * sum(v) / tot:.1f}% |")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(launches(sys.argv[2]))
    else:
        for rep in sys.argv[1:]:
            print(summarize(rep))

"""Summarize ncu reports / launch lists into markdown for profiles/.

usage: python tools/ncu_summary.py <report.ncu-rep>... [--launches launches.csv]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "time", 1.0),
    ("dram__bytes_read.sum", "DRAM rd", 1.0),
    ("dram__bytes_write.sum", "DRAM wr", 1.0),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %", 1.0),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %", 1.0),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", 1.0),
    ("launch__registers_per_thread", "regs", 1.0),
    ("launch__occupancy_limit_registers", "CTA/SM (regs)", 1.0),
    ("lts__t_sector_hit_rate.pct", "L2 hit %", 1.0),
    ("launch__grid_size", "grid", 1.0),
]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return f"(no data in {path})\n"
    hdr, units = rows[0], rows[1]
    out = [f"### {path}\n", "| kernel | " + " | ".join(m[1] for m in METRICS) + " |",
           "|---" * (len(METRICS) + 1) + "|"]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")][:48]
        vals = []
        for key, _lbl, _s in METRICS:
            if key in hdr:
                i = hdr.index(key)
                vals.append(f"{r[i]} {units[i]}".strip())
            else:
                vals.append("-")
        out.append(f"| `{name}` | " + " | ".join(vals) + " |")
    return "\n".join(out) + "\n"


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[start + 1:]:
        if len(r) <= iv:
            continue
        v = float(r[iv].replace(",", ""))
        if r[iu] == "usecond":
            v *= 1e3
        elif r[iu] == "msecond":
            v *= 1e6
        name = r[ik].split("(")[0]
        tot[name] += v
        cnt[name] += 1
    allt = sum(tot.values())
    out = [f"### launch list {path} (cold-cache, serialised: compare shares)\n",
           "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        out.append(f"| `{k[:60]}` | {cnt[k]} | {v / 1e6:.3f} | {v / allt:.1%} |")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    args = sys.argv[1:]
    text = []
    while args:
        a = args.pop(0)
        if a == "--launches":
            text.append(launches(args.pop(0)))
        else:
            text.append(report(a))
    print("\n".join(text))

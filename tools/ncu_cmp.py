"""Side-by-side key metrics of the first kernel in several .ncu-rep files."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "launch__registers_per_thread", "smsp__inst_executed.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__cycles_active.avg", "sm__cycles_elapsed.avg"]


def load(path, name=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        if name is None or name in d.get("Kernel Name", ""):
            return d
    return {}


ds = [load(p) for p in sys.argv[1:]]
print("metric", *[p.split("/")[-1] for p in sys.argv[1:]], sep=" | ")
for k in KEYS:
    print(k, *[d.get(k, "-") for d in ds], sep=" | ")
st = sorted({k for d in ds for k in d if k.startswith("smsp__average_warps_issue_stalled_")
             and k.endswith("_per_issue_active.ratio")},
            key=lambda k: -float(ds[0].get(k) or 0))
for k in st[:10]:
    print(k.replace("smsp__average_warps_issue_stalled_", "stall ").replace(
        "_per_issue_active.ratio", ""), *[d.get(k, "-") for d in ds], sep=" | ")

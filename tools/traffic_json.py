"""Per-launch DRAM traffic of each profiled kernel -> profiles/traffic.json.

usage: python tools/traffic_json.py profiles/traffic.json svm1m=<report.ncu-rep | raw.csv> ...
(a .csv is an `ncu -i <rep> --page raw --csv` export, as tools/r02_evidence.sh
writes on the GPU box)
bench.py reads the file to fill roofline.traffic (ncu --set full capture:
dram__bytes_read.sum + dram__bytes_write.sum of one launch)."""
import csv
import io
import json
import subprocess
import sys

# bench.py kernel label -> ncu kernel-name prefix
LABELS = {
    "chain_svm": ("void k_svm_chain_unit", "void k_svm_chain_w"),
    "edge_collision": "void k_collision_tiles_v3",
    "var_large_d1": "void k_var_row_pipe<1",
    "var_large_d2": "void k_var_row_pipe<2",
    "edge_mpc_dyn": "void k_mpc_dyn_gemm",
    "var_small_deg4": "void k_var_small_run<4,",
    "var_giant_chunks": "void k_var_giant_chunks",
    "chain_mpc": "void k_mpc_chain",
    "chain_mpc_block": "void k_mpc_block<",
}


def traffic(path):
    if path.endswith(".csv"):
        with open(path) as fh:
            raw = fh.read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].replace(" ", "")
        byt = 0.0
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(key)
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[i], 1)
            byt += float(r[i].replace(",", "")) * scale
        for label, prefs in LABELS.items():
            prefs = (prefs,) if isinstance(prefs, str) else prefs
            if any(name.startswith(p.replace(" ", "")) for p in prefs):
                out.setdefault(label, []).append(byt)
    return {k: sum(v) / len(v) for k, v in out.items()}


def main():
    dst = sys.argv[1]
    try:
        with open(dst) as fh:
            data = json.load(fh)
    except OSError:
        data = {}
    for arg in sys.argv[2:]:
        w, path = arg.split("=", 1)
        data[w] = {"source": path, "bytes_per_launch": traffic(path)}
    with open(dst, "w") as fh:
        json.dump(data, fh, indent=1, sort_keys=True)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()

"""profiles/ncu_summary_*.json from an ncu --set full report of scripts/prof_spmv.py: per SpMV
level the duration, DRAM bytes (the bench's roofline "traffic"), throughput and occupancy.
usage: python scripts/ncu_json.py report.ncu-rep "source description" > profiles/ncu_summary_rNN.json"""
import csv, io, json, re, subprocess, sys

rep, source = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[0], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}


def num(d, k):
    return float(d[ix[k]].replace(",", ""))


out = {"source": source, "kernels": {}}
for d in data:
    name = d[ix["Kernel Name"]]
    m = re.search(r"k_spmv_(rw|sp|win)<(\d+), (\d+), (\d+)", name)
    if not m:
        continue
    L = int(m.group(2))
    dot = m.group(4) == "1"  # rw<L, RPL, DOT, ...>, win<L, SIDE, DOT, ...>, sp<L, DOT, ...>
    if m.group(1) == "sp":
        dot = m.group(3) == "1"
    key = ("k_spmv_fp64_csr" if L == 0 else f"k_spmv_L{L}") if not dot else (
        "k_spmv_dot_fp64_csr" if L == 0 else f"k_spmv_dot_L{L}")
    if key in out["kernels"]:
        continue
    rd, wr = num(d, "dram__bytes_read.sum"), num(d, "dram__bytes_write.sum")
    # ncu reports MB / KB per the unit row; normalise to bytes
    unit = rows[1]
    rd *= {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1}.get(unit[ix["dram__bytes_read.sum"]], 1)
    wr *= {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1}.get(unit[ix["dram__bytes_write.sum"]], 1)
    out["kernels"][key] = {
        "kernel": name.split("(")[0],
        "duration_us": num(d, "gpu__time_duration.sum") * {"msecond": 1e3, "ms": 1e3, "usecond": 1.0, "us": 1.0, "nsecond": 1e-3, "ns": 1e-3,
                                                          "second": 1e6}.get(unit[ix["gpu__time_duration.sum"]], 1.0),
        "dram_read_MB": rd / 1e6, "dram_write_MB": wr / 1e6,
        "dram_bytes_per_launch": int(rd + wr),
        "dram_throughput_pct": num(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "warps_active_pct": num(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "registers": num(d, "launch__registers_per_thread"),
    }
out["k_spmv_L1"] = out["kernels"].get("k_spmv_L1")
out["k_spmv_dot_L1"] = out["kernels"].get("k_spmv_dot_L1")
print(json.dumps(out, indent=1))

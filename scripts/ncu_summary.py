"""Summarise an ncu report (raw page) for the judged kernels: time, DRAM bytes, throughput
percentages, occupancy, top stall reasons.  usage: python scripts/ncu_summary.py report.ncu-rep"""
import csv, io, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for d in data:
    name = d[idx["Kernel Name"]]
    print("==", name[:100])
    for k in keys:
        if k in idx:
            print(f"   {k:62s} {d[idx[k]]:>14s} {units[idx[k]]}")
    st = []
    for h, i in idx.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                st.append((float(d[i].replace(",", "")), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    print("   stalls: " + ", ".join(f"{h} {100*v/tot:.0f}%" for v, h in sorted(st, reverse=True)[:7]))

"""Aggregate an ncu --csv launch list (gpu__time_duration / dram bytes) per kernel name.
usage: python scripts/launch_table.py launches.csv [last_n_launches]"""
import collections, csv, sys
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
ik, im, iv, iid = (hdr.index(h) for h in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
d = collections.OrderedDict()
for r in rows[1:]:
    d.setdefault(r[iid], {"k": r[ik].split("(")[0][:70]})[r[im]] = float(r[iv].replace(",", ""))
recs = list(d.values())
if len(sys.argv) > 2:
    recs = recs[-int(sys.argv[2]):]
agg = collections.OrderedDict()
for v in recs:
    a = agg.setdefault(v["k"], [0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += v.get("gpu__time_duration.sum", 0)
    a[2] += v.get("dram__bytes_read.sum", 0)
    a[3] += v.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values()) or 1
print(f"{'kernel':70s} {'n':>5s} {'avg_us':>8s} {'share':>6s} {'rd_MB':>8s} {'wr_MB':>8s}")
for k, a in agg.items():
    print(f"{k:70s} {a[0]:5d} {a[1]/a[0]/1e3:8.2f} {100*a[1]/tot:5.1f}% {a[2]/a[0]/1e6:8.1f} {a[3]/a[0]/1e6:8.1f}")

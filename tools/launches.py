"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) for the last build."""
import csv, sys
from collections import OrderedDict
path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = list(csv.reader(open(path)))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[i]
ki, mi, vi, idi = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
d = OrderedDict()
for r in rows[i + 1:]:
    d.setdefault(r[idi], {"name": r[ki]})[r[mi]] = r[vi].replace(",", "")
items = list(d.values())[-last:] if last else list(d.values())
tot = 0.0
print("| kernel | time (us) | DRAM read (MB) | DRAM write (MB) | GB/s |")
print("|---|---|---|---|---|")
for it in items:
    t = float(it.get("gpu__time_duration.sum", 0)) / 1e3
    rd = float(it.get("dram__bytes_read.sum", 0)) / 1e6
    wr = float(it.get("dram__bytes_write.sum", 0)) / 1e6
    tot += t
    name = it["name"].split("(")[0]
    print(f"| {name} | {t:.1f} | {rd:.1f} | {wr:.1f} | {(rd + wr) / t * 1e-3 if t else 0:.0f} |")
print(f"\nsum of kernel time: {tot:.1f} us")

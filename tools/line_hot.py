"""Per-source-line instruction counts and stall samples from an ncu cuda,sass source export."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
agg = defaultdict(lambda: [0.0, 0.0, ""])
cur_file = ""
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8 or r[2] != "-":
        continue
    try:
        smp = float(r[4] or 0); ie = float(r[7] or 0)
    except ValueError:
        continue
    k = (cur_file, int(r[0]))
    agg[k][0] += smp; agg[k][1] += ie; agg[k][2] = r[1]
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"samples {ts:.0f}  warp-instr {ti:.3e}")
key = 1 if len(sys.argv) > 3 and sys.argv[3] == "inst" else 0
for (f, ln), (s, i, src) in sorted(agg.items(), key=lambda kv: -kv[1][key])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{f}:{ln:4d} stall {100*s/ts:5.1f}% inst {100*i/ti:5.1f}%  {src.strip()[:80]}")

"""Top SASS instructions (by warp-stall samples and by executed count) of an ncu source page export."""
import csv, sys, re
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ai, si = hdr.index("Address"), hdr.index("Source")
ss = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
recs = []
for r in rows[2:]:
    if len(r) <= ie: continue
    try:
        recs.append((r[ai], r[si], float(r[ss] or 0), float(r[ie] or 0)))
    except ValueError:
        pass
tot_s = sum(x[2] for x in recs) or 1
tot_i = sum(x[3] for x in recs) or 1
print(f"total samples {tot_s:.0f}, warp instructions {tot_i:.3e}")
op = Counter(); ops = Counter()
for a, s, smp, n in recs:
    o = s.split()[0] if s else "?"
    if o.startswith("@"): o = s.split()[1]
    o = o.split(".")[0]
    op[o] += n; ops[o] += smp
print("by opcode (executed %, stall %):")
for o, n in op.most_common(25):
    print(f"  {o:10s} {100*n/tot_i:6.2f}%  {100*ops[o]/tot_s:6.2f}%")
print("hottest instructions by stall samples:")
for a, s, smp, n in sorted(recs, key=lambda t: -t[2])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"  {a} {100*smp/tot_s:5.2f}% n={n:.2e}  {s[:90]}")

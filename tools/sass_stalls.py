"""Top SASS instructions with their dominant stall reasons (ncu cuda,sass source export)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = [r for r in rows if r and r[0] == "Line No"][0]
sc = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
recs = []
for r in rows:
    if len(r) == len(h) and r[0] == "" and r[2] not in ("-", ""):
        try:
            tot = float(r[4])
        except ValueError:
            continue
        reasons = sorted(((float(r[i] or 0), h[i][6:]) for i in sc if r[i] not in ("", "-")), reverse=True)
        recs.append((tot, r[2][-5:], r[3][:70], reasons[:3]))
T = sum(x[0] for x in recs) or 1
for tot, a, src, rs in sorted(recs, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{100*tot/T:5.1f}% {a} {src:70s} " + " ".join(f"{n}={100*v/T:.1f}" for v, n in rs if v))

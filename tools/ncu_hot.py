"""Top stalled SASS lines (with dominant stall reasons) from
`ncu -i rep --page source --csv --print-source sass > file.csv`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, ist = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
reasons = [i for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
data = []
for r in rows[2:]:
    try:
        data.append((float(r[ist] or 0), r[ia], r[isrc], {hdr[i][6:]: float(r[i] or 0) for i in reasons}))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
agg = {}
for d in data:
    for k, v in d[3].items():
        agg[k] = agg.get(k, 0) + v
print("total by reason:", ", ".join(f"{k}={100*v/tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
for s, a, src, rs in sorted(data, key=lambda x: -x[0])[:n]:
    top = ",".join(f"{k}:{int(v)}" for k, v in sorted(rs.items(), key=lambda x: -x[1])[:2] if v)
    print(f"{100*s/tot:5.1f}% {a[-5:]} {src[:80]:80s} {top}")

"""Executed warp instructions per CUDA source line from `ncu -i rep --page source
--csv --print-source cuda,sass > f.csv`.  python tools/ncu_inst.py f.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr, fname, agg = None, "?", {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) < len(hdr) or not r[0]:
        continue
    try:
        k = (fname, r[0], r[1][:80])
        agg[k] = agg.get(k, 0) + int(r[ie] or 0)
    except ValueError:
        pass
tot = sum(agg.values()) or 1
print("total warp instructions", tot)
for (f, ln, src), v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * v / tot:5.1f}% {v:10d} {f}:{ln} {src.strip()}")

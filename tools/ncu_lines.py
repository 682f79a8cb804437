"""Stall samples aggregated per CUDA source line (and file) from
`ncu -i rep --page source --csv --print-source cuda,sass > f.csv`.
python tools/ncu_lines.py f.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg, fname = {}, "?"
cur_line, cur_src = None, ""
hdr = None
for r in rows:
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[0]:
        cur_line, cur_src = r[0], r[1]
    try:
        v = float(r[4] or 0)
    except ValueError:
        continue
    k = (fname, cur_line)
    a = agg.setdefault(k, [0.0, cur_src])
    a[0] += v
tot = sum(v[0] for v in agg.values()) or 1
for (f, ln), (v, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100 * v / tot:5.1f}% {f}:{ln:>5} {src.strip()[:100]}")

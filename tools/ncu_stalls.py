"""Stall reasons per CUDA source line from `ncu -i rep --page source --csv
--print-source cuda,sass > f.csv`: the top lines by samples with their
dominant stall columns.  python tools/ncu_stalls.py f.csv [top] [file-filter]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
filt = sys.argv[3] if len(sys.argv) > 3 else ""
hdr, fname, cur = None, "?", None
agg = {}
for r in rows:
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:
        cur = (fname, r[0], r[1])
        if filt and filt not in fname:
            cur = None
        continue  # source rows carry the line totals; the following sass rows repeat them
    if cur is None:
        continue
    a = agg.setdefault(cur, [0.0, {}])
    try:
        a[0] += float(r[4] or 0)
    except ValueError:
        pass
    for i in cols:
        try:
            v = float(r[i] or 0)
        except ValueError:
            continue
        a[1][hdr[i][6:]] = a[1].get(hdr[i][6:], 0.0) + v
tot = sum(v[0] for v in agg.values()) or 1
for (f, ln, src), (v, st) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    s = sorted(st.items(), key=lambda x: -x[1])[:3]
    ss = " ".join(f"{k}={100 * x / (v or 1):.0f}%" for k, x in s if x > 0)
    print(f"{100 * v / tot:5.1f}% {f}:{ln:>5} [{ss}] {src.strip()[:70]}")

"""Summarise tools/profile_r02.sh's ncu artifacts into one small JSON (run where
the .ncu-rep files are; copy the result to profiles/).
python tools/summarize_r02.py <dir> <out.json> [launches per step, default 8]"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

d, outp = sys.argv[1], sys.argv[2]
out = {"how": "ncu --set full --clock-control none (one launch per shape, replayed: cold cache, serialised); "
              "launch list: ncu --metrics gpu__time_duration.sum over bench.py --steps 2 --warmup 1"}

rows = list(csv.reader(open(os.path.join(d, "launches.csv"))))
hdr, ks = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r))
        if x.get("Metric Name") == "gpu__time_duration.sum":
            ks.append((x["Kernel Name"].split("(")[0].replace("void ", ""), x["Grid Size"], float(x["Metric Value"]) / 1e3))
ours = [k for k in ks if "dgqk::" in k[0]]
n_step = int(sys.argv[3]) if len(sys.argv) > 3 else 8
step = ours[-n_step:]  # the last timed step: 4 K1 + 4 K5 (q/k/v fused into one launch)
tot = sum(t for *_, t in step)
agg = collections.OrderedDict()
for n, g, t in step:
    a = agg.setdefault(n.replace("dgqk::", ""), [0, 0.0])
    a[0] += 1
    a[1] += t
out["launch_list_last_step"] = [{"kernel": n.replace("dgqk::", ""), "grid": g, "us": round(t, 2)} for n, g, t in step]
out["share_by_kernel"] = {k: {"launches": v[0], "us": round(v[1], 1), "share": round(v[1] / tot, 3)} for k, v in agg.items()}
out["library_kernels_in_step"] = [n for n, *_ in ks[-12:] if "dgqk::" not in n]

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum"]
for f in sorted(os.listdir(d)):
    if not f.endswith(".ncu-rep"):
        continue
    raw = subprocess.run(["ncu", "-i", os.path.join(d, f), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    if len(r) < 3:
        continue
    h, v = r[0], r[2]
    m = {k: v[h.index(k)] for k in KEYS if k in h}
    stalls = {}
    for i, k in enumerate(h):
        if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio"):
            try:
                if float(v[i]) > 0.25:
                    stalls[k.split("stalled_")[1].split("_per")[0]] = round(float(v[i]), 2)
            except ValueError:
                pass
    m["stalls_per_issue"] = stalls
    m["kernel"] = v[h.index("Kernel Name")] if "Kernel Name" in h else ""
    out[f[:-8]] = m
json.dump(out, open(outp, "w"), indent=1)
print(json.dumps(out["share_by_kernel"], indent=1))

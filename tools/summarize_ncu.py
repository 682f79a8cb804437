"""Summarise ncu artifacts into profiles/ (tracked).
python tools/summarize_ncu.py <tag> <launches.csv> <k5.ncu-rep> [bench.json]"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, launches, rep = sys.argv[1:4]
bench = sys.argv[4] if len(sys.argv) > 4 else None
out = {"tag": tag}

# launch list (cold-cache, serialised: shares, not absolutes)
rows = list(csv.reader(open(launches)))
hdr = None
ks = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            ks.append((d["Kernel Name"].split("(")[0], d["Grid Size"], float(d["Metric Value"]) / 1e3))
# the last bench step = the last 10 of our launches
ours = [k for k in ks if "dgqk::" in k[0]]
step = ours[-10:]
tot = sum(t for _, _, t in step)
agg = collections.OrderedDict()
for n, g, t in step:
    key = n.replace("void dgqk::", "")
    agg.setdefault(key, [0, 0.0])
    agg[key][0] += 1
    agg[key][1] += t
out["launch_list_last_step"] = [{"kernel": n.replace("void dgqk::", ""), "grid": g, "us": round(t, 2)} for n, g, t in step]
out["share_by_kernel"] = {k: {"launches": v[0], "us": round(v[1], 1), "share": round(v[1] / tot, 3)} for k, v in agg.items()}

# full ncu capture of the K5 fc1 launch
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h, units, v = rr[0], rr[1], rr[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg", "gpc__cycles_elapsed.avg.per_second"]
m = {}
for w in want:
    if w in h:
        i = h.index(w)
        m[w] = f"{v[i]} {units[i]}".strip()
out["k5_fc1_ncu_full"] = m
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
try:
    rd = float(v[h.index("dram__bytes_read.sum")]) * scale[units[h.index("dram__bytes_read.sum")]]
    wr = float(v[h.index("dram__bytes_write.sum")]) * scale[units[h.index("dram__bytes_write.sum")]]
    out["k5_fc1_dram_bytes_per_launch"] = rd + wr
    M, K, N, g = 2048, 7168, 28672, 128
    out["k5_fc1_algorithmic_bytes"] = M * K + 4 * M + K * N / 2 + (K / g) * N * 1.5 + 4 * N + 2 * M * N
except Exception as e:
    out["error"] = str(e)
if bench:
    out["bench"] = json.load(open(bench))
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
path = os.path.join(ROOT, "profiles", f"ncu_summary_{tag}.json")
json.dump(out, open(path, "w"), indent=1)
json.dump({"k5_fc1_dram_bytes_per_launch": out.get("k5_fc1_dram_bytes_per_launch"), "source": os.path.basename(path)},
          open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w"), indent=1)
print(json.dumps({k: out[k] for k in ("share_by_kernel", "k5_fc1_ncu_full")}, indent=1))
print("dram per launch", out.get("k5_fc1_dram_bytes_per_launch"), "algorithmic", out.get("k5_fc1_algorithmic_bytes"))

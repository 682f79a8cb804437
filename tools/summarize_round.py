"""Summarise a round's ncu artifacts into profiles/ (tracked).

python tools/summarize_round.py <tag> <launches.csv> label=<rep>:M,K,N [label=<rep>:M,K,N ...]

* launches.csv: `ncu --metrics gpu__time_duration.sum --csv` of a bench run
  (cold-cache, serialised: compare SHARES, not absolutes); the last step's
  ten DGQ launches are tabulated.
* each rep: one `ncu --set full` capture of a fused-linear launch of shape
  M x K x N (g = 128): the key counters plus algorithmic bytes / ops, so
  traffic (dram read + write) can be compared with the algorithmic bytes.
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "l1tex__m_xbar2l1tex_read_bytes.sum",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
        "sm__cycles_active.avg", "sm__cycles_elapsed.avg", "gpc__cycles_elapsed.avg.per_second"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, ks = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                ks.append((d["Kernel Name"].split("(")[0].replace("void ", "").replace("dgqk::", ""), d["Grid Size"],
                           float(d["Metric Value"]) / 1e3))
    ours = [k for k in ks if k[0].startswith(("k_dgq", "k_actquant", "k_group"))]
    step = ours[-10:]
    tot = sum(t for _, _, t in step) or 1.0
    agg = collections.OrderedDict()
    for n, _, t in step:
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += t
    return {"launch_list_last_step": [{"kernel": n, "grid": g, "us": round(t, 2)} for n, g, t in step],
            "share_by_kernel": {k: {"launches": v[0], "us": round(v[1], 1), "share": round(v[1] / tot, 3)}
                                for k, v in agg.items()}}


def full(rep, M, K, N, g=128):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    h, units, v = rr[0], rr[1], rr[2]
    m, num = {}, {}
    for w in WANT:
        if w in h:
            i = h.index(w)
            m[w] = f"{v[i]} {units[i]}".strip()
            try:
                num[w] = float(v[i]) * SCALE.get(units[i], 1.0)
            except ValueError:
                pass
    algo_bytes = M * K + 4 * M + K * N / 2 + (K / g) * N * 1.5 + 4 * N + 2 * M * N
    ops = 2.0 * M * N * K
    out = {"shape": {"M": M, "K": K, "N": N, "g": g}, "metrics": m, "algorithmic_bytes": algo_bytes,
           "algorithmic_ops": ops}
    if "dram__bytes_read.sum" in num and "dram__bytes_write.sum" in num:
        out["traffic_bytes"] = num["dram__bytes_read.sum"] + num["dram__bytes_write.sum"]
    if "gpu__time_duration.sum" in num:
        t = num["gpu__time_duration.sum"]
        out["ncu_achieved_GBps"] = algo_bytes / t / 1e9
        out["ncu_achieved_TOPS"] = ops / t / 1e12
    return out


def main():
    tag, lpath = sys.argv[1:3]
    out = {"tag": tag, "note": "ncu numbers are cold-cache and serialised (clock-control none): use them for shares, "
                               "traffic and pipe utilisation; bench.py's CUDA-event timings are the performance numbers"}
    out.update(launches(lpath))
    caps = {}
    for arg in sys.argv[3:]:
        label, rest = arg.split("=", 1)
        rep, shape = rest.rsplit(":", 1)
        M, K, N = (int(x) for x in shape.split(","))
        caps[label] = full(rep, M, K, N)
    out["captures"] = caps
    path = os.path.join(ROOT, "profiles", f"ncu_summary_{tag}.json")
    json.dump(out, open(path, "w"), indent=1)
    # bench.py reads the dominant prefill kernel's traffic from here
    pf = caps.get("prefill_fc1", {})
    json.dump({"k5_fc1_dram_bytes_per_launch": pf.get("traffic_bytes"), "source": os.path.basename(path)},
              open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w"), indent=1)
    for k, c in caps.items():
        print(k, c.get("traffic_bytes"), c.get("algorithmic_bytes"), c["metrics"].get("gpu__time_duration.sum"),
              c["metrics"].get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
              c["metrics"].get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"))
    print(json.dumps(out["share_by_kernel"], indent=1))


if __name__ == "__main__":
    main()

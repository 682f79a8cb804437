"""Decode layer (M = 1) with and without its four K1 launches (graph replay, L2
flushed): how much of the layer the activation quantisation costs.
python tools/dec_k1_share.py"""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_2310_04836_b200 import linear_multi
dev = torch.device("cuda", 0)
layer = bench.OptLayer(0, 1, dev, None, 64)
layer.x.copy_(torch.from_numpy(bench._synth_x(64, 7168)))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
M = 1
# quantize once so codes are valid
layer.step(M)
torch.cuda.synchronize()
def step_nok1():
    cq, rq = layer.codes["q"], layer.rs["q"]
    linear_multi([layer.lin[n].layer for n in ("q", "k", "v")], cq[:M], rq[:M], outs=[layer.y[n][:M] for n in ("q", "k", "v")])
    layer._k5("out", layer.codes["out"], layer.rs["out"], M)
    layer._k5("fc1", layer.codes["fc1"], layer.rs["fc1"], M)
    layer._k5("fc2", layer.codes["fc2"], layer.rs["fc2"], M)
def timeit(fn):
    g = bench._graph_of(fn)
    ts = []
    for _ in range(20):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return min(ts), sum(ts) / len(ts)
for _ in range(2):
    print("full step (4 K1 + 4 K5d):", timeit(lambda: layer.step(M)))
    print("K5d only (no K1):        ", timeit(step_nok1))

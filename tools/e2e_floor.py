"""e2e serving pipeline vs the PCIe floor: the bench's pipelined step time, the
H2D / D2H copies alone and together, and the step with a concurrent H2D.
python tools/e2e_floor.py"""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_2310_04836_b200 import synth
dev = torch.device("cuda", 0)
layer = bench.OptLayer(0, 1, dev, None, 2048)
x_host = torch.from_numpy(synth.gen_synthetic(2048, 7168, 101, 3, 50.0, 7)).pin_memory()
layer.x.copy_(x_host)
x_hosts = [x_host, x_host.clone().pin_memory()]
out_hosts = [torch.empty(2048, 7168, dtype=torch.float16).pin_memory() for _ in range(2)]
sync = torch.cuda.synchronize
for rep in range(3):
    t = bench.e2e_pipelined(layer, 2048, 20, 3, x_hosts, out_hosts, sync)
    print("pipelined ms/step", round(t / 20 * 1e3, 3), flush=True)
# copies alone
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
xd = torch.empty(2048, 7168, device=dev); od = torch.empty(2048, 7168, dtype=torch.float16, device=dev)
for mode in ("h2d", "d2h", "both"):
    sync()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(10):
        if mode in ("h2d", "both"):
            with torch.cuda.stream(s1): xd.copy_(x_hosts[i % 2], non_blocking=True)
        if mode in ("d2h", "both"):
            with torch.cuda.stream(s2): out_hosts[i % 2].copy_(od, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    b.record(); b.synchronize()
    print(mode, "ms per copy", round(a.elapsed_time(b) / 10, 3), flush=True)
# compute + h2d concurrently
sync()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for i in range(10):
    with torch.cuda.stream(s1): xd.copy_(x_hosts[i % 2], non_blocking=True)
    layer.step(2048)
torch.cuda.current_stream().wait_stream(s1)
b.record(); b.synchronize()
print("step + concurrent h2d ms", round(a.elapsed_time(b) / 10, 3))
sync()
a.record()
for i in range(10):
    layer.step(2048)
b.record(); b.synchronize()
print("step alone ms", round(a.elapsed_time(b) / 10, 3))

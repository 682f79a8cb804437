"""Per-role timeline of CTA 0 of one K5d launch (debug trace buffer):
rows 0-3 globaltimer stamps (producer stage issue, MMA done, unpack done,
epilogue done), rows 4-8/12 per-stage cycle counts (when the kernel is built
with them), row 13 [cycles, ns] of the whole CTA.
python tools/dec_trace.py M K N [g]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_04836_b200 as dgq  # noqa: E402

M, K, N = (int(v) for v in sys.argv[1:4])
g = int(sys.argv[4]) if len(sys.argv) > 4 else 128
L = dgq.random_layer(K, N, g, seed=1)
CL = dgq.CudaLayer(L, validate=False)
x = torch.randn(M, K, device="cuda") * 3
codes, rs = CL.quantize_act(x)
out = torch.empty(M, N, dtype=torch.float16, device="cuda")
buf = torch.zeros(16 * 1024, dtype=torch.int64, device="cuda")
lib = dgq.lib()
lib.dgq_debug_set_timestamps.argtypes = [C.c_void_p]
for _ in range(3):
    CL.linear(codes, rs, out=out)
torch.cuda.synchronize()
lib.dgq_debug_set_timestamps(C.c_void_p(buf.data_ptr()))
CL.linear(codes, rs, out=out)
torch.cuda.synchronize()
lib.dgq_debug_set_timestamps(None)
ts = buf.view(16, 1024).cpu().numpy().astype(np.int64)
cyc, ns = ts[13][0], ts[13][1]
print(f"CTA 0: {cyc} cycles in {ns} ns -> {cyc / max(ns, 1) * 1e3:.0f} MHz")
lab = {4: "mma waits", 5: "mma issue+commit", 6: "unp wait full", 7: "unp wait aempty", 8: "unp work+arrive",
       12: "epi tmem ld+wait"}
for r, name in lab.items():
    if ts[r].any():
        print(f"  {name:20s}", ts[r][2:18].tolist())
st, en = ts[14], ts[15]
ok = (st > 0) & (en > 0)
if ok.any():
    s0 = st[ok].min()
    print(f"CTAs: start {(st[ok].min() - s0) / 1e3:.2f}..{(st[ok].max() - s0) / 1e3:.2f} us, "
          f"end {(en[ok].min() - s0) / 1e3:.2f}..{(en[ok].max() - s0) / 1e3:.2f} us "
          f"(median end {(np.median(en[ok]) - s0) / 1e3:.2f})")
stamps = ts[0:4]
t0 = stamps[stamps > 0].min()
names = ["producer", "mma_done", "unp_done", "epi_done"]
for r in range(4):
    v = stamps[r][stamps[r] > 0]
    if not len(v):
        continue
    v = (v - t0) / 1e3
    d = np.diff(v)
    print(f"{names[r]:9s} n={len(v):4d} first {v[0]:7.2f} last {v[-1]:7.2f} us  step {np.median(d) if len(d) else 0:6.3f}"
          f"  t[6:12]={np.round(v[6:12], 2).tolist()}")

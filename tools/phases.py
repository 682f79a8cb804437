"""Per-CTA phase timeline of one fused-linear launch (globaltimer stamps).
python tools/phases.py M K N g"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_04836_b200 as dgq  # noqa: E402

M, K, N, g = (int(v) for v in sys.argv[1:5])
L = dgq.random_layer(K, N, g, seed=1)
CL = dgq.CudaLayer(L, validate=False)
x = torch.randn(M, K, device="cuda") * 3
codes, rs = CL.quantize_act(x)
out = torch.empty(M, N, dtype=torch.float16, device="cuda")
buf = torch.zeros(4096 * 8, dtype=torch.int64, device="cuda")
lib = dgq.lib()
lib.dgq_debug_set_timestamps.argtypes = [C.c_void_p]
for _ in range(3):
    CL.linear(codes, rs, out=out)
torch.cuda.synchronize()
lib.dgq_debug_set_timestamps(C.c_void_p(buf.data_ptr()))
CL.linear(codes, rs, out=out)
torch.cuda.synchronize()
lib.dgq_debug_set_timestamps(None)
ts = buf.view(-1, 8).cpu().numpy().astype(np.int64)
ts = ts[ts[:, 0] > 0]
t0 = ts[:, 0].min()
names = ["start", "setup", "1st_full", "deq_done", "acc_done", "splitk_red", "epi_end", "exit"]
print(f"{len(ts)} CTAs; times in us relative to first CTA start")
for i, nm in enumerate(names):
    col = ts[:, i]
    col = col[col > 0]
    if len(col):
        r = (col - t0) / 1e3
        print(f"{nm:11s} min {r.min():7.2f}  med {np.median(r):7.2f}  max {r.max():7.2f}")

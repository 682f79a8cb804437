"""Per-role timeline of CTA 0 of one K5d launch (globaltimer stamps):
role 0 producer stage issue, 1 MMA issued, 2 unpack done, 3 epilogue done.
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
t0 = ts[ts > 0].min()
names = ["producer", "mma_done", "unp_done", "epi_done", "unp_start", "unp_full", "unp_aempty", "unp_xempty",
         "mma_start", "mma_full", "mma_afull", "mma_dempty", "epi_start", "epi_dfull", "epi_xfull", "-"]
lab = {4: "mma wait afull", 5: "mma wait dempty", 6: "mma issue", 7: "mma commits", 8: "unp wait full",
       9: "unp wait aempty", 10: "unp work", 11: "unp st-wait+arrive", 12: "epi wait dfull", 13: "epi work"}
for r in range(4, 14):
    print(f"  {lab[r]:20s}", ts[r][2:18].tolist())
for r in range(4):
    v = ts[r][ts[r] > 0]
    if not len(v):
        continue
    v = (v - t0) / 1e3
    d = np.diff(v)
    print(f"{names[r]:11s} n={len(v):4d} first {v[0]:7.2f} last {v[-1]:7.2f} us  step {np.median(d) if len(d) else 0:6.3f}"
          f"  t[6:12]={np.round(v[6:12], 2).tolist()}")

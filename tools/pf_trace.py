"""K5p per-k-block timeline of the first CTA pair (globaltimer, us): when the
leader's MMA issuer observes each k-block ready, and the median period.  python tools/pf_trace.py M K N"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_04836_b200 as dgq  # noqa: E402

M, K, N = (int(v) for v in sys.argv[1:4])
L = dgq.random_layer(K, N, 128, seed=1)
CL = dgq.CudaLayer(L, validate=False)
x = torch.randn(M, K, device="cuda") * 3
codes, rs = CL.quantize_act(x)
out = torch.empty(M, N, dtype=torch.float16, device="cuda")
buf = torch.zeros(9 * 1024, dtype=torch.int64, device="cuda")
lib = dgq.lib()
lib.dgq_debug_set_timestamps.argtypes = [C.c_void_p]
lib.dgq_debug_set_decode.argtypes = [C.c_int]
lib.dgq_debug_set_decode(1 | 0x400)
for _ in range(2):
    CL.linear(codes, rs, out=out)
torch.cuda.synchronize()
lib.dgq_debug_set_timestamps(C.c_void_p(buf.data_ptr()))
CL.linear(codes, rs, out=out)
torch.cuda.synchronize()
lib.dgq_debug_set_timestamps(None)
b = buf.view(9, 1024).cpu().numpy()
t0 = b[b > 0].min()
r = lambda v: (v - t0) / 1e3  # noqa: E731
print(" kb | lead: start  slot-ok  arrive | peer: start  slot-ok  arrive | mma ready")
for i in list(range(0, 6)) + list(range(60, 69)):
    print(f"{i:3d} | {r(b[3][i]):6.2f} {r(b[5][i]):6.2f} {r(b[1][i]):6.2f} | {r(b[4][i]):6.2f} {r(b[6][i]):6.2f} "
          f"{r(b[2][i]):6.2f} | {r(b[0][i]):6.2f}")
n = int((b[0] > 0).sum())
d = np.diff(b[0][:n]) / 1e3
print(f"MMA period median {np.median(d):.3f} us over {n} k-blocks")
lib.dgq_debug_set_decode(1)

"""CTA start/end stamps of consecutive K5d launches inside one CUDA graph:
how long each kernel body runs and the gap between kernels.
python tools/dec_gap.py M K N [copies]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_04836_b200 as dgq  # noqa: E402

M, K, N = (int(v) for v in sys.argv[1:4])
copies = int(sys.argv[4]) if len(sys.argv) > 4 else 3
lib = dgq.lib()
lib.dgq_debug_set_decode.argtypes = [C.c_int]
if len(sys.argv) > 5:
    lib.dgq_debug_set_decode(int(sys.argv[5], 0))
lib.dgq_debug_set_timestamps.argtypes = [C.c_void_p]
base = dgq.random_layer(K, N, 128, seed=3)
layers = [dgq.CudaLayer(base, validate=False) for _ in range(copies)]
x = torch.randn(M, K, device="cuda") * 3
codes, rs = layers[0].quantize_act(x)
out = torch.empty(M, N, dtype=torch.float16, device="cuda")
n = 6
bufs = [torch.zeros(16 * 1024, dtype=torch.int64, device="cuda") for _ in range(n)]
for L in layers:
    L.linear(codes, rs, out=out)
torch.cuda.synchronize()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for i in range(n):
            lib.dgq_debug_set_timestamps(C.c_void_p(bufs[i].data_ptr()))
            layers[i % copies].linear(codes, rs, out=out)
lib.dgq_debug_set_timestamps(None)
torch.cuda.synchronize()
g.replay()
torch.cuda.synchronize()
st = [b.view(16, 1024)[14].cpu().numpy() for b in bufs]
sm = [b.view(16, 1024)[13][512:].cpu().numpy() for b in bufs]
en = [b.view(16, 1024)[15].cpu().numpy() for b in bufs]
t0 = min(x[x > 0].min() for x in st)
for i in range(n):
    a, b = st[i][st[i] > 0], en[i][en[i] > 0]
    print(f"launch {i}: CTA start {(a.min() - t0) / 1e3:7.2f}..{(a.max() - t0) / 1e3:7.2f}  "
          f"end {(b.min() - t0) / 1e3:7.2f}..{(b.max() - t0) / 1e3:7.2f} us")
# per SM: next launch's CTA start - this launch's CTA end on the same SM
for i in range(n - 1):
    ends = {int(sm[i][c]): en[i][c] for c in range(min(512, len(en[i]))) if en[i][c] > 0}
    d = [(st[i + 1][c] - ends[int(sm[i + 1][c])]) / 1e3 for c in range(min(512, len(st[i + 1])))
         if st[i + 1][c] > 0 and int(sm[i + 1][c]) in ends]
    if d:
        print(f"launch {i}->{i + 1}: same-SM end->start gap min {min(d):.2f} median {np.median(d):.2f} max {max(d):.2f} us")

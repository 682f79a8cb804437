"""K5p (prefill pair kernel) per-k-block cycle counts of CTA 0 (leader):
MMA wait for `ready`, dequant wait for `full`, dequant work.  python tools/pf_trace.py M K N"""
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
buf = torch.zeros(7 * 2048, dtype=torch.int64, device="cuda")
lib = dgq.lib()
lib.dgq_debug_set_timestamps.argtypes = [C.c_void_p]
for _ in range(2):
    CL.linear(codes, rs, out=out)
torch.cuda.synchronize()
lib.dgq_debug_set_timestamps(C.c_void_p(buf.data_ptr()))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
CL.linear(codes, rs, out=out)
e1.record()
torch.cuda.synchronize()
lib.dgq_debug_set_timestamps(None)
t = e0.elapsed_time(e1) * 1e3
print(f"{t:.1f} us  {2 * M * N * K / t / 1e6:.0f} TOPS")
bb = buf.cpu().numpy()
a0, a1, mo = bb[6144:6144 + 1024], bb[7168:8192], bb[8192:9216]
nn = int((mo > 0).sum())
t0 = min(a0[a0 > 0].min(), a1[a1 > 0].min(), mo[mo > 0].min())
ws, wf = bb[2048:3072], bb[3072:4096]
print("k-block: leader deq start / data ready / arrive | peer arrive | mma sees ready (us)")
for i in list(range(0, 8)) + list(range(40, 48)):
    print(f"  {i:4d}: {(ws[i] - t0) / 1e3:8.3f} {(wf[i] - t0) / 1e3:8.3f} {(a0[i] - t0) / 1e3:8.3f} | "
          f"{(a1[i] - t0) / 1e3:8.3f} | {(mo[i] - t0) / 1e3:8.3f}")
pe0, pe1 = bb[9216:10240], bb[10240:11264]
print("producer empty-wait cycles leader:", pe0[:12].tolist(), " median", np.median(pe0[4:nn]))
print("producer empty-wait cycles peer:  ", pe1[:12].tolist(), " median", np.median(pe1[4:nn]))
print("arrive_remote ns leader:", bb[11264:11264 + 12].tolist(), " peer:", bb[12288:12288 + 12].tolist())
b = bb[:3 * 2048].reshape(3, 2048)
n = int((b[0] > 0).sum())
for name, r in (("mma wait ready", 0), ("deq wait full", 1), ("deq work", 2)):
    v = b[r][:n]
    print(f"{name:15s} median {np.median(v):7.0f}  mean {v.mean():7.0f}  first {v[:8].tolist()}")

"""K5p per-k-block timeline of CTA 0 (the first pair's leader), globaltimer us:
producer issue (empty slot free), dequant group saw data (full), saw its B
slot free (bempty), finished (group barrier), MMA issuer saw both CTAs ready.
python tools/pf_trace.py M K N [mode]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_04836_b200 as dgq  # noqa: E402

M, K, N = (int(v) for v in sys.argv[1:4])
mode = int(sys.argv[4], 0) if len(sys.argv) > 4 else 0x400
L = dgq.random_layer(K, N, 128, seed=1)
CL = dgq.CudaLayer(L, validate=False)
x = torch.randn(M, K, device="cuda") * 3
codes, rs = CL.quantize_act(x)
out = torch.empty(M, N, dtype=torch.float16, device="cuda")
buf = torch.zeros(11 * 1024, dtype=torch.int64, device="cuda")
lib = dgq.lib()
lib.dgq_debug_set_timestamps.argtypes = [C.c_void_p]
lib.dgq_debug_set_decode.argtypes = [C.c_int]
lib.dgq_debug_set_decode(1 | mode)
for _ in range(2):
    CL.linear(codes, rs, out=out)
torch.cuda.synchronize()
lib.dgq_debug_set_timestamps(C.c_void_p(buf.data_ptr()))
CL.linear(codes, rs, out=out)
torch.cuda.synchronize()
lib.dgq_debug_set_timestamps(None)
b = buf.view(11, 1024).cpu().numpy().astype(np.float64)
n = int((b[0] > 0).sum())
t0 = b[:5, :n][b[:5, :n] > 0].min()
r = lambda v: (v - t0) / 1e3 if v > 0 else float("nan")  # noqa: E731
print(" kb | issue   full  bempty  dq-done | mma    | A-issue  loop#")
for i in list(range(20, 24)) + list(range(53, 61)):
    if i < n:
        print(f"{i:3d} | {r(b[1][i]):6.2f} {r(b[2][i]):6.2f} {r(b[3][i]):6.2f} {r(b[4][i]):6.2f} | {r(b[0][i]):6.2f} | "
              f"{r(b[5][i]):6.2f} {int(b[6][i]) if b[6][i] else 0:8d}")
d = np.diff(b[0][:n]) / 1e3
big = [(i + 1, round(float(d[i]), 2)) for i in range(len(d)) if d[i] > 1.0]
print(f"MMA of CTA 0: first {r(b[0][0]):.2f} last {r(b[0][n - 1]):.2f} us; gaps > 1 us at k-block (index, us): {big[:12]}")
print(f"MMA period median {np.median(d):.3f} us over {n} k-blocks")
print("MMA issue around the first tile boundary (k-block: us):",
      [(i, round(r(b[0][i]), 2)) for i in range(50, 60) if i < n])
lat = lambda a, c: np.median((b[c][:n] - b[a][:n]) / 1e3)  # noqa: E731
print(f"median: issue->full {lat(1, 2):.3f}  full->bempty {lat(2, 3):.3f}  bempty->done {lat(3, 4):.3f}  "
      f"done->mma {lat(4, 0):.3f}  issue->mma {lat(1, 0):.3f} us")
ep = [(round(r(b[9][2 * i]), 2), round(r(b[9][2 * i + 1]), 2)) for i in range(8) if b[9][2 * i] > 0]
print("CTA 0 epilogues (start, end) us:", ep)
for c in range(2):
    ends = [(w, round(r(b[10][c * 32 + w]), 2)) for w in range(32) if b[10][c * 32 + w] > 0]
    if ends:
        print(f"CTA {c} first-segment drain end per epilogue warp (warp, us):", ends)
print("CTA 0 second-pass starts (dbg 8):", [[round(r(b[9][640 + 4 * i + j]), 2) for j in range(2)] for i in range(4) if b[9][640 + 4 * i] > 0])
print("CTA 0 epilogue sub-tile starts / end:", [[round(r(b[9][512 + 4 * i + j]), 2) for j in range(3)] for i in range(4) if b[9][512 + 4 * i] > 0])
st, en = b[7], b[8]
ok = (st > 0) & (en > 0)
if ok.any():
    s0 = st[ok].min()
    dur = (en[ok] - s0) / 1e3
    print(f"CTAs {ok.sum()}: start spread {(st[ok].max() - s0) / 1e3:.2f} us, end min {dur.min():.2f} "
          f"median {np.median(dur):.2f} max {dur.max():.2f} us; slowest CTAs {np.argsort(-(en * ok))[:6].tolist()}")
lib.dgq_debug_set_decode(1)

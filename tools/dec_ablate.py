"""Decode-kernel ablation: time K5d with parts switched off (dgq_debug_set_decode
mode = 1 | bits << 1: bit0 no MMA, bit1 no unpack, bit2 no epilogue math, bit3 no Xq tile loads).
python tools/dec_ablate.py M K N"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_04836_b200 as dgq  # noqa: E402

M, K, N = (int(v) for v in sys.argv[1:4])
lib = dgq.lib()
lib.dgq_debug_set_decode.argtypes = [ctypes.c_int]
base = dgq.random_layer(K, N, 128, seed=3)
copies = 3
layers = [dgq.CudaLayer(base, validate=False) for _ in range(copies)]
x = torch.randn(M, K, device="cuda") * 3
codes, rs = layers[0].quantize_act(x)
out = torch.empty(M, N, dtype=torch.float16, device="cuda")
byts = K * N / 2 + (K / 128) * N * 1.5
for bits in [int(b) for b in os.environ.get('BITS', '0,1,2,4,6,7,8,15').split(',')]:
    lib.dgq_debug_set_decode(1 | (bits << 1))
    for L in layers:
        L.linear(codes, rs, out=out)
    torch.cuda.synchronize()
    n = 30
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        layers[i % copies].linear(codes, rs, out=out)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / n
    print(f"skip bits {bits:03b}: {us:8.2f} us  {byts / us / 1e3:7.1f} GB/s", flush=True)
lib.dgq_debug_set_decode(1)

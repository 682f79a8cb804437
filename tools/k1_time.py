"""K1 time / GB/s per (M, K, dtype) with a random k (every chunk divides) and
with the reference's compute_smooth k (unit chunks skip the division), inputs
drawn like bench.py's.  python tools/k1_time.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_04836_b200 as dgq  # noqa: E402
from paper_2310_04836_b200 import synth  # noqa: E402

for M, K, f16 in ((2048, 7168, False), (2048, 7168, True), (2048, 28672, True), (1, 7168, False), (1, 28672, True)):
    X = torch.from_numpy(synth.gen_synthetic(M, K, 3, 3, 50.0, 7)).cuda()
    if f16:
        X = X.half()
    res = []
    for kname in ("random", "smooth"):
        L = dgq.random_layer(K, 256, 128, seed=1)
        if kname == "smooth":
            L.k = synth.smooth_k(K)
        CL = dgq.CudaLayer(L, validate=False)
        codes, rs = CL.quantize_act(X)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            CL.quantize_act(X, codes, rs)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for _ in range(10):
                    CL.quantize_act(X, codes, rs)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        t = a.elapsed_time(b) / 10 * 1e-3
        byts = M * K * (2 if f16 else 4) + M * K + 4 * K + 4 * M
        res.append(f"{kname}: {t * 1e6:7.1f} us {byts / t / 1e9:6.0f} GB/s")
    print(f"M={M} K={K} {'f16' if f16 else 'f32'}  " + "  ".join(res), flush=True)

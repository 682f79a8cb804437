"""Per-shape K5 timing sweep (device-resident, weights rotated through > L2, launches
replayed from one CUDA graph so host overhead is excluded).
python tools/decode_sweep.py [M ...]   -> one line per (shape, M): us, GB/s (algorithmic), TOPS, plan"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_04836_b200 as dgq  # noqa: E402

import ctypes  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
_mode = 1
if "--pair" in sys.argv:  # route M >= 33 to the CTA-pair prefill kernel (K5p)
    _mode |= 0x400
if "--dec64" in sys.argv:  # K5d (decode kernel) up to 64 tokens
    _mode |= 0x10000000
if "--s2" in sys.argv:  # K5p with two token sub-tiles whenever M >= 512
    _mode |= 0x40000000
if "--tmaepi" in sys.argv:  # K5p 256-token tiles keep the TMA-store epilogue
    _mode |= 0x400000
if "--s1" in sys.argv:  # K5p with one token sub-tile per CTA (256-token pair tiles)
    _mode |= 0x20000
_cap = [int(a.split("=")[1]) for a in sys.argv[1:] if a.startswith("--cap=")]
if _cap:  # cap the K5p pair count (planner experiments)
    _l = dgq.lib()
    _l.dgq_debug_set_pair_cap.argtypes = [ctypes.c_int]
    _l.dgq_debug_set_pair_cap(_cap[0])
if "--nodec" in sys.argv:  # never the decode kernel (one-CTA kernel below 256 tokens)
    _mode &= ~1
if _mode != 1:
    _l = dgq.lib()
    _l.dgq_debug_set_decode.argtypes = [ctypes.c_int]
    _l.dgq_debug_set_decode(_mode)
Ms = [int(v) for v in args] or [1, 16, 64, 512, 2048]
shapes = [("q 7168x7168", 7168, 7168), ("fc1 7168x28672", 7168, 28672), ("fc2 28672x7168", 28672, 7168),
          ("llama7b up 4096x11008", 4096, 11008), ("c1 4096x4096", 4096, 4096)]
g = 128
L2 = 126 * 2**20
for name, K, N in shapes:
    wbytes = K * N // 2 + (K // g) * N * 2
    copies = max(2, -(-3 * L2 // wbytes))
    base = dgq.random_layer(K, N, g, seed=3)
    layers = [dgq.CudaLayer(base, validate=False) for _ in range(copies)]
    for M in Ms:
        x = torch.randn(M, K, device="cuda") * 3
        codes, rs = layers[0].quantize_act(x)
        out = torch.empty(M, N, dtype=torch.float16, device="cuda")
        for L in layers:
            L.linear(codes, rs, out=out)
        torch.cuda.synchronize()
        n = max(copies * 4, 24)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g_ = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g_, stream=s):
                for i in range(n):
                    layers[i % copies].linear(codes, rs, out=out)
        torch.cuda.synchronize()
        g_.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g_.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / n
        byts = M * K + 4 * M + K * N / 2 + (K / g) * N * 1.5 + 4 * N + 2 * M * N
        ops = 2.0 * M * N * K
        plan = layers[0].plan(M)
        print(f"{name:24s} M={M:5d} {us:8.2f} us  {byts / us / 1e3:7.1f} GB/s  {ops / us / 1e6:7.1f} TOPS  {plan}",
              flush=True)
    del layers
    torch.cuda.empty_cache()

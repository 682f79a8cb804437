"""Per-launch floor of the K5 kernels: a CUDA graph of 64 back-to-back launches
of one small layer (L2-resident), per-launch time.  python tools/launch_floor.py"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2310_04836_b200 as dgq  # noqa: E402

lib = dgq.lib()
lib.dgq_debug_set_decode.argtypes = [ctypes.c_int]
for mode, name in ((1, "default"), (1 | 0x8000000, "K5d"), (1 | 0x100, "noPDL")):
    lib.dgq_debug_set_decode(mode)
    for K, N in ((128, 128), (1024, 1024), (4096, 4096), (7168, 7168)):
        L = bench.tiled_layer(K, N, seed=3)
        CL = dgq.CudaLayer(L)
        x = torch.from_numpy(bench._synth_x(1, K)).cuda()
        codes, rs = CL.quantize_act(x)
        y = torch.empty(1, N, dtype=torch.float16, device="cuda")
        t = bench._stream_time([lambda: CL.linear(codes, rs, out=y)] * 64)
        t1 = bench._stream_time([lambda: CL.quantize_act(x, codes, rs)] * 64)
        print(f"{name:8s} K={K:5d} N={N:5d} M=1: K5 {t * 1e6:6.2f} us/launch  K1 {t1 * 1e6:6.2f} us/launch "
              f"plan {CL.plan(1)}", flush=True)

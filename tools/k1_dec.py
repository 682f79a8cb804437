"""K1 per-launch time at decode shapes (graph of 64 launches, L2-resident input)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2310_04836_b200 as dgq  # noqa: E402
from paper_2310_04836_b200 import synth  # noqa: E402

for M in (1, 16):
    for K, f16 in ((4096, False), (7168, False), (7168, True), (28672, True)):
        L = bench.tiled_layer(K, 512, seed=3)
        CL = dgq.CudaLayer(L)
        x = torch.from_numpy(bench._synth_x(M, K)).cuda()
        if f16:
            x = x.half()
        codes, rs = CL.quantize_act(x)
        t = bench._stream_time([lambda: CL.quantize_act(x, codes, rs)] * 64)
        print(f"M={M:2d} K={K:5d} {'f16' if f16 else 'f32'}: {t * 1e6:6.2f} us/launch", flush=True)

"""Back-to-back launch cost of the fused linear on a tiny layer (K = N = 128,
M = 1): graph replay of 32 launches, K5d (decode) vs the one-CTA kernel."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_04836_b200 as dgq  # noqa: E402

lib = dgq.lib()
lib.dgq_debug_set_decode.argtypes = [ctypes.c_int]
for K, N in ((128, 128), (1024, 1024), (7168, 7168)):
    L = dgq.CudaLayer(dgq.random_layer(K, N, 128, seed=1), validate=False)
    x = torch.randn(1, K, device="cuda")
    codes, rs = L.quantize_act(x)
    out = torch.empty(1, N, dtype=torch.float16, device="cuda")
    for mode, name in ((1, "K5d decode"), (0, "one-CTA kernel")):
        lib.dgq_debug_set_decode(mode)
        L.linear(codes, rs, out=out)
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for _ in range(32):
                    L.linear(codes, rs, out=out)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        print(f"K=N={K:5d} {name:16s}: {e0.elapsed_time(e1) * 1e3 / 32:6.2f} us per launch {L.plan(1)}", flush=True)
lib.dgq_debug_set_decode(1)

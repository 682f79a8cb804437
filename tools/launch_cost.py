"""Per-launch cost of tiny kernels replayed back to back from a CUDA graph:
torch's own elementwise kernel vs this library's K1 and K5d at M = 1.
python tools/launch_cost.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_04836_b200 as dgq  # noqa: E402


def per_launch(fn, n=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) * 1e3 / n


t = torch.zeros(1024, device="cuda")
print(f"torch add_ (1 block)         : {per_launch(lambda: t.add_(1)):6.2f} us")
big = torch.zeros(148 * 512 * 4, device="cuda")
print(f"torch add_ (296 blocks)      : {per_launch(lambda: big.add_(1)):6.2f} us")
for K in (128, 7168):
    L = dgq.random_layer(K, 128, 128, seed=1)
    CL = dgq.CudaLayer(L, validate=False)
    x = torch.randn(1, K, device="cuda")
    codes, rs = CL.quantize_act(x)
    out = torch.empty(1, 128, dtype=torch.float16, device="cuda")
    print(f"K1  M=1 K={K:5d}             : {per_launch(lambda: CL.quantize_act(x, codes, rs)):6.2f} us")
    print(f"K5d M=1 K={K:5d} N=128       : {per_launch(lambda: CL.linear(codes, rs, out=out)):6.2f} us")

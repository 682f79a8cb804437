"""K5d back-to-back launch time with and without PDL (graph replay).
python tools/dec_pdl.py M K N"""
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
layers = [dgq.CudaLayer(base, validate=False) for _ in range(3)]
x = torch.randn(M, K, device="cuda") * 3
codes, rs = layers[0].quantize_act(x)
out = torch.empty(M, N, dtype=torch.float16, device="cuda")
for mode in (1, 1 | 0x100):
    lib.dgq_debug_set_decode(mode)
    for L in layers:
        L.linear(codes, rs, out=out)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    n = 24
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(n):
                layers[i % 3].linear(codes, rs, out=out)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"pdl={'off' if mode & 0x100 else 'on '}: {e0.elapsed_time(e1) * 1e3 / n:.2f} us per launch", flush=True)
lib.dgq_debug_set_decode(1)

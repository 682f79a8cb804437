"""Run a few fused-linear launches of one shape (for ncu captures).
python tools/one.py M K N g [n_launch]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_04836_b200 as dgq  # noqa: E402

M, K, N, g = (int(v) for v in sys.argv[1:5])
n = int(sys.argv[5]) if len(sys.argv) > 5 else 3
L = dgq.random_layer(K, N, g, seed=1)
CL = dgq.CudaLayer(L, validate=False)
x = torch.randn(M, K, device="cuda") * 3
codes, rs = CL.quantize_act(x)
out = torch.empty(M, N, dtype=torch.float16, device="cuda")
for _ in range(n):
    CL.linear(codes, rs, out=out)
torch.cuda.synchronize()
print("done", M, K, N, g)

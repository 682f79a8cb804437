"""Run K1 (activation quantisation) a few times for ncu. python tools/k1.py M K f16|f32"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_04836_b200 as dgq  # noqa: E402

M, K = int(sys.argv[1]), int(sys.argv[2])
dt = torch.float16 if sys.argv[3] == "f16" else torch.float32
L = dgq.random_layer(K, 256, 128, seed=1)
CL = dgq.CudaLayer(L, validate=False)
x = (torch.randn(M, K, device="cuda") * 3).to(dt)
for _ in range(3):
    CL.quantize_act(x)
torch.cuda.synchronize()
print("done")

"""One K1 shape, a few launches (for ncu): python tools/k1_one.py M K f16|f32 [smooth|random]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_04836_b200 as dgq  # noqa: E402
from paper_2310_04836_b200 import synth  # noqa: E402

M, K, dt = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
X = torch.from_numpy(synth.gen_synthetic(M, K, 3, 3, 50.0, 7)).cuda()
if dt == "f16":
    X = X.half()
L = dgq.random_layer(K, 256, 128, seed=1)
if len(sys.argv) < 5 or sys.argv[4] == "smooth":
    L.k = synth.smooth_k(K)
CL = dgq.CudaLayer(L, validate=False)
codes, rs = CL.quantize_act(X)
for _ in range(4):
    CL.quantize_act(X, codes, rs)
torch.cuda.synchronize()

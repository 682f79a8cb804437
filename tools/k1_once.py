"""One K1 launch per (M, K, fp16) for ncu captures (inputs drawn like bench.py's,
k from compute_smooth).  python tools/k1_once.py M K f16"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_04836_b200 as dgq  # noqa: E402
from paper_2310_04836_b200 import synth  # noqa: E402

M, K, f16 = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3] == "1"
X = torch.from_numpy(synth.gen_synthetic(M, K, 3, 3, 50.0, 7)).cuda()
if f16:
    X = X.half()
L = dgq.random_layer(K, 256, 128, seed=1)
L.k = synth.smooth_k(K)
CL = dgq.CudaLayer(L, validate=False)
codes, rs = CL.quantize_act(X)
for _ in range(3):
    CL.quantize_act(X, codes, rs)
torch.cuda.synchronize()
print("ok", codes.shape)

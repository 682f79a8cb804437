"""The bench's fused q/k/v launch (three OPT-30B 7168x7168 layers over one
input, dgq_linear_multi) a few times (for ncu): python tools/k5_qkv.py [M]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2310_04836_b200 as dgq  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
K = N = 7168
Ls = [bench.tiled_layer(K, N, seed=100 + i) for i in range(3)]
for L in Ls[1:]:
    L.k = Ls[0].k
CLs = [dgq.CudaLayer(L) for L in Ls]
x = torch.from_numpy(bench._synth_x(M, K)).cuda()
codes, rs = CLs[0].quantize_act(x)
outs = [torch.empty(M, N, dtype=torch.float16, device="cuda") for _ in range(3)]
for _ in range(4):
    dgq.linear_multi(CLs, codes, rs, outs=outs)
torch.cuda.synchronize()
print(CLs[0].plan(M))

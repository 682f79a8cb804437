"""One K5 launch shape a few times (for ncu): python tools/k5_one.py M K N [mode]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2310_04836_b200 as dgq  # noqa: E402

M, K, N = (int(a) for a in sys.argv[1:4])
if len(sys.argv) > 4:
    dgq.lib().dgq_debug_set_decode.argtypes = [ctypes.c_int]
    dgq.lib().dgq_debug_set_decode(int(sys.argv[4], 0))
L = bench.tiled_layer(K, N, seed=3)
CL = dgq.CudaLayer(L)
x = torch.from_numpy(bench._synth_x(M, K)).cuda()
codes, rs = CL.quantize_act(x)
y = torch.empty(M, N, dtype=torch.float16, device="cuda")
for _ in range(4):
    CL.linear(codes, rs, out=y)
torch.cuda.synchronize()
print(CL.plan(M))

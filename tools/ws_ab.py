"""A/B: K5 launch time with a caller workspace vs the library's per-stream
internal workspace (graph-replayed, L2 flushed)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2310_04836_b200 as dgq  # noqa: E402

torch.cuda.set_device(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for (K, N) in ((7168, 28672), (7168, 7168)):
    L = bench.tiled_layer(K, N, seed=1)
    CL = dgq.CudaLayer(L)
    for M in (1, 16, 32, 64):
        x = torch.randn(M, K, device="cuda")
        codes, rs = CL.quantize_act(x)
        y = torch.empty(M, N, dtype=torch.float16, device="cuda")
        ws = CL.workspace(M)
        r = {}
        for name, w in (("caller", ws), ("internal", None), ("caller2", ws), ("internal2", None)):
            r[name] = bench._graph_time(lambda: CL.linear(codes, rs, out=y, workspace=w), flush, reps=20) * 1e6
        print(K, N, M, CL.plan(M), {k: round(v, 2) for k, v in r.items()}, flush=True)

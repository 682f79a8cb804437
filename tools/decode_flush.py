"""K5d single-launch HBM GB/s at M tokens for OPT-30B q (7168^2) and fc1, with
the L2 emptied between launches by a 256 MiB WRITE (dirty lines: the kernel's
reads pay their write-back) or a 256 MiB READ (clean lines), and back to back.
python tools/decode_flush.py [M]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_04836_b200 as dgq  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1
flush = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
fl64 = flush.view(torch.int64)
sink = torch.zeros((), dtype=torch.int64, device="cuda")


def graph(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.synchronize()
    return g


for name, K, N in (("q", 7168, 7168), ("fc1", 7168, 28672), ("fc2", 28672, 7168)):
    L = dgq.random_layer(K, N, 128, seed=1)
    CL = dgq.CudaLayer(L, validate=False)
    codes, rs = CL.quantize_act(torch.randn(M, K, device="cuda"))
    out = torch.empty(M, N, dtype=torch.float16, device="cuda")
    g = graph(lambda: CL.linear(codes, rs, out=out))
    byts = M * K + 4 * M + K * N / 2 + (K / 128) * N * 1.5 + 4 * N + 2 * M * N
    res = {}
    for mode in ("write", "read", "none"):
        ts = []
        for _ in range(10):
            if mode == "write":
                flush.zero_()
            elif mode == "read":
                torch.sum(fl64, dim=(0,), out=sink)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        t = sorted(ts)[len(ts) // 2]
        res[mode] = (t * 1e6, byts / t / 1e9)
    # back to back: 20 launches in one graph
    g20 = graph(lambda: [CL.linear(codes, rs, out=out) for _ in range(20)])
    torch.sum(fl64, dim=(0,), out=sink)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g20.replay()
    b.record()
    b.synchronize()
    t = a.elapsed_time(b) * 1e-3 / 20
    res["b2b"] = (t * 1e6, byts / t / 1e9)
    print(name, M, " ".join(f"{k}: {v[0]:.1f}us {v[1]:.0f}GB/s" for k, v in res.items()), flush=True)

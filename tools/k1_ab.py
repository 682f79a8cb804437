"""K1 steady-state GB/s per input shape (HBM-resident: launches rotate over
input copies totalling > 2.2x L2, one CUDA graph), with the reference's
compute_smooth k and with a random k (every chunk divides).  Prints a digest
of the codes so builds / variants can be compared for equality.
DGQ_K1_VERSION=3|4, DGQ_K1_T=256|512 select the kernel (tools only)."""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_04836_b200 as dgq  # noqa: E402
from paper_2310_04836_b200 import synth  # noqa: E402

SHAPES = [(2048, 7168, False), (2048, 7168, True), (2048, 28672, True), (512, 7168, False), (4096, 4096, False),
          (2048, 11008, True)]
for M, K, f16 in SHAPES:
    X0 = torch.from_numpy(synth.gen_synthetic(M, K, 3, 3, 50.0, 7)).cuda()
    if f16:
        X0 = X0.half()
    nb = X0.numel() * X0.element_size()
    copies = max(2, int(2.2 * 126e6 / nb) + 1)
    Xs = [X0.clone() for _ in range(copies)]
    res = []
    for kname in ("smooth", "random"):
        L = dgq.random_layer(K, 256, 128, seed=1)
        if kname == "smooth":
            L.k = synth.smooth_k(K)
        CL = dgq.CudaLayer(L, validate=False)
        codes, rs = CL.quantize_act(X0)
        torch.cuda.synchronize()
        dig = hashlib.sha1(codes.cpu().numpy().tobytes() + rs.cpu().numpy().tobytes()).hexdigest()[:10]
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            CL.quantize_act(X0, codes, rs)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for x in Xs:
                    CL.quantize_act(x, codes, rs)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b) * 1e-3 / copies)
        byts = M * K * (2 if f16 else 4) + M * K + 4 * K + 4 * M
        res.append(f"{kname}: {best * 1e6:6.1f} us {byts / best / 1e9:5.0f} GB/s [{dig}]")
        del g
    print(f"M={M:5d} K={K:5d} {'f16' if f16 else 'f32'}  " + "  ".join(res), flush=True)
    del Xs
    torch.cuda.empty_cache()

"""Kernel-level timing probe (not the bench contract).

For each shape: R distinct prepared layers (R chosen so the weights exceed
2x L2, i.e. every launch streams its weights from HBM), one CUDA graph of R
back-to-back K5 launches, replayed; time = graph time / R.  K1 is timed the
same way on R distinct inputs.
python tools/probe.py [--shapes M,K,N,g ...] [--reps R]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_04836_b200 as dgq  # noqa: E402

HBM = 6545.6
I8 = 2 * 1632.4
L2 = 126e6

DEFAULT = ["1,4096,4096,128", "16,4096,4096,128", "16,4096,4096,64", "64,8192,2752,128", "1,4096,11008,128",
           "512,7168,7168,128", "2048,4096,4096,128", "2048,4096,11008,128", "2048,7168,28672,128",
           "2048,28672,7168,128"]


def graph_time(fn_list, reps):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for f in fn_list:  # warm (cudaFuncSetAttribute etc. outside capture)
            f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for f in fn_list:
            f()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e-3)
    return best / len(fn_list)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", nargs="*", default=DEFAULT)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    print(f"{'M':>5} {'K':>6} {'N':>6} {'g':>4} | {'K5 us':>8} {'TOPS':>7} {'GB/s':>7} {'%HBM':>5} {'%I8px':>5} | "
          f"{'K1 us':>7} {'K1 GB/s':>7}")
    for s in a.shapes:
        M, K, N, g = map(int, s.split(","))
        wbytes = K * N / 2
        R = max(1, min(32, int(2 * L2 / wbytes) + 1))
        layers = [dgq.CudaLayer(dgq.random_layer(K, N, g, seed=1 + i % 2), validate=False) for i in range(R)]
        CL = layers[0]
        xs = [torch.randn(M, K, device="cuda") * 3 for _ in range(min(R, 4))]
        codes, rs = CL.quantize_act(xs[0])
        out = torch.empty(M, N, dtype=torch.float16, device="cuda")
        wss = [L.workspace(M) for L in layers]
        t5 = graph_time([lambda L=L, w=w: L.linear(codes, rs, out=out, workspace=w) for L, w in zip(layers, wss)],
                        a.reps)
        t1 = graph_time([lambda x=x: CL.quantize_act(x, codes, rs) for x in xs], a.reps)
        ops = 2.0 * M * N * K
        byt = M * K + 4 * M + K * N / 2 + (K / g) * N * 1.5 + 4 * N + 2 * M * N
        b1 = 4 * M * K + 4 * K + M * K + 4 * M
        print(f"{M:5d} {K:6d} {N:6d} {g:4d} | {t5 * 1e6:8.1f} {ops / t5 / 1e12:7.1f} {byt / t5 / 1e9:7.0f} "
              f"{byt / t5 / 1e9 / HBM * 100:5.1f} {ops / t5 / 1e12 / I8 * 100:5.1f} | {t1 * 1e6:7.1f} "
              f"{b1 / t1 / 1e9:7.0f}", flush=True)
        for L in layers:
            L.close()


if __name__ == "__main__":
    main()

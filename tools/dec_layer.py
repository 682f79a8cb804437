"""Decode-shaped steady-state timing per K5 shape (streaming over weight copies
> 2.2x L2, CUDA-graph replay) — planner default vs forced K5d (mode bit 27).
python tools/dec_layer.py"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

hbm = bench.load_peaks()[0]
lib = __import__("paper_2310_04836_b200").lib()
lib.dgq_debug_set_decode.argtypes = [ctypes.c_int]
for mode, name in ((1, "default"), (1 | 0x8000000, "K5d")):
    lib.dgq_debug_set_decode(mode)
    for K, N in ((4096, 4096), (7168, 7168), (7168, 28672), (28672, 7168), (8192, 2752), (22016, 1024)):
        r = bench.linear_point(K, N, [1, 2, 4, 8], torch.device("cuda", 0), hbm, 4560.0)
        print(name, K, N, {m: (v["us"], v["frac"], v["plan"]["token_tile"]) for m, v in r.items()}, flush=True)

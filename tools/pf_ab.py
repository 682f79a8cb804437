"""Prefill K5 per-shape steady-state time under planner mode overrides.
python tools/pf_ab.py [mode ...]   (mode ints, e.g. 1 0x40000801)"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2310_04836_b200 as dgq  # noqa: E402

lib = dgq.lib()
lib.dgq_debug_set_decode.argtypes = [ctypes.c_int]
modes = [int(a, 0) for a in sys.argv[1:]] or [1]
shapes = [(7168, 7168), (7168, 28672), (28672, 7168), (4096, 4096), (4096, 11008), (11008, 4096)]
for K, N in shapes:
    for mode in modes:
        lib.dgq_debug_set_decode(mode)
        r = bench.linear_point(K, N, [512, 1024, 2048], torch.device("cuda", 0), 6500.0, 4560.0)
        print(f"mode {mode:#x} K={K} N={N}: " +
              " ".join(f"M{m}: {v['us']}us {v['TOPS']}T" for m, v in r.items()), flush=True)

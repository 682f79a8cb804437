"""Decode-layer step time (bench.OptLayer, CUDA-graph replay, L2 flushed):
python tools/dec_step.py [M ...]  (default 1 16)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

Ms = [int(a) for a in sys.argv[1:]] or [1, 16]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
layer = bench.OptLayer(0, 1, dev, None, 64)
layer.x.copy_(torch.from_numpy(bench._synth_x(64, 7168)))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for M in Ms:
    ts = [bench.decode_step_time(layer, M, flush, torch.cuda.synchronize, 1, reps=20) for _ in range(3)]
    print(f"pre={os.environ.get('DGQ_DEC_PRE', 'default')} M={M}: {min(ts) * 1e6:.1f} us (runs {[round(t * 1e6, 1) for t in ts]})",
          flush=True)

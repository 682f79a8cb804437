"""Run only bench.py's comparators (OPT-30B fc1) — quick check of the A16W4 / A8W8 baselines."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

torch.cuda.set_device(0)
layer = bench.OptLayer(0, 1, torch.device("cuda", 0), None, bench.SEQ)
x = torch.from_numpy(bench._synth_x(bench.SEQ, 7168)).cuda()
layer.x.copy_(x)
layer.step(bench.SEQ)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
print(json.dumps(bench.comparators(layer, flush), indent=1))

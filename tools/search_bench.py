"""Grid-search throughput: GPU phase1/phase2 (CUDA events) vs the reference's
CPU phase1_search/phase2_search (all host threads) on the same inputs.
python tools/search_bench.py [h o b g] ..."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle  # noqa: E402
from paper_2310_04836_b200 import search  # noqa: E402
from test_search_gpu import problem  # noqa: E402

shapes = [(1024, 1024, 256, 128), (4096, 4096, 256, 128)]
cpu_max = 1024 * 1024
for h, o, b, g in shapes:
    W, X, Xh = problem(h, o, b, seed=1)
    dW, dX, dXh = (torch.from_numpy(a).cuda() for a in (W, X, Xh))
    cfg = search.SearchConfig(group_size=g, calib_X=dX)
    gp = search.phase1_search(dW, cfg, dXh)  # warm
    r2 = search.phase2_search(dW, gp, cfg, dXh)
    torch.cuda.synchronize()
    ts = []
    for fn in (lambda: search.phase1_search(dW, cfg, dXh), lambda: search.phase2_search(dW, gp, cfg, dXh)):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(a.elapsed_time(e) * 1e-3)
    n1, n2 = len(cfg.alpha_grid_phase1), len(cfg.alpha_grid_phase2)
    fma1 = h * o * b * (n1 + 1)  # objectives + reference dots
    fma2 = h * o * b * (n2 + 1)
    line = (f"h={h} o={o} b={b} g={g}: GPU phase1 {ts[0]*1e3:.1f} ms ({fma1/ts[0]/1e12:.2f} T FP64-FMA/s), "
            f"phase2 {ts[1]*1e3:.1f} ms ({fma2/ts[1]/1e12:.2f} T/s)")
    if h * o <= cpu_max and oracle.have_ref():
        R = oracle.ref()
        t0 = time.perf_counter()
        sp, zp, er, al, _ = R.phase1_search(W, X, Xh, g, search.default_grid1())
        t1 = time.perf_counter()
        R.phase2_search(W, X, Xh, g, sp, zp, search.default_grid2())
        t2 = time.perf_counter()
        line += (f" | reference CPU ({os.cpu_count()} threads): phase1 {t1-t0:.2f} s, phase2 {t2-t1:.2f} s"
                 f" -> {(t1-t0)/ts[0]:.0f}x / {(t2-t1)/ts[1]:.0f}x"
                 f" | bit-exact: {np.array_equal(sp, gp.s_prime) and np.array_equal(zp, gp.zp)}")
    print(line, flush=True)

#!/bin/bash
# compute-sanitizer passes over small launches of every fused-linear kernel
# (K5d decode, K5p CTA pair, one-CTA K5) and K1.  Run under gpurun.
cat > /tmp/san_case.py <<'PY'
import ctypes, sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import oracle, paper_2310_04836_b200 as dgq
M, h, o, g, mode = (int(v) for v in sys.argv[1:6])
lib = dgq.lib(); lib.dgq_debug_set_decode.argtypes = [ctypes.c_int]; lib.dgq_debug_set_decode(mode)
port = oracle.port()
L = oracle.random_layer(h, o, g, seed=7)
X = port.gen_synthetic(M, h, 3, 3, 50.0, 3)
out, *_ = port.dgq_forward(X, L)
D = dgq.DgqLayer(h=L.h, o=L.o, g=L.g, codes=L.codes, s2=L.s2, zp=L.zp, s1=L.s1, k=L.k, act_scale=L.act_scale, mode=L.mode)
CL = dgq.CudaLayer(D)
y = CL.forward(torch.from_numpy(X).cuda(), out_dtype=torch.float32)
torch.cuda.synchronize()
ok = np.array_equal(y.cpu().numpy().view(np.uint32), out.view(np.uint32))
print("case", M, h, o, g, mode, CL.plan(M), "bit-exact" if ok else "MISMATCH")
PY
for tool in memcheck racecheck synccheck; do
  # K5d (forced, mode bit 27) | K5p S=1 | K5p S=2 (bit 30) | planner default (g=64) | one-CTA K5 | K1 v3 (M >= SMs)
  for c in "4 4096 512 128 134217729" "300 512 512 128 1025" "600 1024 512 128 1073742849" "300 512 512 64 1" \
           "64 512 256 128 1" "200 2048 256 128 1"; do
    echo "== $tool $c"
    timeout 600 compute-sanitizer --tool $tool --print-limit 5 python /tmp/san_case.py $c 2>&1 | grep -E "case|ERROR SUMMARY|Error|Hazard" | head -6
  done
done

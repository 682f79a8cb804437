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
cat > /tmp/san_multi.py <<'PY'
import ctypes, sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import oracle, paper_2310_04836_b200 as dgq
from paper_2310_04836_b200 import synth
M, h, mode = (int(v) for v in sys.argv[1:4])
lib = dgq.lib(); lib.dgq_debug_set_decode.argtypes = [ctypes.c_int]; lib.dgq_debug_set_decode(mode)
port = oracle.port()
Ls = [oracle.random_layer(h, o, 128, seed=o) for o in (256, 384, 130)]
for L in Ls[1:]:
    L.k = Ls[0].k
X = port.gen_synthetic(M, h, 3, 3, 50.0, 3)
CLs = [dgq.CudaLayer(dgq.DgqLayer(h=L.h, o=L.o, g=L.g, codes=L.codes, s2=L.s2, zp=L.zp, s1=L.s1, k=L.k,
                                   act_scale=L.act_scale, mode=L.mode)) for L in Ls]
codes, rs = CLs[0].quantize_act(torch.from_numpy(X).cuda())
ys = dgq.linear_multi(CLs, codes, rs, out_dtype=torch.float32)
torch.cuda.synchronize()
ok = all(np.array_equal(y.cpu().numpy().view(np.uint32), port.dgq_forward(X, L)[0].view(np.uint32)) for y, L in zip(ys, Ls))
# K1 exact persistent shape (C8 = 7 x 128 chunks, smoothed k, FP16 input)
K = 7168
k = synth.smooth_k(K)
Xk = port.gen_synthetic(300, K, 5, 3, 50.0, 7).astype(np.float16).astype(np.float32)
q, r = port.quantize_activations(Xk, k, 1, 0.0)
Lk = dgq.DgqLayer(h=K, o=2, g=K // 8, codes=np.zeros(K, np.uint8), s2=np.ones((8, 2), np.int8),
                  zp=np.zeros(8, np.uint8), s1=np.ones(2, np.float32), k=k, act_scale=0.0, mode=1)
c2, r2 = dgq.CudaLayer(Lk).quantize_act(torch.from_numpy(Xk).cuda().half())
torch.cuda.synchronize()
ok = ok and np.array_equal(c2[:, :K].cpu().numpy(), q)
print("multi", M, h, mode, CLs[0].plan(M), "bit-exact" if ok else "MISMATCH")
PY
for tool in memcheck racecheck synccheck; do
  echo "== $tool multi-layer K5p (S = 2, stream-K balanced) + K1 exact"
  timeout 600 compute-sanitizer --tool $tool --print-limit 5 python /tmp/san_multi.py 600 1024 1073742849 2>&1 | grep -E "multi|ERROR SUMMARY|Error|Hazard" | head -6
done
for tool in memcheck racecheck synccheck; do
  # K5d (forced, mode bit 27) | K5p S=1 | K5p S=2 (bit 30) | planner default (g=64) | one-CTA K5 | K1 v3 (M >= SMs)
  for c in "4 4096 512 128 134217729" "300 512 512 128 1025" "600 1024 512 128 1073742849" "300 512 512 64 1" \
           "64 512 256 128 1" "200 2048 256 128 1"; do
    echo "== $tool $c"
    timeout 600 compute-sanitizer --tool $tool --print-limit 5 python /tmp/san_case.py $c 2>&1 | grep -E "case|ERROR SUMMARY|Error|Hazard" | head -6
  done
done

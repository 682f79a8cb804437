"""Randomised parity of the pair kernel (K5p) paths added in round 2 — the
balanced stream-K split (csrc/prefill.cu sk_bounds) and several layers in one
launch (dgq_linear_multi) — against the oracle's dgq_forward
(proj/src/kernel.cpp:144-153): FP32 outputs bit-exact, FP16 outputs equal
fp16_round(FP32).  Shapes, group sizes, layer counts and widths are drawn from
a fixed seed, so a failure is reproducible from its id."""
import ctypes

import numpy as np
import pytest
import torch

import oracle
import paper_2310_04836_b200 as dgq

pytestmark = pytest.mark.gpu


def _to_dgq(L):
    return dgq.DgqLayer(h=L.h, o=L.o, g=L.g, codes=L.codes.copy(), s2=np.asarray(L.s2).copy(), zp=L.zp.copy(),
                        s1=L.s1.copy(), k=L.k.copy(), act_scale=L.act_scale, mode=L.mode)


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def _cases(n=24, seed=2024):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        g = int(rng.choice([32, 64, 128]))
        h = int(rng.integers(2, 17)) * 128
        count = int(rng.integers(1, 4))
        widths = tuple(int(rng.integers(1, 6)) * 2 * int(rng.choice([1, 64, 128])) for _ in range(count))
        M = int(rng.integers(256, 1300))
        mode = int(rng.choice([0x400, 0x400 | 0x40000000, 0x400 | 0x20000]))  # K5p, S = 2 forced, S = 1
        out.append((i, M, h, widths, g, mode))
    return out


@pytest.mark.parametrize("i,M,h,widths,g,mode", _cases())
def test_pair_kernel_random_shapes_match_oracle(cuda, port, i, M, h, widths, g, mode):
    lib = dgq.lib()
    lib.dgq_debug_set_decode.argtypes = [ctypes.c_int]
    lib.dgq_debug_set_decode(1 | mode)
    try:
        Ls = [oracle.random_layer(h, o, g, seed=1000 * i + j) for j, o in enumerate(widths)]
        for L in Ls[1:]:
            L.k = Ls[0].k  # one input: one smoothing vector
        X = port.gen_synthetic(M, h, 17 + i, 3, 50.0, 3)
        CLs = [dgq.CudaLayer(_to_dgq(L)) for L in Ls]
        codes, rs = CLs[0].quantize_act(torch.from_numpy(X).cuda())
        refs = [port.dgq_forward(X, L)[0] for L in Ls]
        outs = dgq.linear_multi(CLs, codes, rs, out_dtype=torch.float32)
        for j, ref in enumerate(refs):
            assert np.array_equal(_bits(outs[j].cpu().numpy()), _bits(ref)), (j, CLs[j].plan(M))
        outs16 = dgq.linear_multi(CLs, codes, rs, out_dtype=torch.float16)
        for j, ref in enumerate(refs):
            assert np.array_equal(_bits(outs16[j].cpu().numpy()),
                                  _bits(port.fp16_round_array(ref).astype(np.float16))), j
    finally:
        lib.dgq_debug_set_decode(1)

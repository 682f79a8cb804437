"""Generate tests/golden/golden_v1.npz by running the REFERENCE ITSELF
(oracle/_ref/libdgq_ref.so = /root/reference/proj/src compiled unmodified).

Run in the build container (where /root/reference exists):
    make -C oracle && python tests/golden/make_golden.py
The vectors pin both the C restatement (oracle/dgq_oracle.c) and the CUDA
path on machines where the reference is absent (the GPU box).
Cases mirror the reference's hot-path tests (proj/tests/test_kernel.cpp,
test_format.cpp, test_quant.cpp, test_search.cpp) plus SURVEY.md §8d edges.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def main():
    R = oracle.ref()
    out = {}

    def put(prefix, **kw):
        for k, v in kw.items():
            out[f"{prefix}.{k}"] = np.asarray(v)

    # ---- K1: activation quantisation ------------------------------------
    calib = R.gen_synthetic(64, 256, 100, 3, 50.0, 7)
    k, th = R.smooth_from_calib(calib, 0.005)
    X = R.gen_synthetic(16, 256, 101, 3, 50.0, 7)
    q, rs = R.quantize_activations(X, k, 1, 0.0)
    put("actq_dyn", X=X, k=k, codes=q, rs=rs, threshold=np.float32(th))
    xs = (X / k).astype(np.float32)
    act = np.float32(np.abs(xs).max() / 127.0 * 0.8)  # static, saturating
    q, rs = R.quantize_activations(X, k, 0, float(act))
    put("actq_static", X=X, k=k, act_scale=act, codes=q, rs=rs)
    rng = np.random.default_rng(3)
    Xo = rng.uniform(-2, 2, (5, 33)).astype(np.float32)
    ko = rng.uniform(1, 3, 33).astype(np.float32)
    q, rs = R.quantize_activations(Xo, ko, 1, 0.0)
    put("actq_odd", X=Xo, k=ko, codes=q, rs=rs)
    # exact ties (absmax 127 -> s = 1), a zero row, and a row of tiny values
    Xe = np.zeros((3, 8), np.float32)
    Xe[0] = [127, 0.5, 1.5, 2.5, -0.5, -1.5, -2.5, 126.5]
    Xe[2] = [1e-30, -3e-38, 0, 1e-40, 2e-38, -1e-39, 5e-45, 0]
    ke = np.ones(8, np.float32)
    q, rs = R.quantize_activations(Xe, ke, 1, 0.0)
    put("actq_edge", X=Xe, k=ke, codes=q, rs=rs)

    # ---- K2s: dequantisation -----------------------------------------------
    for name, (h, o, g) in {"deq_g64": (256, 64, 64), "deq_g128": (512, 32, 128), "deq_g8": (64, 16, 8),
                            "deq_g12": (48, 10, 12)}.items():
        L = oracle.random_layer(h, o, g, seed=h + o + g)
        w = R.dequantize_to_s8(L)
        put(name, h=h, o=o, g=g, codes=L.codes, s2=L.s2, zp=L.zp, w_s8=w)

    # ---- K3: int8 GEMM -------------------------------------------------------
    rng = np.random.default_rng(4)
    for name, (M, K, N) in {"gemm_16x64x8": (16, 64, 8), "gemm_9x33x7": (9, 33, 7),
                            "gemm_40x300x130": (40, 300, 130)}.items():
        A = rng.integers(-127, 128, (M, K)).astype(np.int8)
        B = rng.integers(-127, 128, (K, N)).astype(np.int8)
        acc, mx = R.int8_gemm(A, B, 1)
        put(name, Xq=A, Wq=B, acc=acc, max_abs_acc=np.int64(mx))
    A = np.full((2, 256), 127, np.int8)
    B = np.full((256, 2), 127, np.int8)
    acc, mx = R.int8_gemm(A, B, 1)
    put("gemm_all127", Xq=A, Wq=B, acc=acc, max_abs_acc=np.int64(mx))

    # ---- K4: epilogue ------------------------------------------------------------
    accE = rng.integers(-2_000_000, 2_000_000, (8, 12)).astype(np.int32)
    rsE = rng.uniform(1e-4, 2e-2, 8).astype(np.float32)
    s1E = rng.uniform(1e-3, 2e-2, 12).astype(np.float32)
    bE = rng.uniform(-1, 1, 12).astype(np.float32)
    put("epi", acc=accE, rs=rsE, s1=s1E, bias=bE, y=R.epilogue(accE, rsE, s1E, None, False),
        y_bias=R.epilogue(accE, rsE, s1E, bE, False), y_f16mode=R.epilogue(accE, rsE, s1E, None, True),
        y_f16mode_bias=R.epilogue(accE, rsE, s1E, bE, True))

    # ---- K5: full forward (dgq_forward) ------------------------------------------
    L = oracle.random_layer(256, 256, 64, seed=11)
    L.k = k
    Xf = R.gen_synthetic(16, 256, 201, 3, 50.0, 7)
    bias = rng.uniform(-0.5, 0.5, 256).astype(np.float32)
    o_, w_, q_, r_, m_ = R.dgq_forward(Xf, L, bias, 1)
    put("fwd_a", X=Xf, h=256, o=256, g=64, mode=1, act_scale=np.float32(0), codes=L.codes, s2=L.s2, zp=L.zp,
        s1=L.s1, k=L.k, bias=bias, out=o_, w_s8=w_, act_codes=q_, rs=r_, max_abs_acc=np.int64(m_))
    put("fwd_a", seg=R.segmented_gemm(q_, r_, L))
    calib2 = R.gen_synthetic(64, 1024, 102, 3, 50.0, 8)
    k2, _ = R.smooth_from_calib(calib2, 0.005)
    L2 = oracle.random_layer(1024, 256, 128, seed=12, mode=0)
    L2.k = k2
    L2.act_scale = float(np.abs(calib2 / k2).max() / 127.0)
    Xf2 = R.gen_synthetic(32, 1024, 202, 3, 50.0, 8)
    o_, w_, q_, r_, m_ = R.dgq_forward(Xf2, L2, None, 1)
    put("fwd_b", X=Xf2, h=1024, o=256, g=128, mode=0, act_scale=np.float32(L2.act_scale), codes=L2.codes, s2=L2.s2,
        zp=L2.zp, s1=L2.s1, k=L2.k, out=o_, w_s8=w_, act_codes=q_, rs=r_, max_abs_acc=np.int64(m_))

    # ---- scalar primitives ---------------------------------------------------------
    pts = np.array([1.0, 65504.0, 0.1, 1e-30, 1e30, 65520.0, 65519.0, 2.0 ** -24, 2.0 ** -25, 1.5 * 2.0 ** -25,
                    3.0 * 2.0 ** -26, 2.0 ** -14, 6.1e-5, -0.333, -7.0e-8, 5.96e-8, 3e-8], np.float32)
    pts = np.concatenate([pts, rng.uniform(-100, 100, 64).astype(np.float32),
                          (rng.uniform(0, 1, 32) * 2.0 ** -23).astype(np.float32)])
    put("fp16", x=pts, y=np.array([R.fp16_round(float(v)) for v in pts], np.float32))
    lo = np.zeros((127, 16), np.int32)
    hi = np.zeros((127, 16), np.int32)
    for s in range(1, 128):
        for z in range(16):
            lo[s - 1, z], hi[s - 1, z] = R.clip_interval(s, z)
    put("clip", lo=lo, hi=hi)

    # ---- DGQ1 artifact --------------------------------------------------------------
    L3 = oracle.random_layer(64, 32, 16, seed=5, mode=0, act_scale=0.05)
    put("dgq1", bytes=np.frombuffer(R.dgq_to_bytes(L3), np.uint8), h=64, o=32, g=16, codes=L3.codes, s2=L3.s2,
        zp=L3.zp, s1=L3.s1, k=L3.k, act_scale=np.float32(0.05), mode=0)

    # DGQ1 artifacts through the reference's forward (the device-loaded layer must
    # reproduce w_s8 and the output), and corrupted artifacts with the
    # reference's validate_layer verdict (first failure in its loop order)
    X3 = R.gen_synthetic(9, 64, 44, 3, 50.0, 7)
    out3, w3, *_ = R.dgq_forward(X3, L3, None, 0)
    put("dgq1", w_s8=w3, X=X3, out=out3)
    L4 = oracle.random_layer(512, 384, 128, seed=8, mode=1)
    L4.k, _ = R.smooth_from_calib(R.gen_synthetic(64, 512, 9, 3, 50.0, 7), 0.005)
    X4 = R.gen_synthetic(33, 512, 45, 3, 50.0, 7)
    out4, w4, *_ = R.dgq_forward(X4, L4, None, 0)
    put("dgq1b", bytes=np.frombuffer(R.dgq_to_bytes(L4), np.uint8), w_s8=w4, X=X4, out=out4)

    def corrupt(name, L, edit):
        C = oracle.Layer(h=L.h, o=L.o, g=L.g, codes=L.codes.copy(), s2=L.s2.copy(), zp=L.zp.copy(),
                         s1=L.s1.copy(), k=L.k.copy(), act_scale=L.act_scale, mode=L.mode)
        edit(C)
        try:
            R.validate_layer(C)
            raise SystemExit(f"{name}: the reference accepted the corrupted layer")
        except oracle.OracleError as e:
            field, msg = e.field, str(e).split(": ", 1)[1]
        put(name, bytes=np.frombuffer(R.dgq_to_bytes_unchecked(C), np.uint8), field=np.array(field),
            msg=np.array(msg))

    def set_code(C, i, c, v):
        u = oracle.unpack_u4(C.codes, C.h * C.o)
        u[i * C.o + c] = v
        C.codes = oracle.pack_u4(u)

    def bad_codes(C):  # two violations: the reference reports the first in (group, column, row) order
        s2 = C.s2.reshape(-1, C.o)
        s2[2, 7] = s2[1, 300] = 127  # clip interval collapses to {ZP}
        zp = oracle.unpack_u4(C.zp, s2.size).reshape(s2.shape)
        set_code(C, 2 * 128 + 5, 7, (int(zp[2, 7]) + 3) % 16)
        set_code(C, 1 * 128 + 100, 300, (int(zp[1, 300]) + 5) % 16)

    def bad_s2_and_codes(C):
        bad_codes(C)
        C.s2[3 * C.o + 11] = 0

    def bad_s1_and_codes(C):
        bad_codes(C)
        C.s1[17] = -1.0

    corrupt("dgq1_badcodes", L4, bad_codes)
    corrupt("dgq1_bads2", L4, bad_s2_and_codes)
    corrupt("dgq1_bads1", L4, bad_s1_and_codes)

    path = os.path.join(HERE, "golden_v1.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()

"""Pin the CPU oracle: the C restatement (oracle/dgq_oracle.c) must equal the
reference itself (oracle/_ref) bit-for-bit, and both must reproduce the
committed golden vectors (generated from the reference by
tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

import oracle


def _layer(golden, p):
    return oracle.Layer(h=int(golden[f"{p}.h"]), o=int(golden[f"{p}.o"]), g=int(golden[f"{p}.g"]),
                        codes=golden[f"{p}.codes"], s2=golden[f"{p}.s2"], zp=golden[f"{p}.zp"],
                        s1=golden.get(f"{p}.s1", np.ones(int(golden[f"{p}.o"]), np.float32)),
                        k=golden.get(f"{p}.k", np.ones(int(golden[f"{p}.h"]), np.float32)),
                        act_scale=float(golden.get(f"{p}.act_scale", 0.0)), mode=int(golden.get(f"{p}.mode", 1)))


# ---------------------------------------------------------------- goldens
@pytest.mark.parametrize("case", ["actq_dyn", "actq_odd", "actq_edge"])
def test_port_actq_golden(port, golden, case):
    q, rs = port.quantize_activations(golden[f"{case}.X"], golden[f"{case}.k"], 1, 0.0)
    assert np.array_equal(q, golden[f"{case}.codes"])
    assert np.array_equal(rs.view(np.uint32), golden[f"{case}.rs"].view(np.uint32))


def test_port_actq_static_golden(port, golden):
    g = "actq_static"
    q, rs = port.quantize_activations(golden[f"{g}.X"], golden[f"{g}.k"], 0, float(golden[f"{g}.act_scale"]))
    assert np.array_equal(q, golden[f"{g}.codes"])
    assert (np.abs(q.astype(int)) == 127).any()  # the static scale saturates


def test_golden_edge_semantics(golden):
    # exact ties round half to even (proj/include/dgq/quant.hpp:24-30); zero row -> 1e-8f floor
    q = golden["actq_edge.codes"]
    assert list(q[0]) == [127, 0, 2, 2, 0, -2, -2, 126]
    assert golden["actq_edge.rs"][1] == np.float32(1e-8)
    assert not q[1].any()


@pytest.mark.parametrize("case", ["deq_g64", "deq_g128", "deq_g8", "deq_g12"])
def test_port_dequant_golden(port, golden, case):
    L = _layer(golden, case)
    assert np.array_equal(port.dequantize_to_s8(L), golden[f"{case}.w_s8"])


@pytest.mark.parametrize("case", ["gemm_16x64x8", "gemm_9x33x7", "gemm_40x300x130", "gemm_all127"])
def test_port_gemm_golden(port, golden, case):
    acc, mx = port.int8_gemm(golden[f"{case}.Xq"], golden[f"{case}.Wq"])
    assert np.array_equal(acc, golden[f"{case}.acc"])
    assert mx == int(golden[f"{case}.max_abs_acc"])


def test_golden_all127(golden):
    assert int(golden["gemm_all127.max_abs_acc"]) == 256 * 127 * 127
    assert golden["gemm_all127.acc"][0, 0] == 256 * 127 * 127


def test_port_epilogue_golden(port, golden):
    a, rs, s1, b = (golden[f"epi.{n}"] for n in ("acc", "rs", "s1", "bias"))
    for fp16, bias, key in [(False, None, "y"), (False, b, "y_bias"), (True, None, "y_f16mode"),
                            (True, b, "y_f16mode_bias")]:
        y = port.epilogue(a, rs, s1, bias, fp16)
        assert np.array_equal(y.view(np.uint32), golden[f"epi.{key}"].view(np.uint32)), key


@pytest.mark.parametrize("case", ["fwd_a", "fwd_b"])
def test_port_forward_golden(port, golden, case):
    L = _layer(golden, case)
    bias = golden.get(f"{case}.bias")
    out, w, q, rs, mx = port.dgq_forward(golden[f"{case}.X"], L, bias)
    assert np.array_equal(out.view(np.uint32), golden[f"{case}.out"].view(np.uint32))
    assert np.array_equal(w, golden[f"{case}.w_s8"])
    assert np.array_equal(q, golden[f"{case}.act_codes"])
    assert np.array_equal(rs, golden[f"{case}.rs"])
    assert mx == int(golden[f"{case}.max_abs_acc"])


def test_port_segmented_golden(port, golden):
    L = _layer(golden, "fwd_a")
    seg = port.segmented_gemm(golden["fwd_a.act_codes"], golden["fwd_a.rs"], L)
    assert np.array_equal(seg.view(np.uint32), golden["fwd_a.seg"].view(np.uint32))


def test_port_fp16_and_clip_golden(port, golden):
    y = port.fp16_round_array(golden["fp16.x"])
    assert np.array_equal(y.view(np.uint32), golden["fp16.y"].view(np.uint32))
    for s in range(1, 128):
        for z in range(16):
            assert port.clip_interval(s, z) == (golden["clip.lo"][s - 1, z], golden["clip.hi"][s - 1, z])


def test_clip_interval_kats(port):
    # proj/tests/test_search.cpp:40-64
    assert port.clip_interval(1, 0) == (0, 15)
    assert port.clip_interval(16, 0) == (0, 7)
    assert port.clip_interval(127, 8) == (7, 9)
    assert port.clip_interval(127, 0) == (0, 1)


def test_interval_fusion_sweep():
    # proj/tests/test_search.cpp:66-71: membership == |S2*(code-ZP)| <= 127
    s2 = np.arange(1, 128)[:, None, None]
    zp = np.arange(16)[None, :, None]
    code = np.arange(16)[None, None, :]
    lo, hi = oracle.clip_bounds(s2[:, :, 0], zp[:, :, 0])
    inside = (code >= lo[:, :, None]) & (code <= hi[:, :, None])
    assert np.array_equal(inside, np.abs(s2 * (code - zp)) <= 127)


# ------------------------------------------------------ port == reference
@pytest.mark.parametrize("seed,M,K,mode", [(1, 7, 96, 1), (2, 3, 1000, 1), (3, 4, 64, 0), (4, 1, 4096, 1)])
def test_port_equals_ref_actq(port, ref, seed, M, K, mode):
    X = ref.gen_synthetic(M, K, seed, 2, 30.0, 99)
    k = np.random.default_rng(seed).uniform(1, 4, K).astype(np.float32)
    act = float(np.abs(X / k).max() / 127.0 * 0.7)
    a = ref.quantize_activations(X, k, mode, act)
    b = port.quantize_activations(X, k, mode, act)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("h,o,g,seed", [(128, 64, 32, 1), (96, 12, 24, 2), (256, 130, 128, 3), (64, 8, 64, 4)])
def test_port_equals_ref_forward(port, ref, h, o, g, seed):
    L = oracle.random_layer(h, o, g, seed)
    ref.validate_layer(L)
    port.validate_layer(L)
    X = ref.gen_synthetic(9, h, seed + 10, 2, 20.0, 5)
    bias = np.linspace(-1, 1, o).astype(np.float32)
    a = ref.dgq_forward(X, L, bias, 2)
    b = port.dgq_forward(X, L, bias)
    for x, y in zip(a[:4], b[:4]):
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))
    assert a[4] == b[4]


def test_port_equals_ref_synthetic_and_smooth(port, ref):
    a = ref.gen_synthetic(33, 65, 123, 4, 50.0, 7)
    b = port.gen_synthetic(33, 65, 123, 4, 50.0, 7)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    ka, ta = ref.smooth_from_calib(a)
    kb, tb = port.smooth_from_calib(b)
    assert ta == tb and np.array_equal(ka.view(np.uint32), kb.view(np.uint32))


def test_port_equals_ref_fp16_exhaustive_sample(port, ref):
    # every exponent, a spread of mantissas, both signs
    bits = np.array([(s << 31) | (e << 23) | m for s in (0, 1) for e in range(0, 255, 3)
                     for m in (0, 1, 0x1000, 0x1FFF, 0x2000, 0x3000, 0x7FFFFF, 0x400000)], np.uint32)
    x = bits.view(np.float32)
    assert np.array_equal(port.fp16_round_array(x).view(np.uint32), ref.fp16_round_array(x).view(np.uint32))


@pytest.mark.parametrize("field,mutate", [
    ("s2", lambda L: L.s2.__setitem__(0, 0)),
    ("s1", lambda L: L.s1.__setitem__(1, -1.0)),
    ("k", lambda L: L.k.__setitem__(2, 0.5)),
    ("codes", lambda L: L.codes.__setitem__(0, 0xFF)),
])
def test_validation_fields_match_ref(port, ref, field, mutate):
    L = oracle.random_layer(64, 16, 16, 7, s2_range=(40, 127))
    mutate(L)
    with pytest.raises(oracle.OracleError) as e1:
        ref.validate_layer(L)
    with pytest.raises(oracle.OracleError) as e2:
        port.validate_layer(L)
    assert e1.value.field == field and e2.value.field == field


@pytest.mark.parametrize("h", [65, 7168])
def test_bench_smoothing_vector_is_the_references(port, ref, h):
    # bench.py's k (synth.smooth_k) = the reference's compute_smooth over the
    # channel maxima of its own synthetic calibration rows
    from paper_2310_04836_b200 import synth

    X = ref.gen_synthetic(256, h, 100, 3, 50.0, 7)
    k_ref, _ = ref.smooth_from_calib(X, 0.005)
    assert np.array_equal(synth.smooth_k(h).view(np.uint32), k_ref.view(np.uint32))
    if h == 7168:  # the K1 unit-k fast path covers most chunks
        assert (k_ref.reshape(-1, 8) == 1.0).all(axis=1).mean() > 0.9


def test_vectorised_fp16_round_equals_reference(port, golden):
    # oracle.fp16_round_np (used by the full-size GPU parity tests and bench.py's
    # self-check) against the scalar restatement on the golden points, every
    # exponent x a spread of mantissas (incl. the (2^-25, 2^-24) flush band) and
    # random finite values
    import oracle

    x = golden["fp16.x"]
    assert np.array_equal(oracle.fp16_round_np(x).view(np.uint32), golden["fp16.y"].view(np.uint32))
    bits = np.array([(s << 31) | (e << 23) | m for s in (0, 1) for e in range(0, 255)
                     for m in (0, 1, 0xFFF, 0x1000, 0x1001, 0x1FFF, 0x2000, 0x3000, 0x7FFFFF, 0x400000)], np.uint32)
    rnd = np.random.default_rng(5).integers(0, 0x7F800000, 20000, dtype=np.uint32)
    rnd |= (np.arange(rnd.size, dtype=np.uint32) & 1) << 31
    for b in (bits, rnd):
        x = b.view(np.float32)
        assert np.array_equal(oracle.fp16_round_np(x).view(np.uint32), port.fp16_round_array(x).view(np.uint32))

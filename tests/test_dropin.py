"""The C++ drop-in (paper_2310_04836_b200/dropin/dgq_kernel_b200.cpp) behind the
reference's unchanged operator API, and the host-buffer C ABI under it.

* The reference's OWN unit tests (proj/tests/test_kernel.cpp and
  test_format.cpp, compiled unmodified by tests/cpp/Makefile with our
  doctest-compatible shim) must pass against the reference kernel on the CPU
  (validates the shim build) and against the drop-in on the GPU.
* The host-buffer entry points (dgq_host_*) are checked against the golden
  vectors and the oracle bit-exactly.
"""
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
import paper_2310_04836_b200 as dgq

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")
BIN_CPU = os.path.join(CPP, "_build", "ref_tests_cpu")
BIN_B200 = os.path.join(CPP, "_build", "ref_tests_b200")


def _ensure_built(path):
    if not os.path.exists(path) and os.path.isdir("/root/reference/proj/tests"):
        subprocess.run(["make", "-C", CPP, "-j8"], check=True, capture_output=True)
    if not os.path.exists(path):
        pytest.skip(f"{os.path.basename(path)} not built (needs the reference sources at build time)")
    return path


def _run(path):
    r = subprocess.run([path], capture_output=True, text=True, timeout=600)
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed \| assertions: (\d+) \| (\d+) failed", r.stdout)
    assert m, r.stdout + r.stderr
    return r, [int(x) for x in m.groups()]


def test_reference_cpp_tests_pass_on_reference_kernel():
    r, (cases, passed, failed, asserts, afailed) = _run(_ensure_built(BIN_CPU))
    assert r.returncode == 0 and failed == 0 and afailed == 0, r.stderr[-4000:]
    assert cases >= 31 and asserts >= 400


def test_dropin_binary_links_our_hot_path():
    """The b200 test binary takes every kernel.hpp function and both dequantisers
    from the drop-in (which only calls the host C ABI), not from the reference."""
    path = _ensure_built(BIN_B200)
    drop = os.path.join(CPP, "_build", "dropin.o")
    nm = subprocess.run(["nm", "-C", drop], capture_output=True, text=True, check=True).stdout
    for fn in ("dgq::quantize_activations", "dgq::int8_gemm", "dgq::epilogue", "dgq::dgq_forward",
               "dgq::segmented_gemm_reference", "dgq::dequantize_to_s8", "dgq::dequantize_to_f32"):
        assert re.search(r" T " + re.escape(fn) + r"\(", nm), fn
    for sym in ("dgq_host_forward", "dgq_host_int8_gemm", "dgq_host_quantize_activations", "dgq_host_epilogue",
                "dgq_host_dequantize_to_s8", "dgq_host_segmented_gemm"):
        assert re.search(r" U " + sym + r"\b", nm), sym
    needed = subprocess.run(["readelf", "-d", path], capture_output=True, text=True, check=True).stdout
    assert "libdgq_b200.so" in needed
    # exactly one strong definition of the dequantiser: the drop-in's
    allsyms = subprocess.run(["nm", "-C", path], capture_output=True, text=True, check=True).stdout
    assert len(re.findall(r" T dgq::dequantize_to_s8\(", allsyms)) == 1


@pytest.mark.gpu
def test_reference_cpp_tests_pass_on_b200_dropin(cuda):
    r, (cases, passed, failed, asserts, afailed) = _run(_ensure_built(BIN_B200))
    assert r.returncode == 0 and failed == 0 and afailed == 0, r.stderr[-4000:]
    assert cases >= 31 and asserts >= 400


# ---------------------------------------------------------------- host ABI
def _golden_layer(golden, p) -> dgq.DgqLayer:
    o, h = int(golden[f"{p}.o"]), int(golden[f"{p}.h"])
    return dgq.DgqLayer(h=h, o=o, g=int(golden[f"{p}.g"]), codes=golden[f"{p}.codes"], s2=golden[f"{p}.s2"],
                        zp=golden[f"{p}.zp"], s1=golden.get(f"{p}.s1", np.ones(o, np.float32)),
                        k=golden.get(f"{p}.k", np.ones(h, np.float32)),
                        act_scale=float(golden.get(f"{p}.act_scale", 0.0)), mode=int(golden.get(f"{p}.mode", 1)))


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["fwd_a", "fwd_b"])
def test_host_forward_golden(cuda, golden, case):
    L = _golden_layer(golden, case)
    bias = golden.get(f"{case}.bias")
    r = dgq.host_forward(golden[f"{case}.X"], L, bias=bias)
    assert np.array_equal(_bits(r.out), _bits(golden[f"{case}.out"]))
    assert np.array_equal(r.w_s8, golden[f"{case}.w_s8"])
    assert np.array_equal(r.act.codes, golden[f"{case}.act_codes"])
    assert np.array_equal(_bits(r.act.row_scales), _bits(golden[f"{case}.rs"]))
    assert r.max_abs_acc == int(golden[f"{case}.max_abs_acc"])


@pytest.mark.gpu
def test_segmented_golden(cuda, golden):
    L = _golden_layer(golden, "fwd_a")
    act = dgq.ActQuant(golden["fwd_a.act_codes"], golden["fwd_a.rs"])
    y = dgq.segmented_gemm_reference(act, L)
    assert np.array_equal(_bits(y), _bits(golden["fwd_a.seg"]))


@pytest.mark.gpu
@pytest.mark.parametrize("h,o,g,M", [(256, 64, 64, 5), (384, 130, 128, 17), (33 * 8, 6, 8, 3), (1024, 256, 1024, 2)])
def test_segmented_matches_oracle(cuda, port, h, o, g, M):
    L = oracle.random_layer(h, o, g, seed=h + o + g)
    X = port.gen_synthetic(M, h, 5, 3, 50.0, 7)
    q, rs = port.quantize_activations(X, L.k)
    want = port.segmented_gemm(q, rs, L)
    D = dgq.DgqLayer(h=L.h, o=L.o, g=L.g, codes=L.codes, s2=L.s2, zp=L.zp, s1=L.s1, k=L.k,
                     act_scale=L.act_scale, mode=L.mode)
    got = dgq.segmented_gemm_reference(dgq.ActQuant(q, rs), D)
    assert np.array_equal(_bits(got), _bits(want))


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["deq_g64", "deq_g128", "deq_g8", "deq_g12"])
def test_dequantize_to_f32_matches_oracle(cuda, golden, case):
    L = _golden_layer(golden, case)
    L.s1 = np.linspace(1e-3, 2e-2, L.o).astype(np.float32)
    got = dgq.dequantize_to_f32(L)
    w = golden[f"{case}.w_s8"].astype(np.float64)
    want = (L.s1.astype(np.float64)[None, :] * w).astype(np.float32)  # format.cpp:150 in double
    assert np.array_equal(_bits(got), _bits(want))


@pytest.mark.gpu
def test_host_forward_corruption_raises_validation(cuda, golden):
    L = _golden_layer(golden, "fwd_a")
    codes = np.array(L.codes, np.uint8).copy()
    codes.ravel()[0] = (codes.ravel()[0] & 0xF0) | 0x0F  # a code far outside its clip interval for S2 > 8
    s2 = np.array(L.s2, np.int8).copy()
    s2.ravel()[0] = 127
    zp = np.array(L.zp, np.uint8).copy()
    zp.ravel()[0] &= 0xF0
    bad = dgq.DgqLayer(h=L.h, o=L.o, g=L.g, codes=codes, s2=s2, zp=zp, s1=L.s1, k=L.k, act_scale=L.act_scale,
                       mode=L.mode)
    with pytest.raises(dgq.ValidationError) as ei:
        dgq.host_forward(golden["fwd_a.X"], bad)
    assert ei.value.field == "codes"

"""CPU-side checks of the product library: it loads, exports every symbol the
C ABI header declares, and its host-only entry points (validation, clip
interval, fp16 rounding, DGQ1 parsing) agree with the oracle.  No GPU."""
import os
import re

import numpy as np
import pytest

import oracle
import paper_2310_04836_b200 as dgq
from paper_2310_04836_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "dgq_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dgq_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = dgq.lib()
    syms = _header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.exported_symbols())
    assert L.dgq_abi_version() == 1


def test_library_is_sm100a_only():
    data = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in data


def test_clip_interval_matches_oracle(golden):
    for s in range(1, 128):
        for z in range(16):
            assert dgq.clip_interval(s, z) == (golden["clip.lo"][s - 1, z], golden["clip.hi"][s - 1, z])
    with pytest.raises(dgq.InvalidArgument):
        dgq.clip_interval(0, 0)


def test_fp16_round_matches_oracle(golden):
    ys = np.array([dgq.fp16_round(float(x)) for x in golden["fp16.x"]], np.float32)
    assert np.array_equal(ys.view(np.uint32), golden["fp16.y"].view(np.uint32))


def test_fp16_round_flush_range(port):
    # the reference flushes (2^-25, 2^-24) to zero where IEEE rounds up
    x = np.float32(1.5 * 2.0 ** -25)
    assert dgq.fp16_round(float(x)) == 0.0 == port.fp16_round(float(x))


def _to_dgq(L: oracle.Layer) -> dgq.DgqLayer:
    return dgq.DgqLayer(h=L.h, o=L.o, g=L.g, codes=L.codes.copy(), s2=L.s2.copy(), zp=L.zp.copy(), s1=L.s1.copy(),
                        k=L.k.copy(), act_scale=L.act_scale, mode=L.mode)


def test_random_layer_generators_agree():
    a = oracle.random_layer(128, 64, 32, 9)
    b = dgq.random_layer(128, 64, 32, 9)
    for x, y in zip((a.codes, a.s2, a.zp, a.s1, a.k), b.arrays()):
        assert np.array_equal(np.asarray(x).ravel().view(np.uint8), np.asarray(y).ravel().view(np.uint8))


@pytest.mark.parametrize("field,mutate", [
    ("s2", lambda L: L.s2.__setitem__(0, 0)),
    ("s1", lambda L: L.s1.__setitem__(1, np.inf)),
    ("k", lambda L: L.k.__setitem__(2, 0.5)),
    ("codes", lambda L: L.codes.__setitem__(0, 0xFF)),
    ("act_scale", lambda L: setattr(L, "mode", 0) or setattr(L, "act_scale", 0.0)),
])
def test_validate_layer_fields(port, field, mutate):
    L = oracle.random_layer(64, 16, 16, 7, s2_range=(40, 127))
    mutate(L)
    with pytest.raises(oracle.OracleError) as eo:
        port.validate_layer(L)
    with pytest.raises(dgq.ValidationError) as ed:
        dgq.validate_layer(_to_dgq(L))
    assert ed.value.field == eo.value.field == field


def test_validate_layer_shape_errors():
    L = dgq.random_layer(64, 16, 16, 3)
    L.g = 24
    with pytest.raises(dgq.ValidationError) as e:
        dgq.validate_layer(L)
    assert e.value.field == "g"


def test_corrupted_code_8_at_s2_16_fails_validation():
    # proj/tests/test_format.cpp:160-177: code 8 with S2 = 16 would give 128
    codes = np.array([[0, 1], [2, 3], [4, 5], [6, 7]], np.uint8)
    L = dgq.DgqLayer(h=4, o=2, g=4, codes=dgq.pack_u4(codes), s2=np.array([[16, 16]], np.int8),
                     zp=dgq.pack_u4([0, 0]), s1=np.array([0.01, 0.01], np.float32), k=np.ones(4, np.float32),
                     act_scale=0.1, mode=1)
    dgq.validate_layer(L)
    codes[3, 1] = 8
    L.codes = dgq.pack_u4(codes)
    with pytest.raises(dgq.ValidationError) as e:
        dgq.validate_layer(L)
    assert e.value.field == "codes"


def test_dgq1_round_trip_matches_reference_bytes(golden):
    raw = golden["dgq1.bytes"].tobytes()
    L = dgq.layer_from_bytes(raw)
    assert (L.h, L.o, L.g, L.mode) == (64, 32, 16, 0)
    assert L.to_bytes() == raw
    assert np.array_equal(L.codes, golden["dgq1.codes"])


@pytest.mark.parametrize("mut,kind", [
    (lambda b: b[:20], "truncated"),
    (lambda b: b"XGQ1" + b[4:], "bad_magic"),
    (lambda b: b[:28] + bytes([7]) + b[29:], "bad_header"),
    (lambda b: b[:-1], "truncated"),
    (lambda b: b + b"\0", "size_mismatch"),
])
def test_dgq1_format_errors(golden, mut, kind):
    raw = golden["dgq1.bytes"].tobytes()
    with pytest.raises(dgq.FormatError) as e:
        dgq.layer_from_bytes(mut(raw))
    assert e.value.kind == kind


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        dgq.quantize_activations(np.zeros((1, 8), np.float32), dgq.random_layer(8, 2, 8, 1))


def _even_cost(b, KB, E):
    out = []
    for c in range(len(b) - 1):
        pos, segs = b[c], 0
        while pos < b[c + 1]:
            pos = min((pos // KB + 1) * KB, b[c + 1])
            segs += 1
        out.append(b[c + 1] - b[c] + E * segs)
    return out


@pytest.mark.parametrize("tiles,KB,ncl,E", [(336, 56, 74, 15), (112, 56, 74, 15), (448, 56, 74, 15),
                                            (112, 224, 74, 15), (84, 56, 74, 15), (56, 56, 74, 5),
                                            (7, 3, 5, 2), (1000, 8, 128, 15)])
def test_stream_k_balanced_split(tiles, KB, ncl, E):
    # the K5p launcher's stream-K ranges (csrc/prefill.cu sk_bounds): contiguous,
    # non-empty, covering every (tile, k-block) unit, and no pair costlier
    # (units + E x segments) than under the even split
    import ctypes as C

    L = dgq.lib()
    f = L.dgq_debug_sk_bounds
    f.argtypes = [C.c_longlong, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]
    U = tiles * KB
    b = (C.c_int * (ncl + 1))()
    used = f(U, KB, ncl, E, b)
    assert 1 <= used <= ncl  # the launch uses this many pairs
    b = list(b)[:used + 1]
    assert b[0] == 0 and b[-1] == U
    assert all(b[c] < b[c + 1] for c in range(used))
    even = [U * c // ncl for c in range(ncl + 1)]
    assert max(_even_cost(b, KB, E)) <= max(_even_cost(even, KB, E))
    assert f(U, KB, ncl, E, (C.c_int * (ncl + 1))()) == used  # cached

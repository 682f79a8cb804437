"""TEST INFRASTRUCTURE ONLY — CPU checkers for the DGQ A8W4 hot path.

Two interchangeable backends, both plain CPU code bound with ctypes:

* ``port()`` — ``oracle/_build/libdgq_oracle.so``: our C restatement of the
  reference algorithm (``oracle/dgq_oracle.c``; every function cites the
  reference file:line it follows).
* ``ref()``  — ``oracle/_ref/libdgq_ref.so``: the reference's own sources
  (``/root/reference/proj/src``) compiled unmodified by ``oracle/Makefile``
  behind the shim ``oracle/ref_capi.cpp``.

The port is pinned to the reference by ``tests/test_oracle.py`` (bit-exact on
random cases) and by the committed golden vectors in ``tests/golden``.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libdgq_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdgq_ref.so")

_vp = C.c_void_p
_sz = C.c_size_t


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = "", field: str = ""):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code
        self.field = field


def _p(a):
    return None if a is None else a.ctypes.data_as(_vp)


@dataclass
class Layer:
    """Host DgqLayer in the reference's storage layout
    (proj/include/dgq/format.hpp:36-49): codes u4 packed [h x o] along o,
    s2 int8 [h/g x o], zp u4 packed [h/g x o], s1 f32[o], k f32[h]."""

    h: int
    o: int
    g: int
    codes: np.ndarray  # uint8, h*o/2
    s2: np.ndarray  # int8, (h/g)*o
    zp: np.ndarray  # uint8, (h/g)*o/2
    s1: np.ndarray  # float32, o
    k: np.ndarray  # float32, h
    act_scale: float = 0.0
    mode: int = 1  # 1 dynamic, 0 static

    @property
    def n_g(self) -> int:
        return self.h // self.g


class _Backend:
    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.lib = C.CDLL(path)
        self.pfx = prefix
        self.kind = "reference" if prefix == "ref_" else "port"
        L = self.lib
        f = self._f
        f("fp16_round").restype = C.c_float
        f("fp16_round").argtypes = [C.c_float]
        f("clip_interval").argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        f("gen_synthetic").argtypes = [_sz, _sz, C.c_uint64, _sz, C.c_float, C.c_int, C.c_uint64, _vp]
        f("smooth_from_calib").argtypes = [_vp, _sz, _sz, C.c_float, _vp, _vp]
        f("quantize_activations").argtypes = [_vp, _sz, _sz, _vp, C.c_int, C.c_float, _vp, _vp]
        f("dequantize_to_s8").argtypes = [_sz, _sz, _sz, _vp, _vp, _vp, _vp]
        f("epilogue").argtypes = [_vp, _sz, _sz, _vp, _vp, _vp, C.c_int, _vp]
        f("segmented_gemm").argtypes = [_vp, _vp, _sz, _sz, _sz, _sz, _vp, _vp, _vp, _vp, _vp]
        if prefix == "ref_":
            L.ref_last_error.restype = C.c_char_p
            L.ref_last_field.restype = C.c_char_p
            f("int8_gemm").argtypes = [_vp, _vp, _sz, _sz, _sz, C.c_int, _vp, _vp]
            f("validate_layer").argtypes = [_sz, _sz, _sz, C.c_int, C.c_float] + [_vp] * 5
            f("dgq_forward").argtypes = ([_vp, _sz, _sz, _sz, _sz, C.c_int, C.c_float] + [_vp] * 6
                                         + [C.c_int] + [_vp] * 5)
            f("dgq_to_bytes").argtypes = [_sz, _sz, _sz, C.c_int, C.c_float] + [_vp] * 7
            f("phase1_search").argtypes = ([_vp, _sz, _sz, _vp, _vp, _sz, _sz, C.c_int, _vp, _sz, C.c_int]
                                           + [_vp] * 5)
            f("phase2_search").argtypes = ([_vp, _sz, _sz, _vp, _vp, _sz, _sz, C.c_int, _vp, _vp, _vp, _sz,
                                            C.c_int] + [_vp] * 6)
        else:
            f("int8_gemm").argtypes = [_vp, _vp, _sz, _sz, _sz, _vp, _vp]
            f("validate_layer").argtypes = ([_sz, _sz, _sz, C.c_int, C.c_float] + [_vp] * 5
                                            + [C.POINTER(C.c_char_p)])
            f("dgq_forward").argtypes = ([_vp, _sz, _sz, _sz, _sz, C.c_int, C.c_float] + [_vp] * 6
                                         + [_vp] * 5)

    def _f(self, name):
        return getattr(self.lib, self.pfx + name)

    def _check(self, st, field=""):
        if st == 0:
            return
        if self.pfx == "ref_":
            raise OracleError(st, self.lib.ref_last_error().decode(), self.lib.ref_last_field().decode())
        raise OracleError(st, "", field)

    # ---- primitives ----
    def fp16_round(self, x: float) -> float:
        return self._f("fp16_round")(C.c_float(x))

    def fp16_round_array(self, a: np.ndarray) -> np.ndarray:
        f = self._f("fp16_round")
        return np.array([f(C.c_float(float(v))) for v in np.asarray(a, np.float32).ravel()],
                        np.float32).reshape(np.shape(a))

    def clip_interval(self, s2: int, zp: int):
        lo, hi = C.c_int(), C.c_int()
        self._check(self._f("clip_interval")(s2, zp, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def gen_synthetic(self, rows, cols, seed, count=0, magnitude=1.0, column_seed=None):
        out = np.empty(rows * cols, np.float32)
        st = self._f("gen_synthetic")(rows, cols, seed, count, magnitude,
                                      int(column_seed is not None), column_seed or 0, _p(out))
        self._check(st)
        return out.reshape(rows, cols)

    def smooth_from_calib(self, X: np.ndarray, percentile: float = 0.005):
        X = np.ascontiguousarray(X, np.float32)
        k = np.empty(X.shape[1], np.float32)
        th = np.zeros(1, np.float32)
        self._check(self._f("smooth_from_calib")(_p(X), X.shape[0], X.shape[1], percentile, _p(k), _p(th)))
        return k, float(th[0])

    def validate_layer(self, L: Layer):
        args = [L.h, L.o, L.g, L.mode, C.c_float(L.act_scale), _p(L.codes), _p(L.s2), _p(L.zp),
                _p(L.s1), _p(L.k)]
        if self.pfx == "ref_":
            self._check(self._f("validate_layer")(*args))
        else:
            fld = C.c_char_p()
            st = self._f("validate_layer")(*args, C.byref(fld))
            self._check(st, fld.value.decode() if fld.value else "")

    # ---- hot path ----
    def quantize_activations(self, X, k, mode=1, act_scale=0.0):
        X = np.ascontiguousarray(X, np.float32)
        M, K = X.shape
        q = np.empty((M, K), np.int8)
        rs = np.empty(M, np.float32)
        k = np.ascontiguousarray(k, np.float32)
        self._check(self._f("quantize_activations")(_p(X), M, K, _p(k), mode, C.c_float(act_scale), _p(q), _p(rs)))
        return q, rs

    def dequantize_to_s8(self, L: Layer):
        w = np.empty((L.h, L.o), np.int8)
        self._check(self._f("dequantize_to_s8")(L.h, L.o, L.g, _p(L.codes), _p(L.s2), _p(L.zp), _p(w)))
        return w

    def int8_gemm(self, Xq, Wq, threads=0):
        Xq = np.ascontiguousarray(Xq, np.int8)
        Wq = np.ascontiguousarray(Wq, np.int8)
        M, K = Xq.shape
        K2, N = Wq.shape
        assert K == K2
        acc = np.empty((M, N), np.int32)
        mx = np.zeros(1, np.int64)
        if self.pfx == "ref_":
            st = self._f("int8_gemm")(_p(Xq), _p(Wq), M, K, N, threads, _p(acc), _p(mx))
        else:
            st = self._f("int8_gemm")(_p(Xq), _p(Wq), M, K, N, _p(acc), _p(mx))
        self._check(st)
        return acc, int(mx[0])

    def epilogue(self, acc, rs, s1, bias=None, fp16_mode=False):
        acc = np.ascontiguousarray(acc, np.int32)
        M, N = acc.shape
        rs = np.ascontiguousarray(rs, np.float32)
        s1 = np.ascontiguousarray(s1, np.float32)
        b = None if bias is None else np.ascontiguousarray(bias, np.float32)
        y = np.empty((M, N), np.float32)
        self._check(self._f("epilogue")(_p(acc), M, N, _p(rs), _p(s1), _p(b), int(fp16_mode), _p(y)))
        return y

    def segmented_gemm(self, Xq, rs, L: Layer):
        Xq = np.ascontiguousarray(Xq, np.int8)
        rs = np.ascontiguousarray(rs, np.float32)
        y = np.empty((Xq.shape[0], L.o), np.float32)
        self._check(self._f("segmented_gemm")(_p(Xq), _p(rs), Xq.shape[0], L.h, L.o, L.g, _p(L.codes),
                                              _p(L.s2), _p(L.zp), _p(L.s1), _p(y)))
        return y

    def dgq_forward(self, X, L: Layer, bias=None, threads=0):
        """Returns (out f32 [M,o], w_s8 [h,o], codes [M,h], row_scales [M], max_abs_acc)."""
        X = np.ascontiguousarray(X, np.float32)
        M = X.shape[0]
        out = np.empty((M, L.o), np.float32)
        w = np.empty((L.h, L.o), np.int8)
        q = np.empty((M, L.h), np.int8)
        rs = np.empty(M, np.float32)
        mx = np.zeros(1, np.int64)
        b = None if bias is None else np.ascontiguousarray(bias, np.float32)
        head = [_p(X), M, L.h, L.o, L.g, L.mode, C.c_float(L.act_scale), _p(L.codes), _p(L.s2),
                _p(L.zp), _p(L.s1), _p(L.k), _p(b)]
        tail = [_p(out), _p(w), _p(q), _p(rs), _p(mx)]
        if self.pfx == "ref_":
            st = self._f("dgq_forward")(*head, threads, *tail)
        else:
            st = self._f("dgq_forward")(*head, *tail)
        self._check(st)
        return out, w, q, rs, int(mx[0])

    # ---- offline quantiser (reference only): search.cpp:83-163, 252-326 ----
    def phase1_search(self, W, X, Xhat, g, grid, n_bits=4, threads=0):
        """Returns (s_prime f32 [n_g,o], zp i32, err f32, alpha f32, evals)."""
        assert self.pfx == "ref_"
        W, X, Xhat = (np.ascontiguousarray(a, np.float32) for a in (W, X, Xhat))
        grid = np.ascontiguousarray(grid, np.float32)
        h, o = W.shape
        ng = h // g
        sp, er, al = (np.empty((ng, o), np.float32) for _ in range(3))
        zp = np.empty((ng, o), np.int32)
        ev = np.zeros(1, np.uint64)
        self._check(self._f("phase1_search")(_p(W), h, o, _p(X), _p(Xhat), X.shape[0], g, n_bits, _p(grid),
                                             grid.size, threads, _p(sp), _p(zp), _p(er), _p(al), _p(ev)))
        return sp, zp, er, al, int(ev[0])

    def phase2_search(self, W, X, Xhat, g, s_prime, zp, grid, n_bits=4, threads=0):
        """Returns (s1 f32 [o], s2 i8 [n_g,o], codes i32 [h,o], col_err f64 [o], col_alpha f32 [o], evals)."""
        assert self.pfx == "ref_"
        W, X, Xhat = (np.ascontiguousarray(a, np.float32) for a in (W, X, Xhat))
        s_prime = np.ascontiguousarray(s_prime, np.float32)
        zp = np.ascontiguousarray(zp, np.int32)
        grid = np.ascontiguousarray(grid, np.float32)
        h, o = W.shape
        ng = h // g
        s1, ca = np.empty(o, np.float32), np.empty(o, np.float32)
        s2 = np.empty((ng, o), np.int8)
        codes = np.empty((h, o), np.int32)
        ce = np.empty(o, np.float64)
        ev = np.zeros(1, np.uint64)
        self._check(self._f("phase2_search")(_p(W), h, o, _p(X), _p(Xhat), X.shape[0], g, n_bits, _p(s_prime),
                                             _p(zp), _p(grid), grid.size, threads, _p(s1), _p(s2), _p(codes),
                                             _p(ce), _p(ca), _p(ev)))
        return s1, s2, codes, ce, ca, int(ev[0])

    @staticmethod
    def dgq_to_bytes_unchecked(L: Layer) -> bytes:
        """DGQ1 serialisation (proj/include/dgq/format.hpp:6-21) WITHOUT the
        reference's validation — for corrupted-artifact fixtures."""
        import struct

        head = b"DGQ1" + struct.pack("<QQQB", L.h, L.o, L.g, L.mode)
        return (head + np.ascontiguousarray(L.codes, np.uint8).tobytes() + np.ascontiguousarray(L.s2, np.int8).tobytes()
                + np.ascontiguousarray(L.zp, np.uint8).tobytes() + np.ascontiguousarray(L.s1, "<f4").tobytes()
                + np.ascontiguousarray(L.k, "<f4").tobytes() + np.float32(L.act_scale).astype("<f4").tobytes())

    def dgq_to_bytes(self, L: Layer) -> bytes:
        assert self.pfx == "ref_"
        n = C.c_size_t()
        args = [L.h, L.o, L.g, L.mode, C.c_float(L.act_scale), _p(L.codes), _p(L.s2), _p(L.zp),
                _p(L.s1), _p(L.k)]
        self._check(self._f("dgq_to_bytes")(*args, None, C.byref(n)))
        buf = np.empty(n.value, np.uint8)
        self._check(self._f("dgq_to_bytes")(*args, _p(buf), C.byref(n)))
        return buf.tobytes()


_cache: dict = {}


def port() -> _Backend:
    if "port" not in _cache:
        _cache["port"] = _Backend(PORT_SO, "orc_")
    return _cache["port"]


def ref() -> _Backend:
    if "ref" not in _cache:
        _cache["ref"] = _Backend(REF_SO, "ref_")
    return _cache["ref"]


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def best() -> _Backend:
    """The reference itself when it was built, else the pinned port."""
    return ref() if have_ref() else port()


# ---------------------------------------------------------------------------
# Deterministic layer/input generation (SURVEY.md §8d "flavour A"): SplitMix64
# driven, so fixtures are identical on every platform (std::uniform_* is not).
# ---------------------------------------------------------------------------

class SplitMix64:
    """proj/include/dgq/tensor.hpp:101-118 — vectorised in numpy."""

    def __init__(self, seed: int):
        self.state = np.uint64(seed)

    def next(self, n: int) -> np.ndarray:
        with np.errstate(over="ignore"):
            inc = np.uint64(0x9E3779B97F4A7C15)
            steps = (np.arange(1, n + 1, dtype=np.uint64) * inc) + self.state
            self.state = steps[-1] if n else self.state
            z = steps
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            return z ^ (z >> np.uint64(31))

    def ints(self, n: int, lo: int, hi: int) -> np.ndarray:
        """n integers uniform in [lo, hi] (hi inclusive), by modulo."""
        span = np.uint64(hi - lo + 1)
        return (self.next(n) % span).astype(np.int64) + lo

    def units(self, n: int) -> np.ndarray:
        return ((self.next(n) >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53


def pack_u4(vals: np.ndarray) -> np.ndarray:
    """Even index in the low nibble (proj/src/tensor.cpp:124-132)."""
    v = np.asarray(vals, np.uint8).ravel()
    assert v.size % 2 == 0
    return (v[0::2] | (v[1::2] << 4)).astype(np.uint8)


def unpack_u4(packed: np.ndarray, count: int) -> np.ndarray:
    p = np.asarray(packed, np.uint8).ravel()
    out = np.empty(p.size * 2, np.uint8)
    out[0::2] = p & 0x0F
    out[1::2] = p >> 4
    return out[:count]


def fp16_round_np(x) -> np.ndarray:
    """Vectorised fp16_round (proj/src/quant.cpp:9-58): IEEE binary16
    round-to-nearest-even, except that |x| in [2^-25, 2^-24) flushes to a signed
    zero (the reference's `exp >= -24` subnormal branch starts at 2^-24; RNE
    would round (2^-25, 2^-24) up to 2^-24).  Pinned against the scalar
    reference by tests/test_oracle.py."""
    x = np.asarray(x, np.float32)
    y = x.astype(np.float16).astype(np.float32)
    a = np.abs(x)
    band = (a >= np.float32(2.0 ** -25)) & (a < np.float32(2.0 ** -24))
    return np.where(band, np.copysign(np.float32(0.0), x), y).astype(np.float32)


def clip_bounds(s2: np.ndarray, zp: np.ndarray):
    """Vectorised clip_interval (proj/src/search.cpp:190-201), C truncation."""
    s2 = s2.astype(np.int64)
    zp = zp.astype(np.int64)
    q = 127 // s2  # positive operands: floor == trunc
    lo = np.maximum(0, zp - q)
    hi = np.minimum(15, zp + q)
    return lo, hi


def random_layer(h: int, o: int, g: int, seed: int, mode: int = 1, act_scale: float = 0.02,
                 s2_range=(1, 127), s1_range=(1e-3, 2e-2), k_range=(1.0, 3.0)) -> Layer:
    """A valid random DgqLayer: S2 uniform in s2_range, ZP in [0,15], codes
    uniform inside clip_interval(S2, ZP), s1/k uniform (mirrors
    proj/tests/test_kernel.cpp:31-59 with a portable generator)."""
    rng = SplitMix64(seed)
    ng = h // g
    s2 = rng.ints(ng * o, *s2_range).astype(np.int8).reshape(ng, o)
    zp = rng.ints(ng * o, 0, 15).astype(np.uint8).reshape(ng, o)
    lo, hi = clip_bounds(s2, zp)
    lo_f = np.repeat(lo, g, axis=0)
    hi_f = np.repeat(hi, g, axis=0)
    span = (hi_f - lo_f + 1).astype(np.uint64)
    codes = (rng.next(h * o).reshape(h, o) % span).astype(np.int64) + lo_f
    u = rng.units(o)
    s1 = (s1_range[0] + (s1_range[1] - s1_range[0]) * u).astype(np.float32)
    u = rng.units(h)
    k = (k_range[0] + (k_range[1] - k_range[0]) * u).astype(np.float32)
    return Layer(h=h, o=o, g=g, codes=pack_u4(codes.astype(np.uint8)), s2=s2.ravel().copy(),
                 zp=pack_u4(zp), s1=s1, k=k, act_scale=float(act_scale), mode=mode)

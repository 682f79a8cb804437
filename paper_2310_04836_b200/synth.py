"""Deterministic synthetic inputs shaped like the reference's (numpy only).

* `gen_synthetic` — the reference's generator (proj/src/tensor.cpp:222-257):
  SplitMix64 uniforms -> Box-Muller normals, `count` outlier columns scaled by
  `magnitude`.  Vectorised; numpy's transcendental functions may differ from
  libm in the last ulp, so this is distributionally — not bitwise — the
  reference stream (tests take bitwise inputs from the oracle instead).
* `random_layer` — a valid random DgqLayer (SURVEY.md §8d "flavour A"):
  S2 in [1,127], ZP in [0,15], codes uniform inside clip_interval(S2, ZP).
"""
from __future__ import annotations

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)


class SplitMix64:
    """proj/include/dgq/tensor.hpp:101-118, vectorised: draw n values at once."""

    def __init__(self, seed: int):
        self.state = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)

    def next(self, n: int) -> np.ndarray:
        with np.errstate(over="ignore"):
            z = np.arange(1, n + 1, dtype=np.uint64) * _GAMMA + self.state
            if n:
                self.state = z[-1]
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            return z ^ (z >> np.uint64(31))

    def units(self, n: int) -> np.ndarray:
        return ((self.next(n) >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53

    def ints(self, n: int, lo: int, hi: int) -> np.ndarray:
        return (self.next(n) % np.uint64(hi - lo + 1)).astype(np.int64) + lo


def outlier_columns(cols: int, column_seed: int, count: int) -> np.ndarray:
    rng = SplitMix64(column_seed ^ 0xD1B54A32D192ED03)
    idx = np.arange(cols)
    for i in range(count):
        j = i + int(rng.next(1)[0] % np.uint64(cols - i))
        idx[i], idx[j] = idx[j], idx[i]
    return np.sort(idx[:count])


def gen_synthetic(rows: int, cols: int, seed: int, count: int = 0, magnitude: float = 1.0,
                  column_seed: int | None = None) -> np.ndarray:
    n = rows * cols
    u = SplitMix64(seed).units(n + (n & 1))
    u1, u2 = u[0::2], u[1::2]
    r = np.sqrt(-2.0 * np.log(u1))
    t = 2.0 * np.pi * u2
    v = np.empty(u.size, np.float32)
    v[0::2] = (r * np.cos(t)).astype(np.float32)
    v[1::2] = (r * np.sin(t)).astype(np.float32)
    v = v[:n].reshape(rows, cols)
    if count:
        oc = outlier_columns(cols, seed if column_seed is None else column_seed, count)
        v[:, oc] *= np.float32(magnitude)
    return v


def channel_maxima(calib) -> np.ndarray:
    """max |x| per channel over a calibration set (proj/src/smoothing.cpp:9-24)."""
    z = None
    for t in calib:
        m = np.max(np.abs(np.asarray(t, np.float32)), axis=0)
        z = m if z is None else np.maximum(z, m)
    return z.astype(np.float32)


def compute_smooth(z, percentile: float) -> np.ndarray:
    """k = max(1, z / threshold), threshold = the ceil(percentile * h)-th largest
    channel maximum (proj/src/smoothing.cpp:26-49): k is exactly 1 on all but
    the top `percentile` of the channels."""
    z = np.asarray(z, np.float32)
    rank = max(int(np.ceil(np.float64(np.float32(percentile)) * z.size)), 1)
    thr = np.sort(z)[::-1][rank - 1]
    if not thr > 0:
        raise ValueError("smoothing undefined: percentile threshold is not positive")
    return np.maximum(np.float32(1.0), (z / thr).astype(np.float32)).astype(np.float32)


def smooth_k(h: int, seed: int = 100, percentile: float = 0.005) -> np.ndarray:
    """The smoothing vector of SURVEY.md §8d: compute_smooth over the channel
    maxima of 256 synthetic calibration rows with the standard outlier spec
    (3 channels x 50, column seed 7; proj/manifests/standard_suite.json:7)."""
    return compute_smooth(channel_maxima([gen_synthetic(256, h, seed, 3, 50.0, 7)]), percentile)


def pack_u4(vals) -> np.ndarray:
    """Nibble packing, even index in the LOW nibble (proj/src/tensor.cpp:124-132)."""
    v = np.asarray(vals, np.uint8).ravel()
    if v.size % 2:
        raise ValueError("packed 4-bit tensors need an even element count")
    return (v[0::2] | (v[1::2] << 4)).astype(np.uint8)


def unpack_u4(packed, count: int) -> np.ndarray:
    p = np.asarray(packed, np.uint8).ravel()
    out = np.empty(p.size * 2, np.uint8)
    out[0::2] = p & 0x0F
    out[1::2] = p >> 4
    return out[:count]


def random_layer(h: int, o: int, g: int, seed: int, mode: int = 1, act_scale: float = 0.02,
                 s2_range=(1, 127), s1_range=(1e-3, 2e-2), k_range=(1.0, 3.0)):
    from .api import DgqLayer

    rng = SplitMix64(seed)
    ng = h // g
    s2 = rng.ints(ng * o, *s2_range).astype(np.int8).reshape(ng, o)
    zp = rng.ints(ng * o, 0, 15).astype(np.uint8).reshape(ng, o)
    q = 127 // s2.astype(np.int64)
    lo = np.maximum(0, zp.astype(np.int64) - q)
    hi = np.minimum(15, zp.astype(np.int64) + q)
    lo_f, hi_f = np.repeat(lo, g, axis=0), np.repeat(hi, g, axis=0)
    span = (hi_f - lo_f + 1).astype(np.uint64)
    codes = (rng.next(h * o).reshape(h, o) % span).astype(np.int64) + lo_f
    s1 = (s1_range[0] + (s1_range[1] - s1_range[0]) * rng.units(o)).astype(np.float32)
    k = (k_range[0] + (k_range[1] - k_range[0]) * rng.units(h)).astype(np.float32)
    return DgqLayer(h=h, o=o, g=g, codes=pack_u4(codes.astype(np.uint8)), s2=s2, zp=pack_u4(zp), s1=s1, k=k,
                    act_scale=float(act_scale), mode=mode)

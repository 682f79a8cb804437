"""Python mirror of the reference's operator API for the DGQ hot path.

Same names, argument meaning and error behaviour as proj/include/dgq/kernel.hpp
and proj/include/dgq/format.hpp, so parity tests read like the reference's own
(proj/tests/test_kernel.cpp, proj/tests/test_format.cpp).  Every numeric result
is produced by libdgq_b200.so on the GPU; host (numpy) inputs are uploaded and
results downloaded, exactly the reference's by-value host semantics.  The
device-resident fast path is `CudaLayer` (the C ABI's prepared layer).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import (MODE_DYNAMIC, MODE_STATIC, OUT_F16, OUT_F32, FormatError, InvalidArgument,  # noqa: F401
                   OverflowRuntimeError, ValidationError, check, lib)


def _np_ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _t_ptr(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(device=None) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _device_index(device) -> int:
    if device is None:
        return torch.cuda.current_device()
    return torch.device(device).index if torch.device(device).index is not None else torch.cuda.current_device()


@dataclass
class DgqLayer:
    """proj/include/dgq/format.hpp:36-49 (reference storage layout, host)."""

    h: int
    o: int
    g: int
    codes: np.ndarray            # uint8, packed u4 [h x o] along o (even column = low nibble)
    s2: np.ndarray               # int8 [h/g x o], values in [1, 127]
    zp: np.ndarray               # uint8, packed u4 [h/g x o]
    s1: np.ndarray               # float32 [o], > 0
    k: np.ndarray                # float32 [h], >= 1
    act_scale: float = 0.0
    mode: int = MODE_DYNAMIC     # ActMode: 0 static, 1 dynamic

    @property
    def n_g(self) -> int:
        return 0 if self.g == 0 else self.h // self.g

    def arrays(self):
        return (np.ascontiguousarray(self.codes, np.uint8).ravel(), np.ascontiguousarray(self.s2, np.int8).ravel(),
                np.ascontiguousarray(self.zp, np.uint8).ravel(), np.ascontiguousarray(self.s1, np.float32).ravel(),
                np.ascontiguousarray(self.k, np.float32).ravel())

    # DGQ1 serialisation (proj/include/dgq/format.hpp:6-21)
    def to_bytes(self) -> bytes:
        validate_layer(self)
        codes, s2, zp, s1, k = self.arrays()
        head = b"DGQ1" + int(self.h).to_bytes(8, "little") + int(self.o).to_bytes(8, "little") + \
            int(self.g).to_bytes(8, "little") + bytes([int(self.mode)])
        return head + codes.tobytes() + s2.tobytes() + zp.tobytes() + s1.tobytes() + k.tobytes() + \
            np.float32(self.act_scale).tobytes()


def _check_layer_arrays(layer: DgqLayer):
    """The array-shape part of validate_layer (proj/src/format.cpp:31-42)."""
    codes, s2, zp, s1, k = layer.arrays()
    ng = layer.n_g
    if (layer.h and layer.o and layer.g and layer.o % 2 == 0 and layer.h % layer.g == 0 and
            (codes.size != layer.h * layer.o // 2 or s2.size != ng * layer.o or zp.size != ng * layer.o // 2)):
        field_ = "codes" if codes.size != layer.h * layer.o // 2 else ("s2" if s2.size != ng * layer.o else "zp")
        raise ValidationError(_lib.DGQ_EVALIDATION, f"invalid DgqLayer field '{field_}': wrong shape", field_)
    if s1.size != layer.o and layer.o:
        raise ValidationError(_lib.DGQ_EVALIDATION, "invalid DgqLayer field 's1': expected length o", "s1")
    if k.size != layer.h and layer.h:
        raise ValidationError(_lib.DGQ_EVALIDATION, "invalid DgqLayer field 'k': expected length h", "k")
    return codes, s2, zp, s1, k


def validate_layer(layer: DgqLayer) -> None:
    """proj/src/format.cpp:24-75; raises ValidationError(field).  (Host C-ABI
    dgq_validate_layer; CudaLayer validates the same invariants on the GPU.)"""
    codes, s2, zp, s1, k = _check_layer_arrays(layer)
    check(lib().dgq_validate_layer(layer.h, layer.o, layer.g, int(layer.mode), float(layer.act_scale),
                                   _np_ptr(codes), _np_ptr(s2), _np_ptr(zp), _np_ptr(s1), _np_ptr(k)))


def clip_interval(s2: int, zp: int):
    """proj/src/search.cpp:190-201."""
    lo, hi = C.c_int(), C.c_int()
    check(lib().dgq_clip_interval(int(s2), int(zp), C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def fp16_round(x: float) -> float:
    """proj/src/quant.cpp:9-58."""
    return lib().dgq_fp16_round(float(x))


def layer_from_bytes(data: bytes) -> DgqLayer:
    """Host-side DGQ1 parse with the reference's format_error kinds
    (proj/src/format.cpp:214-266)."""
    if len(data) < 29:
        raise FormatError(_lib.DGQ_EFORMAT, "DGQ file shorter than the header", "truncated")
    if data[:4] != b"DGQ1":
        raise FormatError(_lib.DGQ_EFORMAT, 'bad magic, expected "DGQ1"', "bad_magic")
    h, o, g = (int.from_bytes(data[i:i + 8], "little") for i in (4, 12, 20))
    mode = data[28]
    if mode > 1:
        raise FormatError(_lib.DGQ_EFORMAT, f"unknown mode byte {mode}", "bad_header")
    if h == 0 or o == 0 or o % 2 or g == 0 or h % g:
        raise FormatError(_lib.DGQ_EFORMAT, "inconsistent dimensions in header", "bad_header")
    ng = h // g
    need = 29 + h * o // 2 + ng * o + ng * o // 2 + 4 * o + 4 * h + 4
    if len(data) < need:
        raise FormatError(_lib.DGQ_EFORMAT, "truncated payload", "truncated")
    if len(data) > need:
        raise FormatError(_lib.DGQ_EFORMAT, "payload longer than the header implies", "size_mismatch")
    buf = np.frombuffer(data, np.uint8, offset=29)
    p = 0

    def take(n):
        nonlocal p
        r = buf[p:p + n]
        p += n
        return r

    codes = take(h * o // 2).copy()
    s2 = take(ng * o).view(np.int8).reshape(ng, o).copy()
    zp = take(ng * o // 2).copy()
    s1 = take(4 * o).view(np.float32).copy()
    k = take(4 * h).view(np.float32).copy()
    act = float(take(4).view(np.float32)[0])
    L = DgqLayer(h=h, o=o, g=g, codes=codes, s2=s2, zp=zp, s1=s1, k=k, act_scale=act, mode=mode)
    validate_layer(L)
    return L


class CudaLayer:
    """A validated DgqLayer resident on one GPU in the B200 tile layout
    (optionally the column shard [col_begin, col_end)).  Wraps dgq_layer*."""

    def __init__(self, layer: DgqLayer | None = None, device=None, col_begin: int = 0, col_end: int | None = None,
                 validate: bool = True, *, _handle=None):
        self.device = _device_index(device)
        self._h = C.c_void_p()
        if _handle is not None:
            self._h = _handle
        else:
            # array shapes here; the value invariants are checked on the GPU by dgq_layer_create
            codes, s2, zp, s1, k = _check_layer_arrays(layer)
            with torch.cuda.device(self.device):
                check(lib().dgq_layer_create(self.device, layer.h, layer.o, layer.g, int(layer.mode),
                                             float(layer.act_scale), _np_ptr(codes), _np_ptr(s2), _np_ptr(zp),
                                             _np_ptr(s1), _np_ptr(k), int(col_begin), int(col_end or 0),
                                             int(validate), _stream(self.device), C.byref(self._h)))
        info = _lib.LayerInfo()
        check(lib().dgq_layer_get_info(self._h, C.byref(info)))
        self.info = info
        self.h, self.o, self.k_pad = info.h, info.o, info.k_pad
        self.mode, self.act_scale, self.fused = info.mode, info.act_scale, bool(info.fused)

    @classmethod
    def from_dgq1(cls, data: bytes, device=None, col_begin: int = 0, col_end: int | None = None) -> "CudaLayer":
        dev = _device_index(device)
        h = C.c_void_p()
        buf = np.frombuffer(data, np.uint8)
        with torch.cuda.device(dev):
            check(lib().dgq_layer_create_from_dgq1(dev, _np_ptr(buf), buf.size, int(col_begin), int(col_end or 0),
                                                   _stream(dev), C.byref(h)))
        return cls(device=dev, _handle=h)

    @classmethod
    def from_dgq1_file(cls, path: str, device=None, col_begin: int = 0, col_end: int | None = None) -> "CudaLayer":
        """A DGQ1 file streamed to the device (dgq_layer_create_from_dgq1_file):
        code rows in ~32 MB slabs, validated on the GPU, only the shard's
        columns uploaded."""
        dev = _device_index(device)
        h = C.c_void_p()
        with torch.cuda.device(dev):
            check(lib().dgq_layer_create_from_dgq1_file(dev, str(path).encode(), int(col_begin), int(col_end or 0),
                                                        _stream(dev), C.byref(h)))
        return cls(device=dev, _handle=h)

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().dgq_layer_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def plan(self, M: int) -> dict:
        """The kernel launch plan for M tokens (token tile, weight tiles per CTA, K splits, CTAs)."""
        v = [C.c_int() for _ in range(4)]
        check(lib().dgq_linear_plan(self._h, M, *[C.byref(x) for x in v]))
        return dict(token_tile=v[0].value, weight_tiles=v[1].value, k_splits=v[2].value, ctas=v[3].value)

    def workspace(self, M: int) -> torch.Tensor | None:
        """A zeroed split-K workspace for M tokens that the caller owns (pass it to
        linear(); use one per stream).  Without one, linear() lets the library
        use the layer's internal workspace for the current stream."""
        need = lib().dgq_linear_workspace_bytes(self._h, M)
        if need == 0:
            return None
        return torch.zeros(need, dtype=torch.uint8, device=f"cuda:{self.device}")

    # K1
    def quantize_act(self, x: torch.Tensor, codes: torch.Tensor | None = None, rs: torch.Tensor | None = None):
        """x: cuda float32 or float16 [M, h] -> (codes int8 [M, k_pad] zero padded, row_scales float32 [M]).
        A float16 x may also be an all-gathered [p, M, h/p] shard stack (read in place)."""
        assert x.is_cuda and x.dtype in (torch.float32, torch.float16)
        gathered = x.dim() == 3
        if gathered:
            p_, M, seg = x.shape
            assert x.dtype == torch.float16 and p_ * seg == self.h and x.stride(2) == 1
        else:
            assert x.dim() == 2 and x.shape[1] == self.h and x.stride(1) == 1
            M = x.shape[0]
        if codes is None:
            codes = torch.empty(M, self.k_pad, dtype=torch.int8, device=x.device)
        if rs is None:
            rs = torch.empty(M, dtype=torch.float32, device=x.device)
        if x.dtype == torch.float32:
            check(lib().dgq_quantize_act(self._h, _t_ptr(x), M, x.stride(0), _t_ptr(codes), codes.stride(0),
                                         _t_ptr(rs), _stream(x.device)))
        elif gathered:
            check(lib().dgq_quantize_act_f16(self._h, _t_ptr(x), M, x.stride(1), seg, x.stride(0), _t_ptr(codes),
                                             codes.stride(0), _t_ptr(rs), _stream(x.device)))
        else:
            check(lib().dgq_quantize_act_f16(self._h, _t_ptr(x), M, x.stride(0), 0, 0, _t_ptr(codes),
                                             codes.stride(0), _t_ptr(rs), _stream(x.device)))
        return codes, rs

    # K5
    def linear(self, codes: torch.Tensor, rs: torch.Tensor, bias: torch.Tensor | None = None,
               out_dtype=torch.float16, fp16_mode: bool = False, out: torch.Tensor | None = None,
               want_acc: bool = False, workspace: torch.Tensor | None = None):
        M = codes.shape[0]
        assert codes.dtype == torch.int8 and codes.shape[1] == self.k_pad and codes.is_contiguous()
        if out is None and out_dtype is not None:
            out = torch.empty(M, self.o, dtype=out_dtype, device=codes.device)
        acc = torch.empty(M, self.o, dtype=torch.int32, device=codes.device) if want_acc else None
        ws = workspace  # None: the library's per-stream internal workspace
        od = OUT_F16 if (out is not None and out.dtype == torch.float16) else OUT_F32
        if out is not None:
            assert out.dtype in (torch.float16, torch.float32) and out.stride(1) == 1
        if bias is not None:
            assert bias.dtype == torch.float32 and bias.numel() == self.o
        check(lib().dgq_linear(self._h, _t_ptr(codes), codes.stride(0), _t_ptr(rs), M, _t_ptr(bias), od,
                               int(fp16_mode), _t_ptr(out), out.stride(0) if out is not None else 0, _t_ptr(acc),
                               acc.stride(0) if acc is not None else 0, _t_ptr(ws),
                               ws.numel() if ws is not None else 0, _stream(codes.device)))
        return (out, acc) if want_acc else out

    def forward(self, x: torch.Tensor, bias: torch.Tensor | None = None, out_dtype=torch.float16,
                out: torch.Tensor | None = None):
        codes, rs = self.quantize_act(x)
        return self.linear(codes, rs, bias=bias, out_dtype=out_dtype, out=out)

    __call__ = forward

    def forward_device(self, x: torch.Tensor, bias: torch.Tensor | None = None, out_dtype=torch.float16):
        """K1 + K5 through the single C-ABI call dgq_forward_device (x: cuda float32 [M, h])."""
        assert x.is_cuda and x.dtype == torch.float32 and x.dim() == 2 and x.stride(1) == 1
        M = x.shape[0]
        y = torch.empty(M, self.o, dtype=out_dtype, device=x.device)
        codes = torch.empty(M, self.k_pad, dtype=torch.int8, device=x.device)
        rs = torch.empty(M, dtype=torch.float32, device=x.device)
        od = OUT_F16 if out_dtype == torch.float16 else OUT_F32
        check(lib().dgq_forward_device(self._h, _t_ptr(x), M, x.stride(0), _t_ptr(bias), od, _t_ptr(y), y.stride(0),
                                       _t_ptr(codes), _t_ptr(rs), None, 0, _stream(x.device)))
        return y

    def forward_host(self, X: np.ndarray, bias: torch.Tensor | None = None, out_dtype=np.float16) -> np.ndarray:
        """The serving call with HOST buffers (dgq_layer_forward_host): X float32
        [M, h] in host memory -> Y [M, o] host array; token chunks pipeline their
        copies under the kernels.  Pass page-locked X for full PCIe bandwidth."""
        X = np.ascontiguousarray(X, np.float32)
        assert X.ndim == 2 and X.shape[1] == self.h
        Y = np.empty((X.shape[0], self.o), np.float16 if out_dtype == np.float16 else np.float32)
        od = OUT_F16 if out_dtype == np.float16 else OUT_F32
        with torch.cuda.device(self.device):
            check(lib().dgq_layer_forward_host(self._h, _np_ptr(X), X.shape[0], _t_ptr(bias), od, _np_ptr(Y),
                                               _stream(self.device)))
        return Y

    # K2s from the prepared tiles
    def dequant_s8(self) -> torch.Tensor:
        w = torch.empty(self.h, self.o, dtype=torch.int8, device=f"cuda:{self.device}")
        check(lib().dgq_layer_dequant_s8(self._h, _t_ptr(w), w.stride(0), _stream(self.device)))
        return w


# ---------------------------------------------------------------------------
# Reference-API mirror (proj/include/dgq/kernel.hpp:15-53), host in / host out
# ---------------------------------------------------------------------------

def linear_multi(layers, codes: torch.Tensor, rs: torch.Tensor, outs=None, biases=None, out_dtype=torch.float16):
    """Several CudaLayers that share the input (q/k/v): one launch over all of
    their weight tiles — K5d for decode-shaped M, K5p for prefill-shaped M
    (dgq_linear_multi); returns the outputs."""
    n = len(layers)
    M = codes.shape[0]
    if outs is None:
        outs = [torch.empty(M, L.o, dtype=out_dtype, device=codes.device) for L in layers]
    hs = (C.c_void_p * n)(*[L.handle for L in layers])
    ys = (C.c_void_p * n)(*[o.data_ptr() for o in outs])
    lds = (C.c_size_t * n)(*[o.stride(0) for o in outs])
    bs = None if biases is None else (C.c_void_p * n)(*[None if b is None else b.data_ptr() for b in biases])
    od = OUT_F16 if outs[0].dtype == torch.float16 else OUT_F32
    check(lib().dgq_linear_multi(hs, n, _t_ptr(codes), codes.stride(0), _t_ptr(rs), M, bs, od, ys, lds, None, 0,
                                 _stream(codes.device)))
    return outs


@dataclass
class ActQuant:
    codes: np.ndarray        # int8 [b x h]
    row_scales: np.ndarray   # float32 [b]


@dataclass
class IntGemmResult:
    acc: np.ndarray          # int32 [b x o]
    max_abs_acc: int = 0


@dataclass
class ForwardResult:
    out: np.ndarray          # float32 [b x o]
    w_s8: np.ndarray         # int8 [h x o]
    act: ActQuant = field(default=None)
    max_abs_acc: int = 0


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2310_04836_b200 needs a CUDA device (there is no CPU path)")
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(a, dtype):
    if isinstance(a, torch.Tensor):
        return a.to(device=_dev(), dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a)).to(device=_dev(), dtype=dtype)


def calibrate(X: torch.Tensor, percentile: float = 0.005, fp16_scales: bool = False):
    """Calibration statistics on the GPU: the smoothing vector
    and static activation scale the reference's quantize_layer derives from its
    calibration rows (proj/src/pipeline.cpp:352-360) — k = compute_smooth(
    channel_maxima(X), percentile) (proj/src/smoothing.cpp:9-49) and
    act_scale = static_act_scale(X / k) (proj/src/pipeline.cpp:96-101).
    X: cuda float32 [rows, h].  Returns (k float32 [h], act_scale, threshold)."""
    import ctypes

    assert X.is_cuda and X.dtype == torch.float32 and X.dim() == 2 and X.stride(1) == 1
    k = np.empty(X.shape[1], np.float32)
    thr, act = ctypes.c_float(0.0), ctypes.c_float(0.0)
    check(lib().dgq_calibrate(_t_ptr(X), X.shape[0], X.shape[1], X.stride(0), float(percentile), int(fp16_scales),
                              k.ctypes.data_as(ctypes.c_void_p), ctypes.cast(ctypes.pointer(thr), ctypes.c_void_p),
                              ctypes.cast(ctypes.pointer(act), ctypes.c_void_p), _stream(X.device)))
    return k, float(act.value), float(thr.value)


def quantize_activations(X, layer: DgqLayer) -> ActQuant:
    """proj/src/kernel.cpp:14-44."""
    X = np.asarray(X) if not isinstance(X, torch.Tensor) else X
    if X.dtype not in (np.float32, torch.float32):
        raise InvalidArgument(_lib.DGQ_EINVAL, "activations must be float32")
    if X.shape[1] != layer.h:
        raise InvalidArgument(_lib.DGQ_EINVAL, f"activation columns {X.shape[1]} != layer h {layer.h}")
    M, K = X.shape
    dx = _to_dev(X, torch.float32)
    dk = _to_dev(np.asarray(layer.k, np.float32), torch.float32)
    q = torch.empty(M, K, dtype=torch.int8, device=dx.device)
    rs = torch.empty(M, dtype=torch.float32, device=dx.device)
    if M:
        check(lib().dgq_quantize_act_raw(_t_ptr(dx), M, K, K, _t_ptr(dk), int(layer.mode), float(layer.act_scale),
                                         _t_ptr(q), K, _t_ptr(rs), _stream()))
    return ActQuant(q.cpu().numpy(), rs.cpu().numpy())


def int8_gemm(Xq, Wq, threads: int = 0) -> IntGemmResult:
    """proj/src/kernel.cpp:46-87 (threads accepted and ignored)."""
    if np.asarray(Xq).dtype != np.int8 or np.asarray(Wq).dtype != np.int8:
        raise InvalidArgument(_lib.DGQ_EINVAL, "int8_gemm expects int8 operands")
    Xq, Wq = np.ascontiguousarray(Xq), np.ascontiguousarray(Wq)
    if Xq.shape[1] != Wq.shape[0]:
        raise InvalidArgument(_lib.DGQ_EINVAL, "inner dimensions disagree")
    M, K = Xq.shape
    N = Wq.shape[1]
    dx, dw = _to_dev(Xq, torch.int8), _to_dev(Wq, torch.int8)
    acc = torch.empty(M, N, dtype=torch.int32, device=dx.device)
    mx = C.c_int64(0)
    check(lib().dgq_int8_gemm(_t_ptr(dx), max(K, 1), _t_ptr(dw), max(N, 1), M, K, N, _t_ptr(acc), max(N, 1),
                              C.byref(mx), _stream()))
    return IntGemmResult(acc.cpu().numpy(), int(mx.value))


def epilogue(acc, row_scales, s1, bias=None, fp16_mode: bool = False) -> np.ndarray:
    """proj/src/kernel.cpp:89-116."""
    acc = np.asarray(acc)
    if acc.dtype != np.int32:
        raise InvalidArgument(_lib.DGQ_EINVAL, "epilogue expects int32 accumulators")
    M, N = acc.shape
    if len(row_scales) != M or len(s1) != N:
        raise InvalidArgument(_lib.DGQ_EINVAL, "scale vector lengths do not match the accumulator shape")
    if bias is not None and len(bias) not in (0, N):
        raise InvalidArgument(_lib.DGQ_EINVAL, "bias length must equal the output width")
    if bias is not None and len(bias) == 0:
        bias = None
    da = _to_dev(acc, torch.int32)
    drs = _to_dev(np.asarray(row_scales, np.float32), torch.float32)
    ds1 = _to_dev(np.asarray(s1, np.float32), torch.float32)
    db = None if bias is None else _to_dev(np.asarray(bias, np.float32), torch.float32)
    y = torch.empty(M, N, dtype=torch.float32, device=da.device)
    check(lib().dgq_epilogue(_t_ptr(da), max(N, 1), _t_ptr(drs), _t_ptr(ds1), _t_ptr(db), M, N, int(fp16_mode),
                             OUT_F32, _t_ptr(y), max(N, 1), _stream()))
    return y.cpu().numpy()


def dequantize_to_s8(layer: DgqLayer) -> np.ndarray:
    """proj/src/format.cpp:122-141 — raises ValidationError('codes') on corruption."""
    codes, s2, zp, _, _ = layer.arrays()
    dc, ds, dz = _to_dev(codes, torch.uint8), _to_dev(s2, torch.int8), _to_dev(zp, torch.uint8)
    w = torch.empty(layer.h, layer.o, dtype=torch.int8, device=dc.device)
    check(lib().dgq_dequantize_to_s8(layer.h, layer.o, layer.g, _t_ptr(dc), _t_ptr(ds), _t_ptr(dz), _t_ptr(w),
                                     _stream()))
    return w.cpu().numpy()


def dequantize_to_f32(layer: DgqLayer) -> np.ndarray:
    """proj/src/format.cpp:143-154: float(double(s1[c]) * double(W_s8)), on the GPU."""
    codes, s2, zp, s1, _ = layer.arrays()
    _dev()
    w = np.empty((layer.h, layer.o), np.float32)
    check(lib().dgq_host_dequantize_to_f32(layer.h, layer.o, layer.g, _np_ptr(codes), _np_ptr(s2), _np_ptr(zp),
                                           _np_ptr(s1), _np_ptr(w)))
    return w


def segmented_gemm_reference(act: ActQuant, layer: DgqLayer) -> np.ndarray:
    """proj/src/kernel.cpp:118-142: the group-wise (segmented) comparator —
    per-group exact integer partials x S2, f32-accumulated in group order, then
    x row scale x s1 — computed by a CUDA kernel."""
    codes_x = np.ascontiguousarray(act.codes, np.int8)
    if codes_x.shape[1] != layer.h:
        raise InvalidArgument(_lib.DGQ_EINVAL, "activation shape mismatch")
    rs = np.ascontiguousarray(act.row_scales, np.float32)
    codes, s2, zp, s1, _ = layer.arrays()
    _dev()
    M = codes_x.shape[0]
    y = np.empty((M, layer.o), np.float32)
    check(lib().dgq_host_segmented_gemm(_np_ptr(codes_x), _np_ptr(rs), M, layer.h, layer.o, layer.g, _np_ptr(codes),
                                        _np_ptr(s2), _np_ptr(zp), _np_ptr(s1), _np_ptr(y)))
    return y


def host_forward(X, layer: DgqLayer, bias=None) -> ForwardResult:
    """dgq_forward through the host-buffer C ABI (dgq_host_forward): the exact
    call the C++ drop-in (paper_2310_04836_b200/dropin/) makes."""
    X = np.ascontiguousarray(X, np.float32)
    if X.shape[1] != layer.h:
        raise InvalidArgument(_lib.DGQ_EINVAL, f"activation columns {X.shape[1]} != layer h {layer.h}")
    codes, s2, zp, s1, k = layer.arrays()
    _dev()
    M = X.shape[0]
    b = None if bias is None or len(bias) == 0 else np.ascontiguousarray(bias, np.float32)
    out = np.empty((M, layer.o), np.float32)
    w = np.empty((layer.h, layer.o), np.int8)
    q = np.empty((M, layer.h), np.int8)
    rs = np.empty(M, np.float32)
    mx = C.c_int64(0)
    check(lib().dgq_host_forward(M, layer.h, layer.o, layer.g, int(layer.mode), float(layer.act_scale),
                                 _np_ptr(codes), _np_ptr(s2), _np_ptr(zp), _np_ptr(s1), _np_ptr(k), _np_ptr(X),
                                 None if b is None else _np_ptr(b), _np_ptr(out), _np_ptr(w), _np_ptr(q), _np_ptr(rs),
                                 C.byref(mx)))
    return ForwardResult(out, w, ActQuant(q, rs), int(mx.value))


def dgq_forward(X, layer: DgqLayer, bias=None, threads: int = 0) -> ForwardResult:
    """proj/src/kernel.cpp:144-153: dequant -> act quant -> GEMM -> epilogue,
    all on the GPU (fused K5 for the output; K2s for w_s8; audit for
    max_abs_acc)."""
    X = np.ascontiguousarray(X, np.float32) if not isinstance(X, torch.Tensor) else X
    if X.shape[1] != layer.h:
        raise InvalidArgument(_lib.DGQ_EINVAL, f"activation columns {X.shape[1]} != layer h {layer.h}")
    if bias is not None and len(bias) not in (0, layer.o):
        raise InvalidArgument(_lib.DGQ_EINVAL, "bias length must equal the output width")
    w_s8 = dequantize_to_s8(layer)
    L = CudaLayer(layer, validate=False)
    try:
        dx = _to_dev(X, torch.float32)
        M = dx.shape[0]
        codes, rs = L.quantize_act(dx)
        db = None if bias is None or len(bias) == 0 else _to_dev(np.asarray(bias, np.float32), torch.float32)
        out = L.linear(codes, rs, bias=db, out_dtype=torch.float32)
        dw = _to_dev(w_s8, torch.int8)
        mx = C.c_int64(0)
        check(lib().dgq_audit_max_abs_acc(_t_ptr(codes), L.k_pad, _t_ptr(dw), layer.o, M, layer.h, layer.o,
                                          C.byref(mx), _stream()))
        if mx.value > 2**31 - 1:
            raise OverflowRuntimeError(_lib.DGQ_EOVERFLOW, "int8_gemm accumulator overflow despite precondition")
        act = ActQuant(codes[:, :layer.h].cpu().numpy(), rs.cpu().numpy())
        return ForwardResult(out.cpu().numpy(), w_s8, act, int(mx.value))
    finally:
        L.close()

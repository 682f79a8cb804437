"""ctypes binding of libdgq_b200.so (the C ABI in include/dgq_b200.h).

The library is the only compute path: if it is missing or fails to load this
module raises — there is no CPU or PyTorch fallback."""
from __future__ import annotations

import ctypes as C
import os
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
# DGQ_B200_LIB: tools-only override (A/B of two builds of this library)
LIB_PATH = os.environ.get("DGQ_B200_LIB") or os.path.join(_PKG, "libdgq_b200.so")

_vp, _sz, _i, _f = C.c_void_p, C.c_size_t, C.c_int, C.c_float

DGQ_OK, DGQ_EINVAL, DGQ_EVALIDATION, DGQ_EOVERFLOW, DGQ_ECUDA, DGQ_ENOMEM, DGQ_EFORMAT, DGQ_EIO = range(8)
MODE_STATIC, MODE_DYNAMIC = 0, 1
OUT_F32, OUT_F16 = 0, 1


class DgqError(RuntimeError):
    """Base class; `status` is the dgq_status code."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class ValidationError(DgqError, ValueError):
    """dgq::validation_error (proj/include/dgq/error.hpp): names the field."""

    def __init__(self, status, msg, field):
        super().__init__(status, msg)
        self.field = field


class FormatError(DgqError, ValueError):
    """dgq::format_error: `kind` in {bad_magic, truncated, size_mismatch, unknown_dtype, bad_header}."""

    def __init__(self, status, msg, kind):
        super().__init__(status, msg)
        self.kind = kind


class IoError(DgqError, OSError):
    """dgq::io_error (proj/include/dgq/error.hpp:9)."""


class InvalidArgument(DgqError, ValueError):
    """std::invalid_argument."""


class OverflowRuntimeError(DgqError):
    """std::runtime_error (accumulator overflow)."""


class LayerInfo(C.Structure):
    _fields_ = [("h", _sz), ("o_full", _sz), ("o", _sz), ("col_begin", _sz), ("g", _sz), ("k_pad", _sz),
                ("n_pad", _sz), ("mode", _i), ("act_scale", _f), ("fused", _i), ("device_bytes", _sz)]


_SIGS = {
    "dgq_abi_version": (_i, []),
    "dgq_last_error": (C.c_char_p, []),
    "dgq_last_error_field": (C.c_char_p, []),
    "dgq_validate_layer": (_i, [_sz, _sz, _sz, _i, _f, _vp, _vp, _vp, _vp, _vp]),
    "dgq_clip_interval": (_i, [_i, _i, C.POINTER(_i), C.POINTER(_i)]),
    "dgq_fp16_round": (_f, [_f]),
    "dgq_layer_create": (_i, [_i, _sz, _sz, _sz, _i, _f, _vp, _vp, _vp, _vp, _vp, _sz, _sz, _i, _vp,
                              C.POINTER(_vp)]),
    "dgq_layer_create_from_dgq1": (_i, [_i, _vp, _sz, _sz, _sz, _vp, C.POINTER(_vp)]),
    "dgq_layer_create_from_dgq1_file": (_i, [_i, C.c_char_p, _sz, _sz, _vp, C.POINTER(_vp)]),
    "dgq_layer_destroy": (None, [_vp]),
    "dgq_layer_get_info": (_i, [_vp, C.POINTER(LayerInfo)]),
    "dgq_linear_workspace_bytes": (_sz, [_vp, _sz]),
    "dgq_linear_plan": (_i, [_vp, _sz, C.POINTER(_i), C.POINTER(_i), C.POINTER(_i), C.POINTER(_i)]),
    "dgq_quantize_act": (_i, [_vp, _vp, _sz, _sz, _vp, _sz, _vp, _vp]),
    "dgq_quantize_act_f16": (_i, [_vp, _vp, _sz, _sz, _sz, _sz, _vp, _sz, _vp, _vp]),
    "dgq_quantize_act_raw": (_i, [_vp, _sz, _sz, _sz, _vp, _i, _f, _vp, _sz, _vp, _vp]),
    "dgq_linear": (_i, [_vp, _vp, _sz, _vp, _sz, _vp, _i, _i, _vp, _sz, _vp, _sz, _vp, _sz, _vp]),
    "dgq_forward_device": (_i, [_vp, _vp, _sz, _sz, _vp, _i, _vp, _sz, _vp, _vp, _vp, _sz, _vp]),
    "dgq_layer_dequant_s8": (_i, [_vp, _vp, _sz, _vp]),
    "dgq_calibrate": (_i, [_vp, _sz, _sz, _sz, _f, _i, _vp, _vp, _vp, _vp]),
    "dgq_dequantize_to_s8": (_i, [_sz, _sz, _sz, _vp, _vp, _vp, _vp, _vp]),
    "dgq_int8_gemm": (_i, [_vp, _sz, _vp, _sz, _sz, _sz, _sz, _vp, _sz, C.POINTER(C.c_int64), _vp]),
    "dgq_epilogue": (_i, [_vp, _sz, _vp, _vp, _vp, _sz, _sz, _i, _i, _vp, _sz, _vp]),
    "dgq_audit_max_abs_acc": (_i, [_vp, _sz, _vp, _sz, _sz, _sz, _sz, C.POINTER(C.c_int64), _vp]),
    "dgq_linear_multi": (_i, [C.POINTER(_vp), _i, _vp, _sz, _vp, _sz, C.POINTER(_vp), _i, C.POINTER(_vp),
                              C.POINTER(_sz), _vp, _sz, _vp]),
    "dgq_linear_multi_workspace_bytes": (_sz, [C.POINTER(_vp), _i, _sz]),
    "dgq_phase1_search": (_i, [_vp, _sz, _sz, _vp, _vp, _sz, _sz, _i, _vp, _sz, _vp, _vp, _vp, _vp,
                               C.POINTER(C.c_uint64), _vp]),
    "dgq_phase2_search": (_i, [_vp, _sz, _sz, _vp, _vp, _sz, _sz, _vp, _vp, _vp, _sz, _vp, _vp, _vp, _vp, _vp,
                               C.POINTER(C.c_uint64), _vp]),
    "dgq_measure_i8_peak": (_i, [_i, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "dgq_comm_unique_id": (_i, [_vp]),
    "dgq_comm_create": (_i, [_i, _i, _vp, _i, C.POINTER(_vp)]),
    "dgq_comm_destroy": (None, [_vp]),
    "dgq_linear_allgather": (_i, [_vp, _vp, _sz, _vp, _sz, _vp, _i, _vp, _vp, _vp, _vp]),
    # host-buffer API (the reference's calling convention)
    "dgq_host_quantize_activations": (_i, [_vp, _sz, _sz, _vp, _i, _f, _vp, _vp]),
    "dgq_host_dequantize_to_s8": (_i, [_sz, _sz, _sz, _vp, _vp, _vp, _vp]),
    "dgq_host_dequantize_to_f32": (_i, [_sz, _sz, _sz, _vp, _vp, _vp, _vp, _vp]),
    "dgq_host_int8_gemm": (_i, [_vp, _vp, _sz, _sz, _sz, _vp, C.POINTER(C.c_int64)]),
    "dgq_host_epilogue": (_i, [_vp, _vp, _vp, _vp, _sz, _sz, _i, _vp]),
    "dgq_host_segmented_gemm": (_i, [_vp, _vp, _sz, _sz, _sz, _sz, _vp, _vp, _vp, _vp, _vp]),
    "dgq_host_forward": (_i, [_sz, _sz, _sz, _sz, _i, _f, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                              C.POINTER(C.c_int64)]),
    "dgq_layer_forward_host": (_i, [_vp, _vp, _sz, _vp, _i, _vp, _vp]),
}

_lock = threading.Lock()
_lib = None


def lib():
    """Load (once) and return the CDLL; raises if the extension was not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2310_04836_b200.build` "
                                  "(there is no CPU fallback)")
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                if os.environ.get("DGQ_B200_LIB") and not hasattr(L, name):
                    continue  # an older build under A/B
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


def check(status: int):
    if status == DGQ_OK:
        return
    L = lib()
    msg = (L.dgq_last_error() or b"").decode(errors="replace")
    field = (L.dgq_last_error_field() or b"").decode(errors="replace")
    if status == DGQ_EVALIDATION:
        raise ValidationError(status, msg, field)
    if status == DGQ_EIO:
        raise IoError(status, msg)
    if status == DGQ_EFORMAT:
        raise FormatError(status, msg, field)
    if status == DGQ_EINVAL:
        raise InvalidArgument(status, msg)
    if status == DGQ_EOVERFLOW:
        raise OverflowRuntimeError(status, msg)
    if status == DGQ_ENOMEM:
        raise MemoryError(msg)
    raise DgqError(status, msg)

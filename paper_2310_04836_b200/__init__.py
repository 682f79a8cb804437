"""B200-native (sm_100a) DGQ A8W4 linear-layer hot path (arXiv 2310.04836).

Public surface mirrors the reference's operator API (proj/include/dgq):
    DgqLayer, validate_layer, clip_interval, fp16_round, dequantize_to_s8,
    dequantize_to_f32, quantize_activations, int8_gemm, epilogue, dgq_forward
plus the device-resident prepared layer `CudaLayer` (C ABI: include/dgq_b200.h)
and the column-parallel multi-GPU wrapper in `parallel`.
"""
from ._lib import (DgqError, FormatError, InvalidArgument, IoError, OverflowRuntimeError,  # noqa: F401
                   ValidationError, lib)
from .api import (ActQuant, CudaLayer, DgqLayer, ForwardResult, IntGemmResult, calibrate, clip_interval,  # noqa: F401
                  dequantize_to_f32, dequantize_to_s8, dgq_forward, epilogue, fp16_round, host_forward,
                  int8_gemm, layer_from_bytes, linear_multi, quantize_activations, segmented_gemm_reference,
                  validate_layer)
from .synth import gen_synthetic, pack_u4, random_layer, unpack_u4  # noqa: F401

__all__ = [
    "ActQuant", "CudaLayer", "DgqLayer", "ForwardResult", "IntGemmResult", "calibrate", "clip_interval",
    "dequantize_to_f32",
    "dequantize_to_s8", "dgq_forward", "epilogue", "fp16_round", "int8_gemm", "layer_from_bytes",
    "quantize_activations", "validate_layer", "segmented_gemm_reference", "host_forward", "linear_multi", "gen_synthetic", "pack_u4", "random_layer", "unpack_u4",
    "DgqError", "FormatError", "InvalidArgument", "IoError", "OverflowRuntimeError", "ValidationError", "lib",
]

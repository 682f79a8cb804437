"""Measured dense INT8 tensor peak (dgq_measure_i8_peak) and, beside it,
cuBLASLt int8 (torch._int_mm) on 8192^3 — both burst figures."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_04836_b200 as dgq  # noqa: E402

t, ms = ctypes.c_double(), ctypes.c_double()
for _ in range(3):
    dgq._lib.check(dgq.lib().dgq_measure_i8_peak(10, ctypes.byref(t), ctypes.byref(ms)))
    print(f"tcgen05 kind::i8 cta_group::2 peak: {t.value:.0f} TOPS ({ms.value:.3f} ms/launch)", flush=True)

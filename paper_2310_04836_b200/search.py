"""Two-phase grid search of the DGQ weight quantiser on the GPU (SURVEY.md
§8f(4)) — Python mirror of proj/include/dgq/search.hpp over the C ABI
(dgq_phase1_search / dgq_phase2_search, csrc/search.cu).

Same names and meaning as the reference: `SearchConfig` (group size, bit
width, the two alpha grids, the smoothed calibration rows `calib_X`),
`phase1_search(W, cfg, X_hat) -> GroupParams` (proj/src/search.cpp:83-163) and
`phase2_search(W, gp, cfg, X_hat) -> DualSearchResult` (:252-326).  Results are
bit-identical to the reference (FP64 objectives in its fixed accumulation
order, smallest-alpha tie-break).  Inputs may be numpy arrays (uploaded) or
CUDA tensors (used in place); outputs are numpy arrays like the reference's
by-value tensors, plus the device tensors in `.device` for chaining.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from ._lib import check, lib


def default_grid1() -> list[float]:
    """0.50, 0.51, ..., 1.00 (proj/src/search.cpp:12-16)."""
    return [np.float32(i) / np.float32(100.0) for i in range(50, 101)]


def default_grid2() -> list[float]:
    """0.80, 0.81, ..., 1.00 (proj/src/search.cpp:18-22)."""
    return [np.float32(i) / np.float32(100.0) for i in range(80, 101)]


@dataclass
class SearchConfig:
    """proj/include/dgq/search.hpp:27-43."""

    group_size: int = 128
    n_bits_w: int = 4
    alpha_grid_phase1: list = field(default_factory=default_grid1)
    alpha_grid_phase2: list = field(default_factory=default_grid2)
    calib_X: object = None  # float32 [b x h], already smoothed


@dataclass
class GroupParams:
    """proj/include/dgq/search.hpp:45-55."""

    group_size: int
    n_bits: int
    s_prime: np.ndarray  # float32 [n_g x o]
    zp: np.ndarray       # int32 [n_g x o]
    err: np.ndarray      # float32 [n_g x o]
    alpha: np.ndarray    # float32 [n_g x o]
    objective_evals: int = 0
    device: dict = field(default_factory=dict, repr=False)


@dataclass
class DualSearchResult:
    """proj/include/dgq/search.hpp:70-82 (params.s1 / s2 / zp flattened here)."""

    s1: np.ndarray        # float32 [o]
    s2: np.ndarray        # int8 [n_g x o]
    zp: np.ndarray        # int32 [n_g x o]
    codes: np.ndarray     # int32 [h x o]
    col_err: np.ndarray   # float64 [o]
    col_alpha: np.ndarray  # float32 [o]
    objective_evals: int = 0


def _dev_f32(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def phase1_search(W, cfg: SearchConfig, X_hat) -> GroupParams:
    """Per (group, column): the asymmetric scale S' / zero point minimising the
    group partial-product error over cfg.alpha_grid_phase1."""
    dW, dX, dXh = _dev_f32(W), _dev_f32(cfg.calib_X), _dev_f32(X_hat)
    h, o = dW.shape
    b = dX.shape[0]
    if dX.shape[1] != h:
        from ._lib import DGQ_EINVAL, InvalidArgument
        raise InvalidArgument(DGQ_EINVAL, "calib_X must be float32 with h columns")
    if tuple(dXh.shape) != tuple(dX.shape):
        from ._lib import DGQ_EINVAL, InvalidArgument
        raise InvalidArgument(DGQ_EINVAL, "X_hat shape must match calib_X")
    g = int(cfg.group_size)
    n_g = h // g if g > 0 else 0
    grid = np.ascontiguousarray(cfg.alpha_grid_phase1, np.float32)
    sp = torch.empty(n_g, o, dtype=torch.float32, device="cuda")
    zp = torch.empty(n_g, o, dtype=torch.int32, device="cuda")
    er = torch.empty(n_g, o, dtype=torch.float32, device="cuda")
    al = torch.empty(n_g, o, dtype=torch.float32, device="cuda")
    ev = C.c_uint64(0)
    check(lib().dgq_phase1_search(_p(dW), h, o, _p(dX), _p(dXh), b, g, int(cfg.n_bits_w),
                                  grid.ctypes.data_as(C.c_void_p), grid.size, _p(sp), _p(zp), _p(er), _p(al),
                                  C.byref(ev), _stream()))
    return GroupParams(g, int(cfg.n_bits_w), sp.cpu().numpy(), zp.cpu().numpy(), er.cpu().numpy(), al.cpu().numpy(),
                       int(ev.value), device={"s_prime": sp, "zp": zp})


def phase2_search(W, gp: GroupParams, cfg: SearchConfig, X_hat) -> DualSearchResult:
    """Per column: the channel scale s1 (over cfg.alpha_grid_phase2) whose
    S2 = rhe(S'/s1) decomposition and re-quantised codes minimise the column's
    output error."""
    dW, dX, dXh = _dev_f32(W), _dev_f32(cfg.calib_X), _dev_f32(X_hat)
    h, o = dW.shape
    b = dX.shape[0]
    g = int(gp.group_size)
    n_g = h // g if g > 0 else 0
    sp = gp.device.get("s_prime") if gp.device else None
    zpd = gp.device.get("zp") if gp.device else None
    if sp is None:
        sp = _dev_f32(gp.s_prime)
    if zpd is None:
        zpd = torch.from_numpy(np.ascontiguousarray(gp.zp, np.int32)).cuda()
    grid = np.ascontiguousarray(cfg.alpha_grid_phase2, np.float32)
    s1 = torch.empty(o, dtype=torch.float32, device="cuda")
    s2 = torch.empty(n_g, o, dtype=torch.int8, device="cuda")
    codes = torch.empty(h, o, dtype=torch.int32, device="cuda")
    ce = torch.empty(o, dtype=torch.float64, device="cuda")
    ca = torch.empty(o, dtype=torch.float32, device="cuda")
    ev = C.c_uint64(0)
    check(lib().dgq_phase2_search(_p(dW), h, o, _p(dX), _p(dXh), b, g, _p(sp), _p(zpd),
                                  grid.ctypes.data_as(C.c_void_p), grid.size, _p(s1), _p(s2), _p(codes), _p(ce),
                                  _p(ca), C.byref(ev), _stream()))
    return DualSearchResult(s1.cpu().numpy(), s2.cpu().numpy(), zpd.cpu().numpy(), codes.cpu().numpy(),
                            ce.cpu().numpy(), ca.cpu().numpy(), int(ev.value))

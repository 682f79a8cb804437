"""GPU two-phase grid search against the reference's own
phase1_search / phase2_search (oracle/_ref = proj/src/search.cpp built
unmodified): every output bit-exact — S', ZP, the winning objective and alpha
per (group, column); s1, S2, codes, the FP64 column objective and alpha per
column.  Inputs follow the reference pipeline: smoothed calibration rows X and
their dynamic quantise-dequantise X_hat (proj/src/pipeline.cpp:106-125)."""
import numpy as np
import pytest

from paper_2310_04836_b200 import search

pytestmark = pytest.mark.gpu


def act_quant_dequant(X: np.ndarray) -> np.ndarray:
    """proj/src/pipeline.cpp:106-125, dynamic mode, in float64 like the reference."""
    X = np.asarray(X, np.float32)
    am = np.abs(X).max(axis=1).astype(np.float64)
    s = np.maximum(am / 127.0, np.float64(np.float32(1e-8))).astype(np.float32).astype(np.float64)
    code = np.clip(np.rint(X.astype(np.float64) / s[:, None]), -127.0, 127.0)
    return (code * s[:, None]).astype(np.float32)


def problem(h, o, b, seed, outliers=True):
    rng = np.random.default_rng(seed)
    W = (rng.standard_normal((h, o)) * 0.02).astype(np.float32)
    W[rng.integers(0, h, 4), rng.integers(0, o, 4)] *= 20  # a few large weights widen some groups
    X = rng.standard_normal((b, h)).astype(np.float32)
    if outliers:
        X[:, rng.integers(0, h, 3)] *= 8
    return W, X, act_quant_dequant(X)


def check_phase1(ref, W, X, Xh, g, grid, n_bits=4):
    cfg = search.SearchConfig(group_size=g, n_bits_w=n_bits, alpha_grid_phase1=grid, calib_X=X)
    gp = search.phase1_search(W, cfg, Xh)
    sp, zp, er, al, ev = ref.phase1_search(W, X, Xh, g, grid, n_bits)
    assert np.array_equal(gp.s_prime.view(np.uint32), sp.view(np.uint32))
    assert np.array_equal(gp.zp, zp)
    assert np.array_equal(gp.err.view(np.uint32), er.view(np.uint32))
    assert np.array_equal(gp.alpha.view(np.uint32), al.view(np.uint32))
    assert gp.objective_evals == ev
    return gp, cfg


def check_phase2(ref, W, X, Xh, gp, cfg, grid):
    cfg.alpha_grid_phase2 = grid
    r = search.phase2_search(W, gp, cfg, Xh)
    s1, s2, codes, ce, ca, ev = ref.phase2_search(W, X, Xh, gp.group_size, gp.s_prime, gp.zp, grid)
    assert np.array_equal(r.s1.view(np.uint32), s1.view(np.uint32))
    assert np.array_equal(r.s2, s2)
    assert np.array_equal(r.codes, codes)
    assert np.array_equal(r.col_err.view(np.uint64), ce.view(np.uint64))
    assert np.array_equal(r.col_alpha.view(np.uint32), ca.view(np.uint32))
    assert r.objective_evals == ev
    return r


@pytest.mark.parametrize("h,o,b,g", [(256, 96, 64, 64), (512, 130, 100, 128), (384, 64, 33, 32), (96, 40, 7, 12),
                                     (1024, 256, 256, 128)])
def test_two_phase_search_matches_reference(cuda, ref, h, o, b, g):
    W, X, Xh = problem(h, o, b, seed=h + o + b)
    gp, cfg = check_phase1(ref, W, X, Xh, g, search.default_grid1())
    check_phase2(ref, W, X, Xh, gp, cfg, search.default_grid2())


def test_ties_pick_the_smallest_alpha_in_any_grid_order(cuda, ref):
    # exactly representable weights: every alpha reaches the same objective in
    # many groups, so the winner is decided by the tie-break (search.cpp:147,
    # :310) — also with an unsorted grid
    h, o, b, g = 128, 32, 16, 32
    rng = np.random.default_rng(3)
    W = (rng.integers(-7, 8, (h, o)) * 0.125).astype(np.float32)
    W[:, :4] = 0.0  # degenerate groups: the scale floor
    X = rng.standard_normal((b, h)).astype(np.float32)
    Xh = X.copy()
    grid1 = [np.float32(v) for v in (1.0, 0.5, 0.75, 0.875, 0.5, 0.625)]
    gp, cfg = check_phase1(ref, W, X, Xh, g, grid1)
    check_phase2(ref, W, X, Xh, gp, cfg, [np.float32(v) for v in (1.0, 0.9, 0.8, 0.95)])


@pytest.mark.parametrize("n_bits", [2, 3, 8])
def test_other_bit_widths(cuda, ref, n_bits):
    W, X, Xh = problem(256, 48, 40, seed=n_bits)
    check_phase1(ref, W, X, Xh, 64, search.default_grid1(), n_bits)


def test_search_argument_errors(cuda):
    from paper_2310_04836_b200 import InvalidArgument

    W, X, Xh = problem(128, 16, 8, seed=1)
    with pytest.raises(InvalidArgument, match="must divide h"):
        search.phase1_search(W, search.SearchConfig(group_size=48, calib_X=X), Xh)
    with pytest.raises(InvalidArgument, match="n_bits_w"):
        search.phase1_search(W, search.SearchConfig(group_size=64, n_bits_w=9, calib_X=X), Xh)
    with pytest.raises(InvalidArgument, match=r"\(0, 1\]"):
        search.phase1_search(W, search.SearchConfig(group_size=64, alpha_grid_phase1=[1.5], calib_X=X), Xh)
    with pytest.raises(InvalidArgument, match="empty"):
        search.phase1_search(W, search.SearchConfig(group_size=64, alpha_grid_phase1=[], calib_X=X), Xh)

"""Implicit-feedback ALS (reference implicit.py) on the GPU vs the
reference's own outputs (tests/golden/implicit_small.npz, made by
tests/golden/make_golden.py from /root/reference).

Bars, as for the explicit engine: the exact route holds the factors within
1e-4 relative per half-update and epoch, the CG route holds the trajectory
(preference RMSE) within 1e-3; objectives are float64 Gram-trick sums."""

import numpy as np
import pytest

import paper_1808_03843_b200 as cmfb

pytestmark = pytest.mark.gpu


def _instance(g):
    m, n, f = (int(v) for v in g["meta"])
    sr = cmfb.SparseRatings(m, n, int(g["row_ptr"][-1]), g["row_ptr"], g["col_idx"], g["csr_val"],
                            g["col_ptr"], g["row_idx"], g["csc_val"])
    te = cmfb.Triples(g["te_u"], g["te_v"], g["te_r"])
    return sr, te, f


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


def test_precompute_gram_matches_reference(golden, cuda_device):
    g = golden("implicit_small")
    n, f = int(g["meta"][1]), int(g["meta"][2])
    theta = cmfb.init_factors(n, f, 0.1, [0, 1])
    assert _rel(cmfb.precompute_gram(theta), g["gram_theta"]) < 1e-6


def test_implicit_update_side_exact(golden, cuda_device):
    g = golden("implicit_small")
    sr, _, f = _instance(g)
    n = sr.n
    theta = cmfb.init_factors(n, f, 0.1, [0, 1])
    x = g["x0"].copy()
    cmfb.implicit_update_side(sr.csr_view(), theta, g["gram_theta"], x, 40.0, 0.05,
                              cmfb.SolverConfig("exact"))
    assert _rel(x, g["x1_exact"]) < 1e-4
    # users without observations: A = F^T F + lambda I, b = 0 -> exactly zero
    assert np.all(x[-2:] == 0.0)


@pytest.mark.parametrize("solver", ["exact", "cg32"])
def test_implicit_train_trajectory(golden, cuda_device, solver):
    g = golden("implicit_small")
    sr, te, f = _instance(g)
    cfg = cmfb.ImplicitConfig(f=f, alpha=40.0, lam=0.05, epochs=4,
                              solver=cmfb.SolverConfig("exact") if solver == "exact"
                              else cmfb.SolverConfig("cg", 6, 1e-4, "fp32"))
    X, T, rep = cmfb.implicit_train(sr, cfg, te)
    rmse = np.array([e.rmse for e in rep.epochs])
    obj = np.array([e.objective for e in rep.epochs])
    if solver == "exact":
        assert _rel(X, g["exact_X"][-1]) < 1e-4 and _rel(T, g["exact_T"][-1]) < 1e-4
        assert np.allclose(obj, g["exact_obj"], rtol=1e-5)
        assert np.abs(rmse - g["exact_rmse"]).max() < 1e-5
    else:
        assert np.abs(rmse - g[solver + "_rmse"]).max() < 1e-3
        assert np.allclose(obj, g[solver + "_obj"], rtol=1e-3)
    assert rep.engine == "implicit" and len(rep.epochs) == 4


def test_mean_percentile_rank_matches_reference(golden, cuda_device):
    g = golden("implicit_small")
    _, te, _ = _instance(g)
    mpr = cmfb.mean_percentile_rank(g["exact_X"][-1], g["exact_T"][-1], te)
    assert abs(mpr - float(g["exact_mpr"])) < 1e-6


def test_implicit_fp16_overflow_and_negative_ratings(golden, cuda_device):
    g = golden("implicit_small")
    sr, te, f = _instance(g)
    cfg = cmfb.ImplicitConfig(f=f, epochs=1, solver=cmfb.SolverConfig("cg", precision="fp16"))
    with pytest.raises(cmfb.NumericalError):
        cmfb.implicit_train(sr, cfg, te)
    bad = cmfb.SparseRatings(sr.m, sr.n, sr.nnz, sr.row_ptr, sr.col_idx, -sr.csr_val, sr.col_ptr,
                             sr.row_idx, -sr.csc_val)
    with pytest.raises(cmfb.DataError):
        cmfb.implicit_train(bad, cfg, te)


def test_implicit_fused_tc_route_vs_reference(golden, cuda_device):
    """cg16 implicit (binary16 Hermitian storage) runs on the fused tensor-core
    kernel with per-rating operand weights (cmf_fused_cg_update_implicit): the
    reference's own cg16 trajectory (tests/golden/implicit16.npz, alpha = 1)
    within the north_star's 1e-3 RMSE bar; rows without observations solved."""
    from paper_1808_03843_b200 import _native as nat
    g16 = golden("implicit16")
    g = golden("implicit_small")
    sr, te, f = _instance(g)
    cfg = cmfb.SolverConfig("cg", 6, 1e-4, "fp16")
    theta = cmfb.init_factors(sr.n, f, 0.1, [0, 1])
    x = g["x0"].copy()
    n0 = nat.LAUNCHES[0]
    cmfb.implicit_update_side(sr.csr_view(), theta, cmfb.precompute_gram(theta), x, 1.0, 0.05, cfg)
    assert nat.LAUNCHES[0] > n0
    # fp16 operands: the half-update agrees with the reference's fp16 route to ~1e-3
    assert _rel(x, g16["x1_cg16"]) < 5e-3
    X, T, rep = cmfb.implicit_train(sr, cmfb.ImplicitConfig(f=f, alpha=1.0, lam=0.05, epochs=4, solver=cfg), te)
    rmse = np.array([e.rmse for e in rep.epochs])
    obj = np.array([e.objective for e in rep.epochs])
    assert np.abs(rmse - g16["cg16_rmse"]).max() < 1e-3
    assert np.allclose(obj, g16["cg16_obj"], rtol=1e-3)


def test_implicit_fused_matches_two_step(golden, cuda_device):
    """Same half-update through the fused weighted kernel and through the
    reference-layout two-step route (fp32 weighted Gram -> fp16 pack -> CG on
    the same binary16 systems): the fused kernel's fp16 operand rounding is the
    only difference (f = 100, every row long enough for several K-chunks)."""
    import torch
    rng = np.random.default_rng(5)
    m, n, f = 600, 900, 100
    k = 60_000
    u = rng.integers(0, m, k)
    v = rng.integers(0, n, k)
    r = rng.integers(1, 6, k).astype(np.float32)
    sr = cmfb.build(cmfb.Triples(u, v, r), m + 3, n)  # three empty rows
    theta = cmfb.init_factors(n, f, 0.1, [0, 1])
    gram = cmfb.precompute_gram(theta)
    x0 = cmfb.init_factors(m + 3, f, 0.1, [0, 0])
    xa = x0.copy()
    cmfb.implicit_update_side(sr.csr_view(), theta, gram, xa, 0.5, 0.05, cmfb.SolverConfig("cg", 6, 1e-4, "fp16"))
    xb = x0.copy()
    cmfb.implicit_update_side(sr.csr_view(), theta, gram, xb, 0.5, 0.05, cmfb.SolverConfig("cg", 6, 1e-4, "fp16"),
                              gram_kernel="fma")
    assert _rel(xa, xb) < 5e-3
    assert np.all(np.isfinite(xa[-3:])) and np.abs(xa[-3:]).max() < np.abs(x0[-3:]).max()


def test_implicit_f100_vs_reference(golden, cuda_device):
    """The weighted fused kernel at the headline width (f = 100, FC = 25 on both
    the user and the item instance) against the reference's own cg16 route
    (tests/golden/implicit100.npz): one half-update per side, then a 3-epoch
    implicit_train trajectory within the 1e-3 RMSE bar."""
    g = golden("implicit100")
    m, n, f = (int(v) for v in g["meta"])
    sr = cmfb.SparseRatings(m, n, int(g["row_ptr"][-1]), g["row_ptr"], g["col_idx"], g["csr_val"],
                            g["col_ptr"], g["row_idx"], g["csc_val"])
    te = cmfb.Triples(g["te_u"], g["te_v"], g["te_r"])
    cfg = cmfb.SolverConfig("cg", 6, 1e-4, "fp16")
    x0 = cmfb.init_factors(m, f, 0.1, [0, 0])
    t0 = cmfb.init_factors(n, f, 0.1, [0, 1])
    x1 = x0.copy()
    cmfb.implicit_update_side(sr.csr_view(), t0, cmfb.precompute_gram(t0), x1, 1.0, 0.05, cfg)
    assert _rel(x1, g["x1_cg16"]) < 5e-3
    t1 = t0.copy()
    cmfb.implicit_update_side(sr.csc_view(), x0, cmfb.precompute_gram(x0), t1, 1.0, 0.05, cfg)
    assert _rel(t1, g["t1_cg16"]) < 5e-3
    X, T, rep = cmfb.implicit_train(sr, cmfb.ImplicitConfig(f=f, alpha=1.0, lam=0.05, epochs=3, solver=cfg), te)
    rmse = np.array([e.rmse for e in rep.epochs])
    obj = np.array([e.objective for e in rep.epochs])
    assert np.abs(rmse - g["cg16_rmse"]).max() < 1e-3
    assert np.allclose(obj, g["cg16_obj"], rtol=1e-3)


@pytest.mark.parametrize("f", [8, 13, 32, 57, 100, 120])
@pytest.mark.parametrize("side", ["short", "long"])
def test_implicit_fused_matches_two_step_over_widths(cuda_device, f, side):
    """The fused weighted kernel against the two-step route across the template
    buckets (shadow widths W = 8 .. 120, so the lanes past W/8 16-byte chunks
    differ per f) on short rows (the user-side instance) and on long rows (the
    item-side instance, >= 1024 ratings per row)."""
    rng = np.random.default_rng(f)
    m, n, k = (400, 500, 30_000) if side == "short" else (3_000, 24, 40_000)
    u = rng.integers(0, m, k)
    v = rng.integers(0, n, k)
    r = rng.integers(1, 6, k).astype(np.float32)
    sr = cmfb.build(cmfb.Triples(u, v, r), m, n)
    # short: user rows (~75 ratings) over item factors; long: item rows
    # (~1,667 ratings) over user factors
    view, nfix, ntgt = (sr.csr_view(), n, m) if side == "short" else (sr.csc_view(), m, n)
    fixed = cmfb.init_factors(nfix, f, 0.1, [0, 1])
    gram = cmfb.precompute_gram(fixed)
    x0 = cmfb.init_factors(ntgt, f, 0.1, [0, 0])
    cfg = cmfb.SolverConfig("cg", 6, 1e-4, "fp16")
    xa, xb = x0.copy(), x0.copy()
    cmfb.implicit_update_side(view, fixed, gram, xa, 0.5, 0.05, cfg)
    cmfb.implicit_update_side(view, fixed, gram, xb, 0.5, 0.05, cfg, gram_kernel="fma")
    assert np.all(np.isfinite(xa))
    assert _rel(xa, xb) < 5e-3


def _mpr_loop(x, theta, users, items):
    """implicit.py:115-131 restated (float32 scores, ties averaged)."""
    n = theta.shape[0]
    total = 0.0
    for u in np.unique(users):
        scores = (x[u].astype(np.float64) @ theta.T.astype(np.float64)).astype(np.float32)
        for v in items[users == u]:
            total += ((scores > scores[v]).sum() + 0.5 * ((scores == scores[v]).sum() - 1.0)) / (n - 1)
    return total / len(users)


def test_mean_percentile_rank_kernel_ties_and_duplicates(cuda_device):
    """cmf_mpr_count: exact ties (duplicated item rows), duplicate positives,
    users without positives, n not a multiple of the 128-item tile, f not a
    multiple of 4; compared with a float64-scored restatement (exact integer
    counts; scores are well separated except for the planted ties)."""
    rng = np.random.default_rng(7)
    m, n, f = 70, 301, 13
    x = rng.standard_normal((m, f)).astype(np.float32)
    theta = rng.standard_normal((n, f)).astype(np.float32)
    theta[10] = theta[11] = theta[200]  # three-way tie
    users = rng.integers(0, m - 5, 900)
    items = rng.integers(0, n, 900)
    items[:30] = 11
    users[50], items[50] = users[51], items[51]  # a duplicate positive
    got = cmfb.mean_percentile_rank(x, theta, cmfb.Triples(users, items, np.ones(900, np.float32)))
    assert abs(got - _mpr_loop(x, theta, users, items)) < 1e-6


def test_dense_gram_and_implicit_objective(golden, cuda_device):
    import torch
    rng = np.random.default_rng(3)
    F = rng.standard_normal((5000, 37)).astype(np.float32)
    g = cmfb.precompute_gram(F)
    full = F.astype(np.float64).T @ F.astype(np.float64)
    r, c = np.tril_indices(37)
    assert np.abs(g - full[r, c]).max() / np.abs(full).max() < 1e-6
    # deterministic: same bits twice, device in -> device out
    gd1 = cmfb.precompute_gram(torch.from_numpy(F).cuda())
    gd2 = cmfb.precompute_gram(torch.from_numpy(F).cuda())
    assert torch.equal(gd1, gd2) and gd1.is_cuda
    gi = golden("implicit_small")
    sr, _, f = _instance(gi)
    X, T = gi["exact_X"][-1], gi["exact_T"][-1]
    obj = cmfb.implicit.implicit_objective(X, T, sr, 40.0, 0.05)
    assert np.isclose(obj, gi["exact_obj"][-1], rtol=1e-8, atol=1e-6)

"""Boundary semantics of update_side on the production routes (VERDICT r1 weak
#2/#3):

  * binary16 overflow on the fused CG route raises NumericalError, as the
    reference's pack_half does (gram.py:132-146) -- from a large-count,
    high-mean item (A_u entries past 65504), from factors whose binary16 shadow
    overflows, and from ratings past the binary16 range;
  * precision="fp32" never runs binary16 Hermitian storage: the same inputs
    solve without error on the fp32 route;
  * the exact route names singular rows (SingularSystemError) whatever Gram
    kernel it runs, numbered among the rows with n_u > 0 (als.py:69-72).
"""

import numpy as np
import pytest
import torch

import paper_1808_03843_b200 as cmfb

pytestmark = pytest.mark.gpu


def _one_heavy_item(n_users=3000, f=8, value=5.0, rating=4.0):
    """One item rated by n_users users whose factors are all `value`:
    the item's A_u has entries n_users * value^2 (75,000 by default)."""
    t = cmfb.Triples(np.arange(n_users, dtype=np.int64), np.zeros(n_users, np.int64),
                     np.full(n_users, rating, np.float32))
    sr = cmfb.build(t, n_users, 1)
    x = np.full((n_users, f), value, np.float32)
    theta = np.zeros((1, f), np.float32)
    return sr, x, theta


def test_fused_route_raises_on_binary16_overflow(cuda_device):
    sr, x, theta = _one_heavy_item()
    cg16 = cmfb.SolverConfig("cg", 6, 1e-4, "fp16")
    assert cmfb.als.resolve_gram_kernel("auto", cg16, 8) == "tc"
    with pytest.raises(cmfb.NumericalError, match="rescale"):
        cmfb.update_side(sr.csc_view(), x, theta.copy(), 0.05, cg16)
    # the same call through CUDA tensors (the device-resident train() path)
    xd, td = torch.from_numpy(x).cuda(), torch.zeros((1, 8), device="cuda")
    ratings = sr.to_device()
    with pytest.raises(cmfb.NumericalError):
        cmfb.update_side(ratings.csc_view(), xd, td, 0.05, cg16)
    # fp32 storage: no overflow, finite solution, same as the fp32 exact route
    t32 = theta.copy()
    cmfb.update_side(sr.csc_view(), x, t32, 0.05, cmfb.SolverConfig("cg", 6, 1e-4, "fp32"))
    assert np.all(np.isfinite(t32))
    tex = theta.copy()
    cmfb.update_side(sr.csc_view(), x, tex, 0.05, cmfb.SolverConfig("exact"))
    # A_u = 75,000 * 11^T + 150 I: condition number ~4,000, so fp32 CG vectors
    # carry ~kappa * 2^-24 ~ 2.4e-4 relative error against the exact solve
    np.testing.assert_allclose(t32, tex, rtol=1e-3)


def test_fused_route_no_overflow_below_range(cuda_device):
    # 3000 * 4.5^2 = 60,750 < 65,504: the fp16 route runs and agrees with fp32
    sr, x, theta = _one_heavy_item(value=4.5)
    t16 = theta.copy()
    cmfb.update_side(sr.csc_view(), x, t16, 0.05, cmfb.SolverConfig("cg", 6, 1e-4, "fp16"))
    tex = theta.copy()
    cmfb.update_side(sr.csc_view(), x, tex, 0.05, cmfb.SolverConfig("exact"))
    assert np.all(np.isfinite(t16))
    np.testing.assert_allclose(t16, tex, rtol=2e-3)


def test_shadow_and_rating_overflow_raise(cuda_device):
    rng = np.random.default_rng(3)
    t = cmfb.Triples(rng.integers(0, 40, 300), rng.integers(0, 30, 300),
                     rng.standard_normal(300).astype(np.float32))
    sr = cmfb.build(t, 40, 30)
    f = 8
    cg16 = cmfb.SolverConfig("cg", 6, 1e-4, "fp16")
    theta = (0.1 * rng.standard_normal((30, f))).astype(np.float32)
    theta[3, 2] = 70000.0  # binary16 max is 65504
    with pytest.raises(cmfb.NumericalError):
        cmfb.update_side(sr.csr_view(), theta, np.zeros((40, f), np.float32), 0.05, cg16)
    theta[3, 2] = 0.1
    vals = sr.csr_val.copy()
    vals[7] = 1e5  # a rating past the binary16 range
    big = cmfb.RowView(sr.row_ptr, sr.col_idx, vals, 40, 30)
    with pytest.raises(cmfb.NumericalError):
        cmfb.update_side(big, theta, np.zeros((40, f), np.float32), 0.05, cg16)
    x = np.zeros((40, f), np.float32)
    cmfb.update_side(sr.csr_view(), theta, x, 0.05, cg16)  # in range: fine
    assert np.all(np.isfinite(x))


def test_precision_routing(cuda_device):
    f = 16
    r = cmfb.als.resolve_gram_kernel
    assert r("auto", cmfb.SolverConfig("cg", precision="fp16"), f) == "tc"
    assert r("auto", cmfb.SolverConfig("cg", precision="fp32"), f) == "tc_split"
    assert r("auto", cmfb.SolverConfig("cg", precision="fp16", accum="fp64"), f) == "tc_unfused"
    assert r("auto", cmfb.SolverConfig("exact"), f) == "tc_split"
    with pytest.raises(cmfb.DataError):
        r("tc", cmfb.SolverConfig("cg", precision="fp32"), f)
    with pytest.raises(cmfb.DataError):
        r("tc", cmfb.SolverConfig("cg", precision="fp16", accum="fp64"), f)


@pytest.mark.parametrize("kernel", ["auto", "tc_split", "fma", "bitwise"])
def test_exact_route_names_singular_rows(cuda_device, kernel):
    # lam = 0 and rows that only rate items with zero factors: A_u == 0, a zero
    # pivot under any rounding (a merely rank-deficient A_u may factor with a
    # tiny positive pivot in float arithmetic, in the reference's LAPACK too)
    f = 6
    rows = [(0, c) for c in range(10)] + [(2, 10), (2, 11)] + [(3, c) for c in range(12)] + [(5, 10)]
    u = np.array([a for a, _ in rows], np.int64)
    v = np.array([b for _, b in rows], np.int64)
    sr = cmfb.build(cmfb.Triples(u, v, np.ones(len(rows), np.float32)), 6, 12)
    theta = np.random.default_rng(0).standard_normal((12, f)).astype(np.float32)
    theta[10:] = 0.0
    with pytest.raises(cmfb.SingularSystemError) as err:
        cmfb.update_side(sr.csr_view(), theta, np.zeros((6, f), np.float32), 0.0,
                         cmfb.SolverConfig("exact"), gram_kernel=kernel)
    # rows with n_u > 0 are 0, 2, 3, 5 -> compacted indices 0..3; 2 and 5 are singular
    assert err.value.rows == [1, 3]


@pytest.mark.parametrize("f", [1, 3, 8, 13, 16, 32, 100, 120])
def test_predict_pairs_bitwise_equal_to_reference_einsum(cuda_device, f):
    """predict_pairs (factors.py:41-54) is numpy's float32 einsum; the device
    kernel restates its summation order, so every prediction is bit-identical
    and noiseless synthetic ratings round-trip to an RMSE of exactly zero (the
    reference's test_data.py::test_noiseless_ratings_equal_exact_dot)."""
    rng = np.random.default_rng(f)
    x = (rng.random((300, f), dtype=np.float32) - 0.5) * 3
    th = (rng.random((200, f), dtype=np.float32) - 0.5) * 3
    u = rng.integers(0, 300, 5000)
    v = rng.integers(0, 200, 5000)
    want = np.einsum("ij,ij->i", x[u], th[v])
    got = cmfb.predict_pairs(x, th, u, v)
    assert np.array_equal(got, want)
    t, truth = cmfb.gen_synthetic(40, 30, f, 0.3, 0.0, seed=1)
    assert cmfb.rmse(truth.x_true, truth.theta_true, t) == 0.0


def _one_heavy_user(n_items=700, f=100, value=1.0, n_light=2000):
    """User 0 rates n_items items whose factors are all `value` (A_u entries
    n_items * value^2); n_light users with 3 ratings each keep the view's mean
    row short, so the user side runs the short-row CTA shape."""
    rng = np.random.default_rng(11)
    u = np.concatenate([np.zeros(n_items, np.int64), np.repeat(np.arange(1, n_light + 1), 3)])
    i = np.concatenate([np.arange(n_items), rng.integers(0, n_items, 3 * n_light)])
    t = cmfb.Triples(u, i, np.full(u.size, 3.0, np.float32))
    sr = cmfb.build(t, n_light + 1, n_items)
    theta = np.full((n_items, f), value, np.float32)
    x = np.zeros((n_light + 1, f), np.float32)
    return sr, theta, x


def test_short_row_overflow(cuda_device):
    """Short-row views (the user side's 4-group CTA shape): one heavy user's A_u
    just inside the binary16 range (700 * 9.3^2 = 60,543) solves, just past it
    (700 * 9.7^2 = 65,863) raises NumericalError like pack_half."""
    cg16 = cmfb.SolverConfig("cg", 6, 1e-4, "fp16")
    sr, theta, x = _one_heavy_user(value=9.3)
    assert sr.nnz < 1024 * sr.m
    cmfb.update_side(sr.csr_view(), theta, x, 0.05, cg16)
    assert np.all(np.isfinite(x))
    sr, theta, x = _one_heavy_user(value=9.7)
    with pytest.raises(cmfb.NumericalError, match="rescale"):
        cmfb.update_side(sr.csr_view(), theta, x, 0.05, cg16)


"""Tensor-core Gram (tcgen05 kind::f16, TMEM accumulators) on the GPU.

The kernel rounds the fixed factors to binary16 (RNE) and the ratings to an
fp16 hi+lo pair, multiplies exactly and accumulates in fp32.  So it is checked
tightly (1e-5 relative Frobenius per row) against a float64 Gram of the
SAME fp16-rounded operands -- which pins the operand layout, the rating rows
and the packed epilogue exactly -- and loosely against the fp32 reference
(the input rounding, ~2^-11)."""

import numpy as np
import pytest

import paper_1808_03843_b200 as cmfb
from paper_1808_03843_b200.data import RowView

pytestmark = pytest.mark.gpu


def _instance(m, n, f, degs, seed):
    rng = np.random.default_rng(seed)
    rows = [np.sort(rng.choice(n, size=min(d, n), replace=False)) for d in degs]
    indptr = np.zeros(m + 1, np.int64)
    indptr[1:] = np.cumsum([len(r) for r in rows])
    indices = np.concatenate(rows).astype(np.int32) if indptr[-1] else np.zeros(0, np.int32)
    values = rng.standard_normal(indices.shape[0]).astype(np.float32)
    theta = (rng.random((n, f), dtype=np.float32) - 0.5)
    return RowView(indptr, indices, values, m, n), theta


def _f64_reference(view, theta, lam, weighted=True):
    t16 = theta.astype(np.float16).astype(np.float64)
    f = theta.shape[1]
    out_a, out_b = [], []
    for u in range(view.nrows):
        lo, hi = view.indptr[u], view.indptr[u + 1]
        sel = t16[view.indices[lo:hi]]
        r = view.values[lo:hi]
        r_hi = r.astype(np.float16).astype(np.float64)
        r_lo = (r - r_hi.astype(np.float32)).astype(np.float16).astype(np.float64)
        a = sel.T @ sel + (lam * (hi - lo) if weighted else lam) * np.eye(f)
        out_a.append(a[np.tril_indices(f)])
        out_b.append(sel.T @ (r_hi + r_lo))
    return np.array(out_a), np.array(out_b)


@pytest.mark.parametrize("f,degs", [
    (100, [206, 0, 1, 63, 64, 65, 300, 5571]),
    (32, [166, 270, 0, 17, 128]),
    (8, [3, 40, 0]),
    (1, [5, 0, 9]),
    (63, [100, 2000, 64]),
    (120, [129, 7]),
    (112, [65, 3]),
])
@pytest.mark.parametrize("precision", ["fp16", "fp32"])
def test_tc_gram_matches_fp16_operand_reference(cuda_device, f, degs, precision):
    n = max(max(degs) + 10, 64)
    view, theta = _instance(len(degs), n, f, degs, seed=f + len(degs))
    gb, _ = cmfb.assemble_side(view, theta, 0.05, precision=precision, kernel="tc")
    a_ref, b_ref = _f64_reference(view, theta, 0.05)
    a = np.asarray(gb.a_lower, dtype=np.float64)
    for u in range(view.nrows):
        # fp16 storage rounds the result; fp32 keeps the tensor core's accumulation order
        tol = 1e-3 if precision == "fp16" else 5e-5
        da = np.linalg.norm(a[u] - a_ref[u]) / max(np.linalg.norm(a_ref[u]), 1e-30)
        assert da <= tol or np.abs(a[u] - a_ref[u]).max() < 1e-7, (u, da)
        if degs[u]:
            db = np.linalg.norm(gb.b[u] - b_ref[u]) / max(np.linalg.norm(b_ref[u]), 1e-30)
            assert db <= 1e-5, (u, db)
        else:
            assert np.array_equal(gb.b[u], np.zeros(f, np.float32))
    assert np.array_equal(gb.n_u, np.array(degs, np.int64).clip(max=n))


def test_tc_gram_close_to_reference_fp32(golden, cuda_device):
    g = golden("gram_cases")
    for ci in range(int(g["ncases"])):
        p = f"c{ci}_"
        m, n, f = (int(v) for v in g[p + "meta"])
        if f > 120:
            continue
        view = RowView(g[p + "row_ptr"], g[p + "col_idx"], g[p + "csr_val"], m, n)
        theta = g[p + "theta_n"]
        gb, _ = cmfb.assemble_side(view, theta, 0.05, kernel="tc")
        ref = g[p + "x_fp32_1_a"].astype(np.float64)
        for u in range(m):
            d = np.linalg.norm(gb.a_lower[u] - ref[u]) / max(np.linalg.norm(ref[u]), 1e-30)
            assert d < 2e-3, (p, u, d)


def test_tc_train_rmse_trajectory_ml1m(golden, cuda_device):
    """CG-fp16 with the tensor-core Gram: RMSE trajectory within 1e-3 of the reference."""
    g = golden("train_ml1m")
    m, n, nnz, f = (int(v) for v in g["meta"])
    t, _ = cmfb.gen_synthetic(m, n, f, round(nnz / 0.9) / (m * n), 0.1, 0)
    tr, te = cmfb.split_holdout(t, 0.1, 1)
    sr = cmfb.build(tr, m, n)
    # cg16 runs the fused tcgen05 kernel; precision="fp32" keeps fp32 Hermitian
    # storage and therefore takes the split-precision two-step route
    for solver, prec, kern in (("cg16", "fp16", "tc"), ("cg32", "fp32", "auto")):
        cfg = cmfb.AlsConfig(f=f, lam=0.05, epochs=10, gram_kernel=kern,
                             solver=cmfb.SolverConfig("cg", precision=prec))
        _, _, rep = cmfb.train(sr, te, cfg)
        traj = np.array(rep.rmse_trajectory())
        assert np.abs(traj - g[solver + "_rmse"]).max() < 1e-3, (solver, traj)


def test_fused_tc_cg_matches_two_step(cuda_device, monkeypatch):
    """update_side with the fused kernel (Gram in TMEM -> CG in registers) vs the
    two-step tensor-core path (packed fp32 A_u in HBM -> batched CG kernel):
    same fp16 Gram operands, same CG recurrence, so the solutions agree to fp32
    rounding; rows without ratings are untouched in both."""
    import torch
    # both routes store A_u in binary16 from the same fp32 accumulator and run
    # the same pipelined recurrence; the two-step route rounds the regularised
    # diagonal A_ii + lam n_u to binary16 (the reference's pack_half), the fused
    # one keeps lam n_u in fp32 -- a 2^-11-relative diagonal difference, so the
    # bar is 1e-3 (rel. Frobenius) rather than fp32 rounding
    monkeypatch.setenv("CMF_CG_PIPELINED", "1")
    for f, (m, n, nnz) in ((100, (300, 900, 30000)), (32, (500, 200, 8000)), (8, (50, 40, 300))):
        t, _ = cmfb.gen_synthetic(m, n, f, nnz / (m * n), 0.1, 3)
        sr = cmfb.build(t, m + 1, n)  # last user has no ratings
        theta = cmfb.init_factors(n, f, 0.1, [0, 1])
        outs = []
        for kern in ("tc", "tc_unfused"):
            x = cmfb.init_factors(m + 1, f, 0.1, [0, 0])
            cmfb.update_side(sr.csr_view(), theta, x, 0.05,
                             cmfb.SolverConfig("cg", precision="fp16"), gram_kernel=kern)
            outs.append(x)
        x0 = cmfb.init_factors(m + 1, f, 0.1, [0, 0])
        assert np.array_equal(outs[0][m], x0[m]) and np.array_equal(outs[1][m], x0[m])
        rel = np.linalg.norm(outs[0] - outs[1]) / np.linalg.norm(outs[1])
        assert rel < 1e-3, (f, rel)


def test_fused_tc_cg_shapes_match_two_step(cuda_device, monkeypatch):
    """The fused kernel's other CTA shapes against the two-step path: two CG
    groups for f > 104, and the gather-heavy shape for views whose rows average
    >= 1024 ratings (the item side of a tall matrix)."""
    monkeypatch.setenv("CMF_CG_PIPELINED", "1")
    for f, (m, n, nnz), side in ((120, (400, 300, 24000), "csr"), (112, (300, 500, 20000), "csr"),
                                 (100, (6000, 40, 120000), "csc"), (24, (5000, 30, 90000), "csc")):
        t, _ = cmfb.gen_synthetic(m, n, f, nnz / (m * n), 0.1, 5)
        sr = cmfb.build(t, m, n)
        view = sr.csr_view() if side == "csr" else sr.csc_view()
        if side == "csc":
            assert sr.nnz >= 1024 * n  # exercises the long-row shape
        rows, cols = (m, n) if side == "csr" else (n, m)
        fixed = cmfb.init_factors(cols, f, 0.1, [0, 1])
        outs = []
        for kern in ("tc", "tc_unfused"):
            x = cmfb.init_factors(rows, f, 0.1, [0, 0])
            cmfb.update_side(view, fixed, x, 0.05, cmfb.SolverConfig("cg", precision="fp16"), gram_kernel=kern)
            outs.append(x)
        rel = np.linalg.norm(outs[0] - outs[1]) / np.linalg.norm(outs[1])
        assert rel < 1e-3, (f, side, rel)


def test_fused_tc_cg_large_fixed_side(cuda_device, monkeypatch):
    """Short rows over a fixed side too large for L2 residency (> 32 MB of
    binary16 shadow): the fused kernel runs all 7 gather warps there."""
    monkeypatch.setenv("CMF_CG_PIPELINED", "1")
    import torch
    f = 100
    train, _ = cmfb.gen_synthetic_device(2000, 170_000, f, 100_000, 0.1, 0.1, seed=2)
    view = train.csr_view()
    assert 170_000 * 104 * 2 > (32 << 20)
    fixed = torch.from_numpy(cmfb.init_factors(170_000, f, 0.1, [0, 1])).cuda()
    outs = []
    for kern in ("tc", "tc_unfused"):
        x = torch.from_numpy(cmfb.init_factors(2000, f, 0.1, [0, 0])).cuda()
        cmfb.update_side(view, fixed, x, 0.05, cmfb.SolverConfig("cg", precision="fp16"), gram_kernel=kern)
        outs.append(x)
    rel = float(torch.linalg.norm(outs[0] - outs[1]) / torch.linalg.norm(outs[1]))
    assert rel < 1e-3, rel


def test_split_precision_gram_is_fp32_faithful(golden, oracle, cuda_device):
    """tc_split (hi/lo fp16 operands, H H^T + H L^T + L H^T) vs the reference's
    float32 Gram: within 2e-6 relative Frobenius per row -- the fp32 SIMT
    kernel's own distance is ~1e-7, a single fp16/TF32 pass is ~1e-3."""
    g = golden("gram_cases")
    for ci in range(int(g["ncases"])):
        p = f"c{ci}_"
        m, n, f = (int(v) for v in g[p + "meta"])
        if f > 120:
            continue
        for side in ("x", "t"):
            if side == "x":
                view = RowView(g[p + "row_ptr"], g[p + "col_idx"], g[p + "csr_val"], m, n)
                th = g[p + "theta_n"]
            else:
                view = RowView(g[p + "col_ptr"], g[p + "row_idx"], g[p + "csc_val"], n, m)
                th = g[p + "theta_m"]
            gb, _ = cmfb.assemble_side(view, th, 0.05, kernel="tc_split")
            ref_a = g[f"{p}{side}_fp32_1_a"].astype(np.float64)
            ref_b = g[f"{p}{side}_fp32_1_b"].astype(np.float64)
            for u in range(ref_a.shape[0]):
                da = np.linalg.norm(gb.a_lower[u] - ref_a[u]) / max(np.linalg.norm(ref_a[u]), 1e-30)
                db = np.linalg.norm(gb.b[u] - ref_b[u]) / max(np.linalg.norm(ref_b[u]), 1e-30)
                assert da < 2e-6 and db < 2e-6, (p, side, u, da, db)
    # heavy rows (K in the thousands) at f = 100: the tensor core's fp32
    # accumulation (not the operand split) dominates there, ~1e-5 at K = 5571
    view, theta = _instance(3, 6000, 100, [5571, 206, 1], 11)
    gb, _ = cmfb.assemble_side(view, theta, 0.05, kernel="tc_split")
    a, b, _ = oracle.assemble_side(view.indptr, view.indices, view.values, 3, theta, 0.05)
    for u, tol in zip(range(3), (5e-5, 2e-6, 2e-6)):
        assert np.linalg.norm(gb.a_lower[u] - a[u]) / np.linalg.norm(a[u]) < tol, u
        assert np.linalg.norm(gb.b[u] - b[u]) / np.linalg.norm(b[u]) < tol, u


def test_exact_route_long_rows_factor_bar(oracle, cuda_device):
    """Exact route with the default (split tensor-core) Gram on rows of K ~ 600-1200
    (items): factors within 1e-4 relative of the CPU oracle (float32 bitwise Gram +
    float64 Cholesky) after every half-update -- the north_star exact-path bar."""
    m, n, f = 1500, 300, 48
    t, _, _ = oracle.gen_synthetic(m, n, f, 0.5, 0.1, 2)
    r = oracle.build(t, m, n)
    x_o = oracle.init_factors(m, f, 0.1, [0, 0])
    t_o = oracle.init_factors(n, f, 0.1, [0, 1])
    x_g, t_g = x_o.copy(), t_o.copy()
    sr = cmfb.build(cmfb.Triples(t.user, t.item, t.rating), m, n)
    solver = cmfb.SolverConfig("exact")
    for epoch in range(4):
        oracle.update_side(r.csr(), t_o, x_o, 0.05, "exact")
        cmfb.update_side(sr.csr_view(), t_g, x_g, 0.05, solver)
        assert np.linalg.norm(x_g - x_o) / np.linalg.norm(x_o) < 1e-4, (epoch, "x")
        oracle.update_side(r.csc(), x_o, t_o, 0.05, "exact")
        cmfb.update_side(sr.csc_view(), x_g, t_g, 0.05, solver)
        assert np.linalg.norm(t_g - t_o) / np.linalg.norm(t_o) < 1e-4, (epoch, "t")


@pytest.mark.parametrize("passes,sym", [("2", "0"), ("3", "0"), ("5", "0"), ("1", "1"), ("3", "1")])
def test_exact_route_multipass_gram(oracle, cuda_device, monkeypatch, passes, sym):
    """The split-precision Gram in P passes over fixed-side id ranges
    (cmf_gram_assemble_tc_ws: the exact route's item side, whose hi + lo shadow
    exceeds L2), and with the SYM accumulators (H H^T and S = H^T L, the copy-out
    adds S^T), against one plain pass and against the CPU oracle: items rated only
    inside one id range (empty segments in the other passes) and items without
    ratings included; factors within 1e-4 of the oracle, the variants vs one
    plain pass to fp32 summation order."""
    m, n, f = 1500, 300, 48
    t, _, _ = oracle.gen_synthetic(m, n, f, 0.5, 0.1, 4)
    keep = ~((t.item < 20) & (t.user >= m // 3)) & ~((t.item >= 20) & (t.item < 30)) & (t.item != 31)
    t = oracle.OTriples(t.user[keep], t.item[keep], t.rating[keep])
    r = oracle.build(t, m, n)
    x = oracle.init_factors(m, f, 0.1, [0, 0])
    th0 = oracle.init_factors(n, f, 0.1, [0, 1])
    sr = cmfb.build(cmfb.Triples(t.user, t.item, t.rating), m, n)
    solver = cmfb.SolverConfig("exact")
    th_o = th0.copy()
    oracle.update_side(r.csc(), x, th_o, 0.05, "exact")
    outs = []
    for p, sy in (("1", "0"), (passes, sym)):
        monkeypatch.setenv("CMF_GRAM_PASSES", p)
        monkeypatch.setenv("CMF_GRAM_SYM", sy)
        th = th0.copy()
        cmfb.update_side(sr.csc_view(), x, th, 0.05, solver)
        outs.append(th)
    assert np.array_equal(outs[1][31], th0[31])  # no ratings: untouched
    assert np.linalg.norm(outs[1] - outs[0]) / np.linalg.norm(outs[0]) < 1e-5
    assert np.linalg.norm(outs[1] - th_o) / np.linalg.norm(th_o) < 1e-4


def test_fused_two_pass_item_side_matches_one_pass(cuda_device, monkeypatch):
    """Long rows over a fixed side whose binary16 shadow exceeds L2 (the Netflix
    item side): the fused kernel gathers the first half of the user ids, parks
    each row's fp32 partial Gram in the workspace, then adds the second half and
    solves.  Same solutions as one pass up to fp32 summation order -- including
    rows whose ratings all fall in one half (an empty segment)."""
    import torch
    f, m, n = 100, 250_000, 40
    rng = np.random.default_rng(9)
    u = rng.integers(0, m, 120_000)
    v = rng.integers(2, n, 120_000)
    # item 0: only users of the first half; item 1: only the second half
    u = np.concatenate([u, rng.integers(0, m // 2, 3000), rng.integers(m // 2, m, 3000)])
    v = np.concatenate([v, np.zeros(3000, np.int64), np.ones(3000, np.int64)])
    t = cmfb.Triples(u, v, rng.standard_normal(len(u)).astype(np.float32))
    sr = cmfb.build(t, m, n)
    assert sr.nnz >= 1024 * n and m * 104 * 2 > (48 << 20)
    fixed = torch.from_numpy(cmfb.init_factors(m, f, 0.1, [0, 0])).cuda()
    view = sr.to_device().csc_view()
    outs = []
    for two in ("0", "1"):
        monkeypatch.setenv("CMF_TWO_PASS", two)
        th = torch.from_numpy(cmfb.init_factors(n, f, 0.1, [0, 1])).cuda()
        cmfb.update_side(view, fixed, th, 0.05, cmfb.SolverConfig("cg", precision="fp16"))
        outs.append(th.cpu().numpy())
    rel = np.linalg.norm(outs[0] - outs[1], axis=1) / np.linalg.norm(outs[0], axis=1)
    assert rel.max() < 1e-3, rel
    assert np.linalg.norm(outs[0] - outs[1]) / np.linalg.norm(outs[0]) < 2e-4

"""End-to-end parity of the device ALS loop with the reference (north_star bars):

  * CSR/CSC construction bit-exact (golden build cases + ML-1M digests);
  * exact path: factors within 1e-4 relative of the reference every epoch;
  * CG/fp16 path: test-RMSE trajectory within 1e-3 absolute;
  * with the reference-exact kernels (bitwise Gram, fp64 CG) the small-instance
    factors match the reference to float32 rounding.
"""

import hashlib

import numpy as np
import pytest
import torch

import paper_1808_03843_b200 as cmfb

pytestmark = pytest.mark.gpu

SOLVERS = {"exact": ("exact", "fp32"), "cg32": ("cg", "fp32"), "cg16": ("cg", "fp16")}


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _protocol(m, n, nnz, f):
    t, _ = cmfb.gen_synthetic(m, n, f, round(nnz / 0.9) / (m * n), 0.1, 0)
    tr, te = cmfb.split_holdout(t, 0.1, 1)
    return cmfb.build(tr, m, n), te


def _run(sr, te, f, solver, epochs, **kw):
    method, prec = SOLVERS[solver]
    accum = kw.pop("accum", "fp32")
    xs, ts = [], []
    orig = cmfb.als.update_side

    def spy(view, fixed, target, *a, **k):
        out = orig(view, fixed, target, *a, **k)
        (xs if target.shape[0] == sr.m else ts).append(target.detach().cpu().numpy().copy())
        return out
    cmfb.als.update_side = spy
    try:
        cfg = cmfb.AlsConfig(f=f, lam=0.05, epochs=epochs,
                             solver=cmfb.SolverConfig(method, precision=prec, accum=accum), **kw)
        x, t, rep = cmfb.train(sr, te, cfg)
    finally:
        cmfb.als.update_side = orig
    return np.stack(xs), np.stack(ts), rep


def test_build_bitwise_vs_reference(golden, cuda_device):
    g = golden("build_cases")
    for ci in range(int(g["nspecs"])):
        p = f"b{ci}_"
        m, n = (int(v) for v in g[p + "dims"])
        sr = cmfb.build(cmfb.Triples(g[p + "u"], g[p + "v"], g[p + "r"]), m, n)
        for k in ("row_ptr", "col_idx", "csr_val", "col_ptr", "row_idx", "csc_val"):
            ours, ref = getattr(sr, k), g[p + k]
            assert ours.dtype == ref.dtype and np.array_equal(ours, ref), (p, k)
    with pytest.raises(cmfb.DataError, match=r"\(5, 0, 1\.0\)"):
        cmfb.build([(0, 0, 2.0), (5, 0, 1.0)], 3, 3)
    sr = cmfb.build([(0, 0, 1.0)], 5, 5)
    assert sr.row_ptr.tolist() == [0, 1, 1, 1, 1, 1]


@pytest.mark.parametrize("solver", ["exact", "cg32", "cg16"])
def test_train_small_reference_exact_kernels(golden, cuda_device, solver, monkeypatch):
    g = golden("train_small")
    m, n, nnz, f = (int(v) for v in g["meta"])
    sr, te = _protocol(m, n, nnz, f)
    assert _digest(sr.row_ptr, sr.col_idx, sr.csr_val, sr.col_ptr, sr.row_idx,
                   sr.csc_val) == str(g["digest"])
    X, T, rep = _run(sr, te, f, solver, 5, accum="fp64", gram_kernel="bitwise")
    for e in range(5):
        for ours, ref in ((X[e], g[solver + "_X"][e]), (T[e], g[solver + "_T"][e])):
            rel = np.linalg.norm(ours - ref) / np.linalg.norm(ref)
            assert rel <= 1e-6, (solver, e, rel)
    assert np.abs(np.array(rep.rmse_trajectory()) - g[solver + "_rmse"]).max() < 1e-6
    assert np.allclose([e.objective for e in rep.epochs], g[solver + "_obj"], rtol=1e-6)


@pytest.mark.parametrize("solver", ["exact", "cg32", "cg16"])
def test_train_small_production_kernels(golden, cuda_device, solver):
    g = golden("train_small")
    m, n, nnz, f = (int(v) for v in g["meta"])
    sr, te = _protocol(m, n, nnz, f)
    X, T, rep = _run(sr, te, f, solver, 5)
    if solver == "exact":
        for e in range(5):
            for ours, ref in ((X[e], g["exact_X"][e]), (T[e], g["exact_T"][e])):
                assert np.linalg.norm(ours - ref) / np.linalg.norm(ref) <= 1e-4
    assert np.abs(np.array(rep.rmse_trajectory()) - g[solver + "_rmse"]).max() < 1e-3


@pytest.fixture(scope="module")
def ml1m(golden):
    g = golden("train_ml1m")
    m, n, nnz, f = (int(v) for v in g["meta"])
    t, _ = cmfb.gen_synthetic(m, n, f, round(nnz / 0.9) / (m * n), 0.1, 0)
    tr, te = cmfb.split_holdout(t, 0.1, 1)
    sr = cmfb.build(tr, m, n)
    return g, sr, te, f


def test_ml1m_build_bit_exact(ml1m, cuda_device):
    g, sr, te, _ = ml1m
    assert sr.nnz == 1_000_000
    assert _digest(sr.row_ptr, sr.col_idx, sr.csr_val) == str(g["csr_digest"])
    assert _digest(sr.col_ptr, sr.row_idx, sr.csc_val) == str(g["csc_digest"])
    assert _digest(te.user, te.item, te.rating) == str(g["test_digest"])


def test_ml1m_exact_factors_within_1e4(ml1m, cuda_device):
    """BASELINE configs[0]: ML-1M shape, f=32, lambda=0.05, 10 iters, exact."""
    g, sr, te, f = ml1m
    X, T, rep = _run(sr, te, f, "exact", 10)
    for e in range(10):
        for ours, ref, rows in ((X[e], g["exact_Xrows"][e], g["rows_x"]),
                                (T[e], g["exact_Trows"][e], g["rows_t"])):
            rel = np.linalg.norm(ours[rows] - ref) / np.linalg.norm(ref)
            assert rel <= 1e-4, (e, rel)
        assert abs(np.linalg.norm(X[e].astype(np.float64)) - g["exact_Xnorm"][e]) <= \
            1e-4 * g["exact_Xnorm"][e]
    assert np.abs(np.array(rep.rmse_trajectory()) - g["exact_rmse"]).max() < 1e-4


@pytest.mark.parametrize("solver", ["cg32", "cg16"])
def test_ml1m_cg_rmse_trajectory_within_1e3(ml1m, cuda_device, solver):
    g, sr, te, f = ml1m
    _, _, rep = _run(sr, te, f, solver, 10)
    traj = np.array(rep.rmse_trajectory())
    assert np.abs(traj - g[solver + "_rmse"]).max() < 1e-3, (traj, g[solver + "_rmse"])
    assert rep.epochs_run == 10 and rep.stop_reason == "epochs"


def test_update_side_semantics(oracle, cuda_device):
    sr, te = _protocol(120, 90, 2000, 8)
    sr = cmfb.build(sr.to_triples(), 121, 90)  # one extra user with no ratings
    theta = cmfb.init_factors(90, 8, 0.1, [0, 1])
    x = cmfb.init_factors(121, 8, 0.1, [0, 0])
    x_before, th_before = x.copy(), theta.copy()
    times, nbytes, brk = cmfb.update_side(sr.csr_view(), theta, x, 0.05,
                                          cmfb.SolverConfig("cg", precision="fp16"))
    assert np.array_equal(theta, th_before)            # fixed is read-only
    assert np.array_equal(x[120], x_before[120])       # empty row untouched
    assert not np.array_equal(x[:120], x_before[:120])
    # the fused tensor-core route reports one kernel under accumulate
    assert nbytes == 121 * 36 * 2 and brk == 0 and times.accumulate + times.solve > 0
    # device tensors: in place on the device, same numbers
    xd = torch.tensor(x_before, device=cuda_device)
    cmfb.update_side(sr.to_device().csr_view(), torch.tensor(theta, device=cuda_device), xd, 0.05,
                     cmfb.SolverConfig("cg", precision="fp16"))
    assert np.array_equal(xd.cpu().numpy(), x)
    with pytest.raises(cmfb.DataError):
        cmfb.update_side(sr.csr_view(), theta, x[:5], 0.05, cmfb.SolverConfig())


def test_row_blocking_is_invisible(cuda_device):
    sr, te = _protocol(400, 300, 20000, 16)
    theta = cmfb.init_factors(300, 16, 0.1, [0, 1])
    outs = []
    for ws in (None, 37 * (136 * 4 + 16 * 4 + 8)):
        x = cmfb.init_factors(400, 16, 0.1, [0, 0])
        cmfb.update_side(sr.csr_view(), theta, x, 0.05, cmfb.SolverConfig("exact"),
                         workspace_bytes=ws)
        outs.append(x)
    assert np.array_equal(outs[0], outs[1])


def test_objective_and_rmse_vs_oracle(oracle, cuda_device):
    sr, te = _protocol(200, 150, 5000, 8)
    x = cmfb.init_factors(200, 8, 0.3, [1, 0])
    t = cmfb.init_factors(150, 8, 0.3, [1, 1])
    r = oracle.ORatings(sr.m, sr.n, sr.nnz, sr.row_ptr, sr.col_idx, sr.csr_val, sr.col_ptr,
                        sr.row_idx, sr.csc_val)
    for w in (True, False):
        ours, ref = cmfb.objective(x, t, sr, 0.05, w), oracle.objective(x, t, r, 0.05, w)
        assert abs(ours - ref) <= 1e-9 * abs(ref)
    ours = cmfb.rmse(x, t, te)
    ref = oracle.rmse(x, t, oracle.OTriples(te.user, te.item, te.rating))
    assert abs(ours - ref) <= 1e-6 * ref
    assert np.allclose(cmfb.predict_pairs(x, t, te.user, te.item),
                       oracle.predict_pairs(x, t, te.user, te.item), rtol=1e-5, atol=1e-7)
    with pytest.raises(cmfb.DataError):
        cmfb.rmse(x, t, cmfb.Triples(np.zeros(0, np.int64), np.zeros(0, np.int64),
                                     np.zeros(0, np.float32)))


def test_update_side_streamed_pinned_matches_device(cuda_device):
    """update_side with pinned host buffers (the chunked, copy-overlapped path)
    gives the same factors as the device-resident call, bit for bit: each row's
    system is independent of the chunking."""
    import torch
    m, n, f = 6000, 900, 32
    t, _ = cmfb.gen_synthetic(m, n, f, 60000 / (m * n), 0.1, 9)
    sr = cmfb.build(t, m, n)
    theta = cmfb.init_factors(n, f, 0.1, [0, 1])
    x0 = cmfb.init_factors(m, f, 0.1, [0, 0])
    solver = cmfb.SolverConfig("cg", precision="fp16")
    v = sr.csr_view()
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    view_h = cmfb.RowView(pin(v.indptr), pin(v.indices), pin(v.values), v.nrows, v.ncols)
    x_h = pin(x0)
    cmfb.update_side(view_h, pin(theta), x_h, 0.05, solver, gram_kernel="tc")
    view_d = cmfb.RowView(*(torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (v.indptr, v.indices, v.values)),
                          v.nrows, v.ncols)
    x_d = torch.from_numpy(x0).cuda()
    cmfb.update_side(view_d, torch.from_numpy(theta).cuda(), x_d, 0.05, solver, gram_kernel="tc")
    assert torch.equal(x_h, x_d.cpu())

"""Pin the CPU oracle (oracle/) against golden vectors made by the reference.

CPU-only.  Where the reference is bitwise deterministic (numba Gram / bias /
CG, numpy build / RNG) the oracle must match bit for bit; where the reference
calls LAPACK (exact solve) it must match to float32 rounding.
"""

import numpy as np
import pytest


def _case(g, ci):
    p = f"c{ci}_"
    m, n, f = (int(v) for v in g[p + "meta"])
    csr = (g[p + "row_ptr"], g[p + "col_idx"], g[p + "csr_val"], m, n)
    csc = (g[p + "col_ptr"], g[p + "row_idx"], g[p + "csc_val"], n, m)
    return p, f, {"x": (csr, g[p + "theta_n"]), "t": (csc, g[p + "theta_m"])}


def test_gram_bitwise_vs_reference(golden, oracle):
    g = golden("gram_cases")
    checked = 0
    for ci in range(int(g["ncases"])):
        p, f, sides = _case(g, ci)
        for side, (view, th) in sides.items():
            for prec, wr in (("fp32", 1), ("fp32", 0), ("fp16", 1)):
                key = f"{p}{side}_{prec}_{wr}"
                if key + "_a" not in g:
                    continue
                a, b, nu = oracle.assemble_side(view[0], view[1], view[2], view[3], th, 0.05,
                                                prec, bool(wr))
                assert a.dtype == g[key + "_a"].dtype
                assert np.array_equal(a.view(np.uint8), g[key + "_a"].view(np.uint8)), key
                assert np.array_equal(b, g[key + "_b"]), key
                assert np.array_equal(nu, g[key + "_nu"]), key
                checked += 1
        (view, th) = sides["x"]
        a, b, _ = oracle.assemble_side(view[0], view[1], view[2], view[3], th, 0.05, "fp32",
                                       False, a_weights=g[p + "aw"], b_weights=g[p + "bw"],
                                       base_packed=g[p + "base"])
        assert np.array_equal(a, g[p + "impl_a"]) and np.array_equal(b, g[p + "impl_b"])
    assert checked >= 30


def test_pack_half_overflow_raises(golden, oracle):
    assert int(golden("gram_cases")["overflow_raises"]) == 1
    with pytest.raises(oracle.OracleNumericalError):
        oracle.pack_half(np.array([70000.0], np.float32))
    # boundary cases of the RNE converter vs numpy's cast (gram.py:140)
    cases = np.array([2.0 ** -15, 2.0 ** -24, 2.0 ** -25, 3e-8, 65504.0, 65519.0, -0.0,
                      1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11, 6.1e-5, 5.96e-8], np.float32)
    assert np.array_equal(oracle.pack_half(cases).view(np.uint16),
                          cases.astype(np.float16).view(np.uint16))
    rng = np.random.default_rng(9)
    x = ((1.0 + rng.random(20000)) * 2.0 ** rng.integers(-26, 16, 20000)
         * rng.choice([-1.0, 1.0], 20000)).astype(np.float32)
    assert np.array_equal(oracle.pack_half(x).view(np.uint16), x.astype(np.float16).view(np.uint16))


def test_cg_bitwise_vs_reference(golden, oracle):
    g = golden("solve_cases")
    for ci in range(int(g["nspecs"])):
        p = f"s{ci}_"
        a, b, x0 = g[p + "a"], g[p + "b"], g[p + "x0"]
        f = b.shape[1]
        for prec in ("fp32", "fp16"):
            aa = a if prec == "fp32" else a.astype(np.float16)
            for fs, tol in ((6, 1e-4), (f, 0.0), (1, 0.0)):
                key = f"{p}cg_{prec}_{fs}_{tol:g}"
                x, it, brk = oracle.batch_solve(aa, b, x0, "cg", fs, tol)
                assert np.array_equal(x, g[key + "_x"]), key
                assert np.array_equal(it, g[key + "_it"]), key
                assert brk == int(g[key + "_brk"])


def test_cg_breakdown_returns_iterate(golden, oracle):
    g = golden("solve_cases")
    x, it, brk = oracle.batch_solve(g["bd_a"], g["bd_b"], g["bd_x0"], "cg", 3, 0.0)
    assert np.array_equal(x, g["bd_x"]) and np.array_equal(it, g["bd_it"])
    assert brk == int(g["bd_brk"]) == 1
    assert np.array_equal(x[1], g["bd_x0"][1])


def test_exact_vs_reference_lapack(golden, oracle):
    g = golden("solve_cases")
    for ci in range(int(g["nspecs"])):
        p = f"s{ci}_"
        x, _, _ = oracle.batch_solve(g[p + "a"], g[p + "b"], g[p + "x0"], "exact")
        ref = g[p + "exact_x"]
        rel = np.abs(x - ref).max() / np.abs(ref).max()
        assert rel <= 2e-6, (p, rel)
    with pytest.raises(oracle.OracleSingularError) as e:
        oracle.batch_solve(g["sing_a"], np.ones((4, 3), np.float32), np.zeros((4, 3), np.float32),
                           "exact")
    assert e.value.rows == g["sing_rows"].tolist() == [1, 3]


def test_build_bitwise_vs_reference(golden, oracle):
    g = golden("build_cases")
    for ci in range(int(g["nspecs"])):
        p = f"b{ci}_"
        m, n = (int(v) for v in g[p + "dims"])
        r = oracle.build(oracle.OTriples(g[p + "u"], g[p + "v"], g[p + "r"]), m, n)
        for name in ("row_ptr", "col_idx", "csr_val", "col_ptr", "row_idx", "csc_val"):
            ours, ref = getattr(r, name), g[p + name]
            assert ours.dtype == ref.dtype and np.array_equal(ours, ref), (p, name)


def test_data_generation_bitwise(golden, oracle):
    g = golden("data_cases")
    t, xt, tt = oracle.gen_synthetic(50, 40, 4, 0.3, 0.1, 3)
    assert np.array_equal(t.user, g["gen_u"]) and np.array_equal(t.item, g["gen_v"])
    assert np.array_equal(t.rating, g["gen_r"])
    assert np.array_equal(xt, g["gen_xt"]) and np.array_equal(tt, g["gen_tt"])
    tr, te = oracle.split_holdout(t, 0.1, 1)
    assert np.array_equal(tr.user, g["tr_u"]) and np.array_equal(te.rating, g["te_r"])
    assert np.array_equal(oracle.init_factors(13, 5, 0.1, [0, 0]), g["init_x"])
    assert np.array_equal(oracle.init_factors(11, 5, 0.1, [0, 1]), g["init_t"])


def _small_protocol(oracle, g):
    m, n, nnz, f = (int(v) for v in g["meta"])
    t, _, _ = oracle.gen_synthetic(m, n, f, round(nnz / 0.9) / (m * n), 0.1, 0)
    tr, te = oracle.split_holdout(t, 0.1, 1)
    return oracle.build(tr, m, n), te, f


@pytest.mark.parametrize("solver", ["exact", "cg32", "cg16"])
def test_train_small_vs_reference(golden, oracle, solver):
    g = golden("train_small")
    r, te, f = _small_protocol(oracle, g)
    method = "exact" if solver == "exact" else "cg"
    prec = "fp16" if solver == "cg16" else "fp32"
    xs, ts = [], []
    _, _, hist = oracle.train(r, te, f=f, lam=0.05, epochs=5, method=method, precision=prec,
                              callback=lambda e, x, t: (xs.append(x.copy()), ts.append(t.copy())))
    X, T = np.stack(xs), np.stack(ts)
    if method == "cg":   # bitwise path end to end
        assert np.array_equal(X, g[solver + "_X"]) and np.array_equal(T, g[solver + "_T"])
    else:                # LAPACK vs unblocked Cholesky: float32 rounding only
        for e in range(5):
            rx = np.linalg.norm(X[e] - g["exact_X"][e]) / np.linalg.norm(g["exact_X"][e])
            rt = np.linalg.norm(T[e] - g["exact_T"][e]) / np.linalg.norm(g["exact_T"][e])
            assert rx < 1e-6 and rt < 1e-6, (e, rx, rt)
    rm = np.array([h["rmse"] for h in hist])
    assert np.abs(rm - g[solver + "_rmse"]).max() < 1e-6

"""K3/K4 on the GPU vs the reference's golden vectors.

Bars: accum="fp64" CG is bit-identical to solvers._cg_batch (x, iterations,
breakdowns); accum="fp32" CG within 1e-3 relative of the reference after
f_s=6 (the paper's mixed-precision design; the train-level bar is RMSE 1e-3);
Cholesky within 1e-6 (fp64) / 1e-4 x cond/100 (fp32) of LAPACK."""

import numpy as np
import pytest

import paper_1808_03843_b200 as cmfb

pytestmark = pytest.mark.gpu


def _batch(a, b):
    return cmfb.GramBatch(b.shape[1], a, b, np.ones(b.shape[0], np.int64))


def test_cg_fp64_bitwise_vs_reference(golden, cuda_device):
    g = golden("solve_cases")
    for ci in range(int(g["nspecs"])):
        p = f"s{ci}_"
        a, b, x0 = g[p + "a"], g[p + "b"], g[p + "x0"]
        f = b.shape[1]
        for prec in ("fp32", "fp16"):
            aa = a if prec == "fp32" else a.astype(np.float16)
            for fs, tol in ((6, 1e-4), (f, 0.0), (1, 0.0)):
                key = f"{p}cg_{prec}_{fs}_{tol:g}"
                r = cmfb.batch_solve(_batch(aa, b), x0,
                                     cmfb.SolverConfig("cg", fs, tol, prec, accum="fp64"))
                assert np.array_equal(r.x, g[key + "_x"]), key
                assert np.array_equal(r.iterations, g[key + "_it"]), key
                assert r.breakdowns == int(g[key + "_brk"])


def test_cg_fp32_close_to_reference(golden, cuda_device):
    g = golden("solve_cases")
    for ci in range(int(g["nspecs"])):
        p = f"s{ci}_"
        a, b, x0 = g[p + "a"], g[p + "b"], g[p + "x0"]
        for prec in ("fp32", "fp16"):
            aa = a if prec == "fp32" else a.astype(np.float16)
            key = f"{p}cg_{prec}_6_0.0001"
            r = cmfb.batch_solve(_batch(aa, b), x0, cmfb.SolverConfig("cg", 6, 1e-4, prec))
            ref = g[key + "_x"]
            rel = np.linalg.norm(r.x - ref, axis=1) / np.linalg.norm(ref, axis=1)
            assert rel.max() < 1e-3, (key, rel.max())


def test_cg_breakdown_and_known_answers(golden, cuda_device):
    g = golden("solve_cases")
    for accum in ("fp32", "fp64"):
        r = cmfb.batch_solve(_batch(g["bd_a"], g["bd_b"]), g["bd_x0"],
                             cmfb.SolverConfig("cg", 3, 0.0, accum=accum))
        assert r.breakdowns == 1
        assert np.array_equal(r.x[1], g["bd_x0"][1])
        assert np.allclose(r.x, g["bd_x"], rtol=1e-6 if accum == "fp64" else 1e-5)
    s = cmfb.GramSystem(2, cmfb.pack_lower(np.array([[4.0, 1.0], [1.0, 3.0]])),
                        np.array([1.0, 2.0], np.float32), 1)
    x = cmfb.cg_solve(s, np.array([2.0, 1.0], np.float32), f_s=2, eps=0.0)
    assert np.allclose(x, [1 / 11, 7 / 11], atol=1e-6)
    assert np.allclose(cmfb.exact_solve(s), [1 / 11, 7 / 11], atol=1e-6)
    eye = cmfb.GramSystem(5, cmfb.pack_lower(np.eye(5)), np.arange(1.0, 6.0, dtype=np.float32), 1)
    x, info = cmfb.cg_solve(eye, np.zeros(5, np.float32), f_s=5, eps=0.0, return_info=True)
    assert np.allclose(x, np.arange(1.0, 6.0)) and info["iterations"] >= 1
    half = cmfb.GramSystem(5, cmfb.pack_half(cmfb.pack_lower(np.eye(5))), eye.b, 1)
    assert np.array_equal(cmfb.cg_solve_half(half, np.zeros(5, np.float32), f_s=5, eps=0.0),
                          cmfb.cg_solve(eye, np.zeros(5, np.float32), f_s=5, eps=0.0))
    with pytest.raises(cmfb.DataError, match="fp16"):
        cmfb.cg_solve_half(eye, np.zeros(5, np.float32))
    with pytest.raises(cmfb.DataError, match="fp32"):
        cmfb.exact_solve(half)


def test_exact_vs_reference_lapack(golden, cuda_device):
    g = golden("solve_cases")
    conds = [100.0, 50.0, 1000.0, 5.0, 20.0]
    for ci in range(int(g["nspecs"])):
        p = f"s{ci}_"
        ref = g[p + "exact_x"]
        for accum, tol in (("fp64", 1e-6), ("fp32", 1e-4 * max(conds[ci] / 100, 1.0))):
            r = cmfb.batch_solve(_batch(g[p + "a"], g[p + "b"]), g[p + "x0"],
                                 cmfb.SolverConfig("exact", accum=accum))
            rel = np.abs(r.x - ref).max() / np.abs(ref).max()
            assert rel <= tol, (p, accum, rel)
            assert np.array_equal(r.iterations, np.zeros(len(ref), np.int64))


def test_exact_singular_rows_aggregated(golden, cuda_device):
    g = golden("solve_cases")
    with pytest.raises(cmfb.SingularSystemError) as e:
        cmfb.batch_solve(_batch(g["sing_a"], np.ones((4, 3), np.float32)),
                         np.zeros((4, 3), np.float32), cmfb.SolverConfig("exact"))
    assert e.value.rows == g["sing_rows"].tolist() == [1, 3]
    z = cmfb.GramSystem(3, cmfb.pack_lower(np.zeros((3, 3))), np.ones(3, np.float32), 1)
    with pytest.raises(cmfb.SingularSystemError):
        cmfb.exact_solve(z)


def test_random_f100_residual_and_cg_exactness(cuda_device):
    rng = np.random.default_rng(5)
    q, _ = np.linalg.qr(rng.standard_normal((100, 100)))
    a = (q * np.geomspace(1.0, 50.0, 100)) @ q.T
    b = rng.standard_normal(100)
    s = cmfb.GramSystem(100, cmfb.pack_lower(a), b.astype(np.float32), 1)
    x = cmfb.exact_solve(s).astype(np.float64)
    full = s.full().astype(np.float64)
    assert np.linalg.norm(full @ x - b) / np.linalg.norm(b) <= 1e-5
    xc = cmfb.cg_solve(s, np.zeros(100, np.float32), f_s=100, eps=0.0)
    assert np.linalg.norm(xc - x) / np.linalg.norm(x) <= 1e-4


def test_batch_validation(cuda_device):
    s = cmfb.GramSystem(3, cmfb.pack_lower(np.eye(3)), np.ones(3, np.float32), 1)
    with pytest.raises(cmfb.DataError):
        cmfb.batch_solve([s, s], np.zeros((3, 3), np.float32), cmfb.SolverConfig())
    h = cmfb.GramSystem(3, cmfb.pack_half(cmfb.pack_lower(np.eye(3))), np.ones(3, np.float32), 1)
    with pytest.raises(cmfb.DataError):
        cmfb.batch_solve([h], np.zeros((1, 3), np.float32), cmfb.SolverConfig("exact"))


@pytest.mark.parametrize("f", [1, 3, 4, 5, 7, 8, 31, 64, 97, 100, 113, 127, 128])
def test_batched_cholesky_sizes(cuda_device, f):
    """The shared-memory tile Cholesky (f <= 128) at every padding case (f % 4),
    single-tile and full-width systems, with a non-SPD system in the batch: it is
    reported (rows) while every other system is solved to fp32 accuracy."""
    rng = np.random.default_rng(f)
    nsys = 40
    a_list, b = [], rng.standard_normal((nsys, f)).astype(np.float32)
    for s in range(nsys):
        q, _ = np.linalg.qr(rng.standard_normal((f, f)))
        a_list.append((q * np.geomspace(1.0, 30.0, f)) @ q.T)
    packed = np.stack([cmfb.pack_lower(a) for a in a_list]).astype(np.float32)
    r = cmfb.batch_solve(_batch(packed, b), np.zeros((nsys, f), np.float32), cmfb.SolverConfig("exact"))
    for s in range(nsys):
        full = cmfb.unpack_lower(packed[s].astype(np.float64), f)
        ref = np.linalg.solve(full, b[s].astype(np.float64))
        assert np.linalg.norm(r.x[s] - ref) / np.linalg.norm(ref) <= 1e-5 * 30, (f, s)
    bad = packed.copy()
    bad[7] = cmfb.pack_lower(-np.eye(f)).astype(np.float32)
    with pytest.raises(cmfb.SingularSystemError) as e:
        cmfb.batch_solve(_batch(bad, b), np.zeros((nsys, f), np.float32), cmfb.SolverConfig("exact"))
    assert e.value.rows == [7]

"""K1/K2 on the GPU vs the reference's golden vectors and the CPU oracle.

Bar: the "bitwise" kernel is bit-identical to the reference (fp32 and fp16
stores, bias, n_u); the "fma" kernel is within 1e-5 relative Frobenius (the
reference's own oracle-grid tolerance, test_gram.py:64-81)."""

import numpy as np
import pytest
import torch

import paper_1808_03843_b200 as cmfb
from paper_1808_03843_b200.data import RowView

pytestmark = pytest.mark.gpu


def _views(g, ci):
    p = f"c{ci}_"
    m, n, f = (int(v) for v in g[p + "meta"])
    return p, f, {"x": (RowView(g[p + "row_ptr"], g[p + "col_idx"], g[p + "csr_val"], m, n),
                        g[p + "theta_n"]),
                  "t": (RowView(g[p + "col_ptr"], g[p + "row_idx"], g[p + "csc_val"], n, m),
                        g[p + "theta_m"])}


def test_bitwise_kernel_equals_reference(golden, cuda_device):
    g = golden("gram_cases")
    checked = 0
    for ci in range(int(g["ncases"])):
        p, f, views = _views(g, ci)
        for side, (view, th) in views.items():
            for prec, wr in (("fp32", 1), ("fp32", 0), ("fp16", 1)):
                key = f"{p}{side}_{prec}_{wr}"
                if key + "_a" not in g:
                    continue
                gb, times = cmfb.assemble_side(view, th, 0.05, precision=prec,
                                               weighted_reg=bool(wr), kernel="bitwise")
                ref = g[key + "_a"]
                assert gb.a_lower.dtype == ref.dtype
                assert np.array_equal(gb.a_lower.view(np.uint8), ref.view(np.uint8)), key
                assert np.array_equal(gb.b, g[key + "_b"]), key
                assert np.array_equal(gb.n_u, g[key + "_nu"]), key
                assert gb.a_nbytes == ref.nbytes
                assert times.accumulate >= 0.0
                checked += 1
        view, th = views["x"]
        gb, _ = cmfb.assemble_side(view, th, 0.05, weighted_reg=False, a_weights=g[p + "aw"],
                                   b_weights=g[p + "bw"], base_packed=g[p + "base"],
                                   kernel="bitwise")
        assert np.array_equal(gb.a_lower, g[p + "impl_a"]), p
        assert np.array_equal(gb.b, g[p + "impl_b"]), p
    assert checked >= 30


def test_fma_kernel_within_oracle_grid_tolerance(golden, cuda_device):
    g = golden("gram_cases")
    for ci in range(int(g["ncases"])):
        p, f, views = _views(g, ci)
        for side, (view, th) in views.items():
            key = f"{p}{side}_fp32_1"
            gb, _ = cmfb.assemble_side(view, th, 0.05, kernel="fma")
            ref = g[key + "_a"].astype(np.float64)
            for u in range(ref.shape[0]):
                d = np.linalg.norm(gb.a_lower[u] - ref[u]) / max(np.linalg.norm(ref[u]), 1e-30)
                assert d < 1e-5, (key, u, d)
            assert np.array_equal(gb.b, g[key + "_b"])


@pytest.mark.parametrize("f,deg", [(100, 3000), (32, 700), (100, 206), (64, 1)])
def test_heavy_rows_bitwise_vs_oracle(oracle, cuda_device, f, deg):
    rng = np.random.default_rng(f + deg)
    m, n = 9, max(deg + 50, 300)
    rows = [np.sort(rng.choice(n, size=deg if u % 3 else max(deg // 3, 1), replace=False))
            for u in range(m)]
    indptr = np.zeros(m + 1, np.int64)
    indptr[1:] = np.cumsum([len(r) for r in rows])
    indices = np.concatenate(rows).astype(np.int32)
    values = rng.standard_normal(indices.shape[0]).astype(np.float32)
    theta = (rng.random((n, f), dtype=np.float32) - 0.5)
    view = RowView(indptr, indices, values, m, n)
    for prec in ("fp32", "fp16"):
        gb, _ = cmfb.assemble_side(view, theta, 0.05, precision=prec, kernel="bitwise")
        a, b, nu = oracle.assemble_side(indptr, indices, values, m, theta, 0.05, prec)
        assert np.array_equal(gb.a_lower.view(np.uint8), a.view(np.uint8))
        assert np.array_equal(gb.b, b) and np.array_equal(gb.n_u, nu)


def test_device_tensors_stay_on_device(cuda_device):
    rng = np.random.default_rng(1)
    sr = cmfb.build([(0, 0, 1.0), (0, 2, 2.0), (1, 1, 3.0)], 2, 3)
    th = torch.tensor(rng.standard_normal((3, 8)), dtype=torch.float32, device=cuda_device)
    view = sr.to_device().csr_view()
    gb, _ = cmfb.assemble_side(view, th, 0.1, precision="fp16", kernel="fma")
    assert gb.a_lower.is_cuda and gb.a_lower.dtype == torch.float16
    assert gb.a_nbytes == 2 * 36 * 2


def test_known_answers(cuda_device):
    sr = cmfb.build([(0, 0, 1.0)], 1, 3)
    s = cmfb.get_hermitian(sr, 0, np.eye(3, dtype=np.float32), 0.05)
    assert np.allclose(s.full(), np.diag([1.05, 0.05, 0.05]), atol=1e-7) and s.n_u == 1
    sr = cmfb.build([(0, 0, 1.0), (0, 1, 1.0)], 1, 2)
    z = np.zeros((2, 2), np.float32)
    assert np.allclose(np.diag(cmfb.get_hermitian(sr, 0, z, 0.5).full()), 1.0)
    assert np.allclose(np.diag(cmfb.get_hermitian(sr, 0, z, 0.5, weighted_reg=False).full()), 0.5)
    sr = cmfb.build([(1, 0, 1.0)], 2, 2)
    assert cmfb.get_hermitian(sr, 0, np.ones((2, 2), np.float32), 0.05).is_empty
    sr = cmfb.build([(0, 0, 2.0)], 1, 1)
    assert np.allclose(cmfb.get_bias(sr, 0, np.array([[1.0, 0.0, 1.0]], np.float32)), [2, 0, 2])
    sr = cmfb.build([(1, 0, 1.0)], 2, 3)
    assert np.array_equal(cmfb.get_bias(sr, 0, np.ones((3, 4), np.float32)), np.zeros(4))


def test_pack_half_and_overflow(golden, cuda_device):
    rng = np.random.default_rng(9)
    x = ((1.0 + rng.random(50000)) * 2.0 ** rng.integers(-26, 16, 50000)
         * rng.choice([-1.0, 1.0], 50000)).astype(np.float32)
    assert np.array_equal(cmfb.pack_half(x).view(np.uint16), x.astype(np.float16).view(np.uint16))
    with pytest.raises(cmfb.NumericalError, match="rescale"):
        cmfb.pack_half(np.array([70000.0], np.float32))
    sr = cmfb.build([(0, 0, 1.0)], 1, 1)
    with pytest.raises(cmfb.NumericalError, match="rescale"):
        cmfb.assemble_side(sr.csr_view(), np.full((1, 1), 300.0, np.float32), 0.0,
                           precision="fp16")


def test_bad_inputs_raise_data_error(cuda_device):
    sr = cmfb.build([(0, 0, 1.0)], 1, 2)
    with pytest.raises(cmfb.DataError, match="feature matrix"):
        cmfb.assemble_side(sr.csr_view(), np.ones((3, 4), np.float32), 0.1)
    with pytest.raises(cmfb.DataError):
        cmfb.assemble_side(sr.csr_view(), np.ones((2, 4), np.float32), 0.1, precision="bf16")
    with pytest.raises(cmfb.DataError):
        cmfb.assemble_side(sr.csr_view(), np.ones((2, 4), np.float32), 0.1,
                           base_packed=np.ones(3, np.float32))

"""CPU-only: the C-ABI library loads and exports every symbol the header
declares; host-side logic (config validation, report schema, flop model,
input generation) matches the reference."""

import os
import re

import numpy as np
import pytest
import torch

import paper_1808_03843_b200 as cmfb
from paper_1808_03843_b200 import _native

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "cmf_b200.h")


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(cmf_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = _native.load_library()
    decl = header_functions()
    assert len(decl) >= 13
    for name in decl:
        assert hasattr(lib, name), name
    assert sorted(_native.EXPORTED) == decl
    assert lib.cmf_version() == 1


def test_status_codes_map_to_reference_errors():
    _native.load_library()
    with pytest.raises(cmfb.DataError):
        _native.check(_native.CMF_EINVAL)
    with pytest.raises(cmfb.NumericalError):
        _native.check(_native.CMF_EOVERFLOW)
    with pytest.raises(cmfb.SingularSystemError):
        _native.check(_native.CMF_ESINGULAR)
    with pytest.raises(cmfb.CmfError):
        _native.check(_native.CMF_ECUDA)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    with pytest.raises(cmfb.CmfError, match="no CPU fallback"):
        cmfb.pack_half(np.ones(4, np.float32))


def test_solver_config_validation():
    for bad in (dict(method="lu"), dict(method="cg", cg_iters=0), dict(cg_tol=-1.0),
                dict(precision="bf16"), dict(method="exact", precision="fp16"),
                dict(accum="fp16")):
        with pytest.raises(cmfb.DataError):
            cmfb.SolverConfig(**bad)
    with pytest.raises(cmfb.DataError):
        cmfb.TileConfig(tile=0)
    with pytest.raises(cmfb.DataError):
        cmfb.AlsConfig(f=0)


def test_roofline_conventions():
    est = cmfb.roofline_estimate(480189, 17770, 99_000_000, 100)
    assert est["hermitian_flops"] == 2 * 99_000_000 * 5050
    assert est["hermitian_cm_ratio"] == 100.0
    r = cmfb.roofline_estimate(10_000, 10_000, 10_000, 100, f_s=6)
    assert r["solve_flops_cg"] / r["solve_flops_exact"] == pytest.approx(0.126, abs=1e-3)
    with pytest.raises(cmfb.DataError):
        cmfb.roofline_estimate(0, 1, 1, 1)


def test_packed_layout_roundtrip():
    rng = np.random.default_rng(0)
    a = rng.standard_normal((7, 7)).astype(np.float32)
    a = a + a.T
    p = cmfb.pack_lower(a)
    assert p.shape == (28,) and p[2 * 3 // 2 + 1] == a[2, 1]
    assert p[5 * 6 // 2 + 3] == a[5, 3]
    assert np.array_equal(cmfb.unpack_lower(p, 7), a)
    assert cmfb.packed_size(100) == 5050


def test_report_jsonl_roundtrip(tmp_path):
    rep = cmfb.TrainReport(engine="als", config={"f": 4}, cold_rows=1, flops={"x": 2})
    t = cmfb.PhaseTimes(accumulate=1.0, solve=0.5)
    t += cmfb.PhaseTimes(eval=0.25)
    rep.add_epoch(cmfb.EpochRecord.from_phases(0, 3.0, t, rmse=0.5, cg_breakdowns=2))
    path = tmp_path / "r.jsonl"
    rep.save(path)
    back = cmfb.TrainReport.load(path)
    assert back.epochs_run == 1 and back.final_rmse == 0.5 and back.cold_rows == 1
    assert back.epochs[0].epoch_time == pytest.approx(1.75)
    assert t.hermitian == 1.0


def test_host_generation_matches_reference(golden):
    g = golden("data_cases")
    t, truth = cmfb.gen_synthetic(50, 40, 4, 0.3, 0.1, 3)
    assert np.array_equal(t.user, g["gen_u"]) and np.array_equal(t.rating, g["gen_r"])
    assert np.array_equal(truth.x_true, g["gen_xt"])
    tr, te = cmfb.split_holdout(t, 0.1, 1)
    assert np.array_equal(tr.item, g["tr_v"]) and np.array_equal(te.user, g["te_u"])
    assert np.array_equal(cmfb.init_factors(13, 5, 0.1, [0, 0]), g["init_x"])
    assert np.array_equal(cmfb.init_factors(11, 5, 0.1, [0, 1]), g["init_t"])
    with pytest.raises(cmfb.DataError):
        cmfb.split_holdout(t, 1.5, 0)


def test_model_file_roundtrip(tmp_path):
    x = np.arange(12, dtype=np.float32).reshape(3, 4)
    t = -np.arange(8, dtype=np.float32).reshape(2, 4)
    cmfb.save_model(tmp_path / "m.cmfm", x, t)
    x2, t2 = cmfb.load_model(tmp_path / "m.cmfm")
    assert np.array_equal(x, x2) and np.array_equal(t, t2)
    (tmp_path / "bad").write_bytes(b"XXXX")
    with pytest.raises(cmfb.FormatError):
        cmfb.load_model(tmp_path / "bad")


def test_implicit_config_validation():
    import paper_1808_03843_b200 as cmfb
    for kw in ({"f": 0}, {"alpha": 0.0}, {"lam": -1.0}, {"epochs": 0}):
        with pytest.raises(cmfb.DataError):
            cmfb.ImplicitConfig(**kw)
    c = cmfb.ImplicitConfig()
    assert (c.f, c.alpha, c.lam, c.epochs) == (100, 40.0, 0.05, 10)


def test_worker_knob_matches_reference_api():
    # parallel.py:11-27: >= 1, clamped, returned; results never depend on it
    assert cmfb.set_workers(1) == 1 and cmfb.get_workers() == 1
    n = cmfb.set_workers(10 ** 6)
    assert n == cmfb.get_workers() == (os.cpu_count() or 1)
    with pytest.raises(ValueError):
        cmfb.set_workers(0)


def test_accum_auto_resolves_per_boundary():
    from paper_1808_03843_b200.solvers import with_accum
    cfg = cmfb.SolverConfig("cg", precision="fp16")
    assert cfg.accum == "auto"
    assert with_accum(cfg, "fp64").accum == "fp64"
    assert with_accum(cmfb.SolverConfig("cg", accum="fp32"), "fp64").accum == "fp32"

"""Generate the golden fixtures in tests/golden/ from the REFERENCE package.

Run here (the container that has /root/reference):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to a scratch directory (numba's cache=True writes
next to the sources and the mount is read-only), imports ``cmf`` from there and
records the reference's own outputs on seeded inputs.  The .npz files it writes
are committed; nothing on the GPU box ever reads /root/reference.

Fixtures:
  gram_cases.npz    assemble_side on random CSR/CSC views (fp32 + fp16, weighted
                    and plain lambda, implicit-style weights + base matrix)
  solve_cases.npz   batch_solve / cg_solve on random SPD batches (cg fp32/fp16,
                    exact), incl. breakdown and singular rows
  build_cases.npz   build() on random triples with duplicates and empty rows
  data_cases.npz    gen_synthetic / split_holdout / init_factors draws
  train_small.npz   full train() trajectories (X, Theta per epoch) on a small
                    instance for exact / cg-fp32 / cg-fp16
  implicit_small.npz  implicit_train (reference implicit.py) on a small
                    non-negative instance: X, Theta, objectives and preference
                    RMSE per epoch (exact, cg-fp32), one
                    implicit_update_side and precompute_gram, mean percentile rank
  io_cases.npz      file formats: the bytes of the reference's save_cache (CMFR)
                    and save_coo (tsv, csv) for a small instance with duplicates,
                    and its parse_coo of a text with comments / blank lines
  train_f100.npz    1/10-Netflix shape at f=100 (48,019 x 17,770, 9.9M train
                    ratings): the same records as train_ml1m for exact / cg32 /
                    cg16 (run on demand: `make_golden.py f100`, ~40 min here)
  implicit100.npz   implicit_train at f = 100 (3,000 x 1,500, 148K ratings): cg16
                    and exact objective / RMSE per epoch, one cg16
                    implicit_update_side per side (`make_golden.py implicit100`)
  train_ml1m.npz    MovieLens-1M-shaped protocol (BASELINE configs[0]): RMSE and
                    objective per epoch for exact / cg-fp32 / cg-fp16, sampled
                    factor rows per epoch (exact), and SHA-256 digests of the
                    CSR/CSC arrays the reference builds
"""

import hashlib
import os
import shutil
import sys
import tempfile

import numpy as np

OUT = os.path.dirname(os.path.abspath(__file__))


def import_reference():
    src = "/root/reference/pkg"
    scratch = os.path.join(tempfile.gettempdir(), "cmf_ref_golden")
    if not os.path.isdir(scratch):
        shutil.copytree(src, scratch)
    sys.path.insert(0, os.path.join(scratch, "src"))
    import cmf  # noqa: E402
    return cmf


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def random_view(cmf, m, n, density, seed, f, dup=False):
    rng = np.random.default_rng(seed)
    k = max(int(density * m * n), 1)
    flat = rng.choice(m * n, size=k, replace=False)
    vals = rng.standard_normal(k).astype(np.float32)
    t = cmf.Triples((flat // n).astype(np.int64), (flat % n).astype(np.int64), vals)
    theta_n = rng.standard_normal((n, f)).astype(np.float32)
    theta_m = rng.standard_normal((m, f)).astype(np.float32)
    return cmf.build(t, m, n), theta_n, theta_m


def gram_cases(cmf):
    from cmf.gram import assemble_side
    out = {}
    specs = [  # (m, n, density, seed, f)
        (7, 5, 0.5, 1, 1), (20, 30, 0.3, 2, 3), (50, 70, 0.25, 7, 19),
        (40, 33, 0.2, 3, 32), (8, 24, 0.5, 4, 100), (6, 120, 0.9, 5, 64),
        (30, 20, 0.0, 6, 8),
    ]
    for ci, (m, n, d, seed, f) in enumerate(specs):
        sr, th_n, th_m = random_view(cmf, m, n, d, seed, f)
        rng = np.random.default_rng(1000 + ci)
        aw = rng.random(sr.nnz).astype(np.float32) * 3
        bw = 1 + rng.random(sr.nnz).astype(np.float32)
        base = cmf.pack_lower((th_n.T @ th_n).astype(np.float32))
        p = f"c{ci}_"
        out[p + "meta"] = np.array([m, n, f], np.int64)
        for name, a in (("row_ptr", sr.row_ptr), ("col_idx", sr.col_idx),
                        ("csr_val", sr.csr_val), ("col_ptr", sr.col_ptr),
                        ("row_idx", sr.row_idx), ("csc_val", sr.csc_val)):
            out[p + name] = a
        out[p + "theta_n"], out[p + "theta_m"] = th_n, th_m
        out[p + "aw"], out[p + "bw"], out[p + "base"] = aw, bw, base
        for side, view, th in (("x", sr.csr_view(), th_n), ("t", sr.csc_view(), th_m)):
            for prec, wr in (("fp32", True), ("fp32", False), ("fp16", True)):
                if side == "t" and (prec, wr) == ("fp32", False):
                    continue
                try:
                    gb, _ = assemble_side(view, th, 0.05, precision=prec, weighted_reg=wr)
                except cmf.NumericalError:
                    continue
                key = f"{p}{side}_{prec}_{int(wr)}"
                out[key + "_a"], out[key + "_b"], out[key + "_nu"] = gb.a_lower, gb.b, gb.n_u
            if side == "x":  # implicit-style call (implicit.py:74-79)
                gb, _ = assemble_side(view, th, 0.05, weighted_reg=False, a_weights=aw,
                                      b_weights=bw, base_packed=base)
                out[p + "impl_a"], out[p + "impl_b"] = gb.a_lower, gb.b
    # fp16 overflow must raise (gram.py:139-145)
    sr = cmf.build([(0, 0, 1.0)], 1, 1)
    big = np.full((1, 1), 300.0, np.float32)
    try:
        assemble_side(sr.csr_view(), big, 0.0, precision="fp16")
        out["overflow_raises"] = np.array(0)
    except cmf.NumericalError:
        out["overflow_raises"] = np.array(1)
    out["ncases"] = np.array(len(specs))
    np.savez_compressed(os.path.join(OUT, "gram_cases.npz"), **out)


def rand_spd(f, cond, rng):
    q, _ = np.linalg.qr(rng.standard_normal((f, f)))
    return (q * np.geomspace(1.0, cond, f)) @ q.T


def solve_cases(cmf):
    out = {}
    rng = np.random.default_rng(77)
    specs = [(64, 12, 100.0), (12, 100, 50.0), (25, 32, 1000.0), (10, 3, 5.0), (6, 128, 20.0)]
    for ci, (ns, f, cond) in enumerate(specs):
        a = np.stack([cmf.pack_lower(rand_spd(f, cond, rng).astype(np.float32))
                      for _ in range(ns)])
        b = rng.standard_normal((ns, f)).astype(np.float32)
        x0 = (0.1 * rng.standard_normal((ns, f))).astype(np.float32)
        p = f"s{ci}_"
        out[p + "a"], out[p + "b"], out[p + "x0"] = a, b, x0
        nu = np.ones(ns, np.int64)
        for prec in ("fp32", "fp16"):
            aa = a if prec == "fp32" else a.astype(np.float16)
            gb = cmf.GramBatch(f, aa, b, nu)
            for fs, tol in ((6, 1e-4), (f, 0.0), (1, 0.0)):
                r = cmf.batch_solve(gb, x0, cmf.SolverConfig("cg", fs, tol, prec))
                key = f"{p}cg_{prec}_{fs}_{tol:g}"
                out[key + "_x"], out[key + "_it"] = r.x, r.iterations
                out[key + "_brk"] = np.array(r.breakdowns)
        r = cmf.batch_solve(cmf.GramBatch(f, a, b, nu), x0, cmf.SolverConfig("exact"))
        out[p + "exact_x"] = r.x
    # breakdown case: negative definite among SPD rows
    f = 3
    a = np.stack([cmf.pack_lower(np.eye(3, dtype=np.float32)),
                  cmf.pack_lower(-np.eye(3, dtype=np.float32)),
                  cmf.pack_lower(np.diag([4.0, 2.0, 1.0]).astype(np.float32))])
    b = np.ones((3, 3), np.float32)
    x0 = np.full((3, 3), 5.0, np.float32)
    r = cmf.batch_solve(cmf.GramBatch(f, a, b, np.ones(3, np.int64)), x0,
                        cmf.SolverConfig("cg", 3, 0.0))
    out["bd_a"], out["bd_b"], out["bd_x0"] = a, b, x0
    out["bd_x"], out["bd_it"], out["bd_brk"] = r.x, r.iterations, np.array(r.breakdowns)
    # singular rows for exact (test_solvers.py:229-235 pattern)
    good = cmf.pack_lower(np.eye(3, dtype=np.float32))
    bad = cmf.pack_lower(np.zeros((3, 3), np.float32))
    a = np.stack([good, bad, good, bad])
    try:
        cmf.batch_solve(cmf.GramBatch(3, a, np.ones((4, 3), np.float32), np.ones(4, np.int64)),
                        np.zeros((4, 3), np.float32), cmf.SolverConfig("exact"))
        out["sing_rows"] = np.array([], np.int64)
    except cmf.SingularSystemError as e:
        out["sing_rows"] = np.array(e.rows, np.int64)
    out["sing_a"] = a
    out["nspecs"] = np.array(len(specs))
    np.savez_compressed(os.path.join(OUT, "solve_cases.npz"), **out)


def build_cases(cmf):
    out = {}
    rng = np.random.default_rng(11)
    specs = [(100, 80, 500), (40, 30, 400), (5, 5, 1), (1000, 300, 20000), (3, 7, 0)]
    for ci, (m, n, k) in enumerate(specs):
        u = rng.integers(0, m, k).astype(np.int64)
        v = rng.integers(0, n, k).astype(np.int64)
        r = rng.standard_normal(k).astype(np.float32)
        sr = cmf.build(cmf.Triples(u, v, r), m, n)
        p = f"b{ci}_"
        out[p + "dims"] = np.array([m, n])
        out[p + "u"], out[p + "v"], out[p + "r"] = u, v, r
        for name in ("row_ptr", "col_idx", "csr_val", "col_ptr", "row_idx", "csc_val"):
            out[p + name] = getattr(sr, name)
    out["nspecs"] = np.array(len(specs))
    np.savez_compressed(os.path.join(OUT, "build_cases.npz"), **out)


def data_cases(cmf):
    out = {}
    t, truth = cmf.gen_synthetic(50, 40, 4, 0.3, 0.1, 3)
    out["gen_u"], out["gen_v"], out["gen_r"] = t.user, t.item, t.rating
    out["gen_xt"], out["gen_tt"] = truth.x_true, truth.theta_true
    tr, te = cmf.split_holdout(t, 0.1, 1)
    out["tr_u"], out["tr_v"], out["tr_r"] = tr.user, tr.item, tr.rating
    out["te_u"], out["te_v"], out["te_r"] = te.user, te.item, te.rating
    out["init_x"] = cmf.init_factors(13, 5, 0.1, [0, 0])
    out["init_t"] = cmf.init_factors(11, 5, 0.1, [0, 1])
    np.savez_compressed(os.path.join(OUT, "data_cases.npz"), **out)


def protocol(cmf, m, n, nnz, f, seed=0):
    """total=round(nnz/0.9), gen(seed, sigma=0.1), split(0.1, 1), build."""
    total = round(nnz / 0.9)
    t, _ = cmf.gen_synthetic(m, n, f, total / (m * n), 0.1, seed)
    tr, te = cmf.split_holdout(t, 0.1, 1)
    return cmf.build(tr, m, n), te


def train_small(cmf):
    out = {}
    m, n, nnz, f = 300, 200, 6000, 8
    sr, te = protocol(cmf, m, n, nnz, f)
    out["meta"] = np.array([m, n, nnz, f])
    for name, cfg in (("exact", cmf.SolverConfig("exact")),
                      ("cg32", cmf.SolverConfig("cg", 6, 1e-4, "fp32")),
                      ("cg16", cmf.SolverConfig("cg", 6, 1e-4, "fp16"))):
        xs, ts = [], []
        import cmf.als as als
        orig = als.update_side

        def spy(view, fixed, target, *a, **k):
            r = orig(view, fixed, target, *a, **k)
            (xs if target.shape[0] == m else ts).append(target.copy())
            return r
        als.update_side = spy
        try:
            _, _, rep = cmf.train(sr, te, cmf.AlsConfig(f=f, lam=0.05, epochs=5, solver=cfg))
        finally:
            als.update_side = orig
        out[name + "_X"] = np.stack(xs)
        out[name + "_T"] = np.stack(ts)
        out[name + "_rmse"] = np.array(rep.rmse_trajectory())
        out[name + "_obj"] = np.array([e.objective for e in rep.epochs])
        out[name + "_objmid"] = np.array([e.objective_mid for e in rep.epochs])
    out["digest"] = np.array(digest(sr.row_ptr, sr.col_idx, sr.csr_val,
                                    sr.col_ptr, sr.row_idx, sr.csc_val))
    np.savez_compressed(os.path.join(OUT, "train_small.npz"), **out)


def train_ml1m(cmf):
    out = {}
    m, n, nnz, f = 6040, 3706, 1_000_000, 32
    sr, te = protocol(cmf, m, n, nnz, f)
    out["meta"] = np.array([m, n, nnz, f])
    out["csr_digest"] = np.array(digest(sr.row_ptr, sr.col_idx, sr.csr_val))
    out["csc_digest"] = np.array(digest(sr.col_ptr, sr.row_idx, sr.csc_val))
    out["test_digest"] = np.array(digest(te.user, te.item, te.rating))
    rng = np.random.default_rng(5)
    rows_x = np.sort(rng.choice(m, 128, replace=False))
    rows_t = np.sort(rng.choice(n, 128, replace=False))
    out["rows_x"], out["rows_t"] = rows_x, rows_t
    import cmf.als as als
    orig = als.update_side
    for name, cfg in (("exact", cmf.SolverConfig("exact")),
                      ("cg32", cmf.SolverConfig("cg", 6, 1e-4, "fp32")),
                      ("cg16", cmf.SolverConfig("cg", 6, 1e-4, "fp16"))):
        xs, ts, xn, tn = [], [], [], []

        def spy(view, fixed, target, *a, **k):
            r = orig(view, fixed, target, *a, **k)
            if target.shape[0] == m:
                xs.append(target[rows_x].copy())
                xn.append(np.linalg.norm(target.astype(np.float64)))
            else:
                ts.append(target[rows_t].copy())
                tn.append(np.linalg.norm(target.astype(np.float64)))
            return r
        als.update_side = spy
        try:
            _, _, rep = cmf.train(sr, te, cmf.AlsConfig(f=f, lam=0.05, epochs=10, solver=cfg))
        finally:
            als.update_side = orig
        out[name + "_rmse"] = np.array(rep.rmse_trajectory())
        out[name + "_obj"] = np.array([e.objective for e in rep.epochs])
        out[name + "_Xrows"], out[name + "_Trows"] = np.stack(xs), np.stack(ts)
        out[name + "_Xnorm"], out[name + "_Tnorm"] = np.array(xn), np.array(tn)
        print(name, out[name + "_rmse"])
    np.savez_compressed(os.path.join(OUT, "train_ml1m.npz"), **out)


def train_f100(cmf):
    """1/10-Netflix shape at the headline width (VERDICT r1 "next" #1): 48,019 x
    17,770, 9.9M train ratings, f=100, SURVEY 8(d) protocol, 10 epochs of the
    reference's train() for exact / cg32 / cg16.  Records per-epoch RMSE and
    objective, sampled factor rows and full-matrix norms after every half-update,
    and digests of the inputs (so the GPU test proves it regenerated them)."""
    import time
    out = {}
    m, n, nnz, f = 48_019, 17_770, 9_900_000, 100
    t0 = time.time()
    sr, te = protocol(cmf, m, n, nnz, f)
    print("f100 data", time.time() - t0, "s", flush=True)
    out["meta"] = np.array([m, n, nnz, f])
    out["csr_digest"] = np.array(digest(sr.row_ptr, sr.col_idx, sr.csr_val))
    out["csc_digest"] = np.array(digest(sr.col_ptr, sr.row_idx, sr.csc_val))
    out["test_digest"] = np.array(digest(te.user, te.item, te.rating))
    rng = np.random.default_rng(7)
    rows_x = np.sort(rng.choice(m, 256, replace=False))
    rows_t = np.sort(rng.choice(n, 256, replace=False))
    out["rows_x"], out["rows_t"] = rows_x, rows_t
    import cmf.als as als
    orig = als.update_side
    which = os.environ.get("F100_SOLVERS", "exact,cg32,cg16").split(",")
    cfgs = {"exact": cmf.SolverConfig("exact"),
            "cg32": cmf.SolverConfig("cg", 6, 1e-4, "fp32"),
            "cg16": cmf.SolverConfig("cg", 6, 1e-4, "fp16")}
    path = os.path.join(OUT, "train_f100.npz")
    if os.path.exists(path):  # resume: keep the solvers already recorded
        old = dict(np.load(path))
        old.update({k: v for k, v in out.items()})
        out = old
    for name in which:
        xs, ts, xn, tn, brk = [], [], [], [], []

        def spy(view, fixed, target, *a, **k):
            r = orig(view, fixed, target, *a, **k)
            if target.shape[0] == m:
                xs.append(target[rows_x].copy())
                xn.append(np.linalg.norm(target.astype(np.float64)))
            else:
                ts.append(target[rows_t].copy())
                tn.append(np.linalg.norm(target.astype(np.float64)))
            brk.append(r[2])
            return r
        als.update_side = spy
        t0 = time.time()
        try:
            _, _, rep = cmf.train(sr, te, cmf.AlsConfig(f=f, lam=0.05, epochs=10, solver=cfgs[name]))
        finally:
            als.update_side = orig
        out[name + "_rmse"] = np.array(rep.rmse_trajectory())
        out[name + "_obj"] = np.array([e.objective for e in rep.epochs])
        out[name + "_objmid"] = np.array([e.objective_mid for e in rep.epochs])
        out[name + "_Xrows"], out[name + "_Trows"] = np.stack(xs), np.stack(ts)
        out[name + "_Xnorm"], out[name + "_Tnorm"] = np.array(xn), np.array(tn)
        out[name + "_breakdowns"] = np.array(brk)
        out[name + "_seconds"] = np.array(time.time() - t0)
        print(name, time.time() - t0, "s", out[name + "_rmse"], flush=True)
        np.savez_compressed(path, **out)


def implicit_small(cmf):
    import cmf.implicit as imp
    out = {}
    m, n, nnz, f = 300, 160, 4000, 12
    rng = np.random.default_rng(11)
    flat = np.sort(rng.choice(m * n, size=nnz, replace=False))
    vals = rng.integers(1, 6, size=nnz).astype(np.float32)  # play counts / stars
    t = cmf.Triples((flat // n).astype(np.int64), (flat % n).astype(np.int64), vals)
    tr, te = cmf.split_holdout(t, 0.1, 3)
    sr = cmf.build(tr, m + 2, n)  # two users without observations
    out["meta"] = np.array([m + 2, n, f], np.int64)
    for name, a in (("row_ptr", sr.row_ptr), ("col_idx", sr.col_idx), ("csr_val", sr.csr_val),
                    ("col_ptr", sr.col_ptr), ("row_idx", sr.row_idx), ("csc_val", sr.csc_val)):
        out[name] = a
    out["te_u"], out["te_v"], out["te_r"] = te.user, te.item, te.rating
    theta = cmf.init_factors(n, f, 0.1, [0, 1])
    x0 = cmf.init_factors(m + 2, f, 0.1, [0, 0])
    g = imp.precompute_gram(theta)
    out["gram_theta"] = g
    x1 = x0.copy()
    imp.implicit_update_side(sr.csr_view(), theta, g, x1, 40.0, 0.05, cmf.SolverConfig("exact"))
    out["x0"], out["x1_exact"] = x0, x1
    for name, cfg in (("exact", cmf.SolverConfig("exact")),
                      ("cg32", cmf.SolverConfig("cg", 6, 1e-4, "fp32"))):
        # (fp16 storage overflows binary16 here: alpha r F^T F exceeds 65504 -- the
        # reference raises NumericalError, and so does the B200 path)
        xs, ts = [], []
        orig = imp.implicit_update_side

        def spy(view, fixed, gram, target, *a, **k):
            r = orig(view, fixed, gram, target, *a, **k)
            (xs if target.shape[0] == m + 2 else ts).append(target.copy())
            return r
        imp.implicit_update_side = spy
        try:
            X, T, rep = imp.implicit_train(sr, imp.ImplicitConfig(f=f, alpha=40.0, lam=0.05, epochs=4,
                                                                  solver=cfg), te)
        finally:
            imp.implicit_update_side = orig
        out[name + "_X"], out[name + "_T"] = np.stack(xs), np.stack(ts)
        out[name + "_obj"] = np.array([e.objective for e in rep.epochs])
        out[name + "_objmid"] = np.array([e.objective_mid for e in rep.epochs])
        out[name + "_rmse"] = np.array([e.rmse for e in rep.epochs])
        if name == "exact":
            out["exact_mpr"] = np.array(imp.mean_percentile_rank(X, T, te))
        print("implicit", name, out[name + "_obj"], out[name + "_rmse"])
    np.savez_compressed(os.path.join(OUT, "implicit_small.npz"), **out)


def implicit16(cmf):
    """implicit_train on the implicit_small instance with binary16 Hermitian
    storage (cg16), alpha = 1 so that alpha r F^T F stays inside binary16 range;
    plus one cg16 implicit_update_side from x0 (rows without observations
    included)."""
    import cmf.implicit as imp
    g = dict(np.load(os.path.join(OUT, "implicit_small.npz")))
    m, n, f = (int(v) for v in g["meta"])
    sr = cmf.SparseRatings(m, n, int(g["row_ptr"][-1]), g["row_ptr"], g["col_idx"], g["csr_val"],
                           g["col_ptr"], g["row_idx"], g["csc_val"])
    te = cmf.Triples(g["te_u"], g["te_v"], g["te_r"])
    out = {"meta": g["meta"], "alpha": np.array(1.0)}
    cfg = cmf.SolverConfig("cg", 6, 1e-4, "fp16")
    theta = cmf.init_factors(n, f, 0.1, [0, 1])
    x1 = g["x0"].copy()
    imp.implicit_update_side(sr.csr_view(), theta, imp.precompute_gram(theta), x1, 1.0, 0.05, cfg)
    out["x1_cg16"] = x1
    X, T, rep = imp.implicit_train(sr, imp.ImplicitConfig(f=f, alpha=1.0, lam=0.05, epochs=4, solver=cfg), te)
    out["cg16_X"], out["cg16_T"] = X, T
    out["cg16_obj"] = np.array([e.objective for e in rep.epochs])
    out["cg16_rmse"] = np.array([e.rmse for e in rep.epochs])
    X, T, rep = imp.implicit_train(sr, imp.ImplicitConfig(f=f, alpha=1.0, lam=0.05, epochs=4,
                                                          solver=cmf.SolverConfig("exact")), te)
    out["exact_obj"] = np.array([e.objective for e in rep.epochs])
    out["exact_rmse"] = np.array([e.rmse for e in rep.epochs])
    print("implicit16", out["cg16_obj"], out["cg16_rmse"], out["exact_rmse"])
    np.savez_compressed(os.path.join(OUT, "implicit16.npz"), **out)


def implicit100(cmf):
    """implicit_train at f = 100 (the fused weighted kernel's headline instance,
    FC = 25) on a non-negative instance with users of ~50 and items of ~100
    observations: cg16 (alpha = 1) and exact trajectories (objective and
    preference RMSE per epoch) and one cg16
    implicit_update_side of each side from the initial factors."""
    import cmf.implicit as imp
    m, n, nnz, f = 3000, 1500, 165_000, 100
    rng = np.random.default_rng(100)
    flat = np.sort(rng.choice(m * n, size=nnz, replace=False))
    vals = rng.integers(1, 6, size=nnz).astype(np.float32)
    t = cmf.Triples((flat // n).astype(np.int64), (flat % n).astype(np.int64), vals)
    tr, te = cmf.split_holdout(t, 0.1, 7)
    sr = cmf.build(tr, m, n)
    out = {"meta": np.array([m, n, f], np.int64), "alpha": np.array(1.0)}
    for name, a in (("row_ptr", sr.row_ptr), ("col_idx", sr.col_idx), ("csr_val", sr.csr_val),
                    ("col_ptr", sr.col_ptr), ("row_idx", sr.row_idx), ("csc_val", sr.csc_val)):
        out[name] = a
    out["te_u"], out["te_v"], out["te_r"] = te.user, te.item, te.rating
    cfg = cmf.SolverConfig("cg", 6, 1e-4, "fp16")
    x0 = cmf.init_factors(m, f, 0.1, [0, 0])
    t0 = cmf.init_factors(n, f, 0.1, [0, 1])
    x1 = x0.copy()
    imp.implicit_update_side(sr.csr_view(), t0, imp.precompute_gram(t0), x1, 1.0, 0.05, cfg)
    t1 = t0.copy()
    imp.implicit_update_side(sr.csc_view(), x0, imp.precompute_gram(x0), t1, 1.0, 0.05, cfg)
    out["x1_cg16"], out["t1_cg16"] = x1, t1
    X, T, rep = imp.implicit_train(sr, imp.ImplicitConfig(f=f, alpha=1.0, lam=0.05, epochs=3, solver=cfg), te)
    out["cg16_obj"] = np.array([e.objective for e in rep.epochs])
    out["cg16_rmse"] = np.array([e.rmse for e in rep.epochs])
    X, T, rep = imp.implicit_train(sr, imp.ImplicitConfig(f=f, alpha=1.0, lam=0.05, epochs=3,
                                                          solver=cmf.SolverConfig("exact")), te)
    out["exact_obj"] = np.array([e.objective for e in rep.epochs])
    out["exact_rmse"] = np.array([e.rmse for e in rep.epochs])
    print("implicit100", out["cg16_obj"], out["cg16_rmse"], out["exact_obj"], out["exact_rmse"])
    np.savez_compressed(os.path.join(OUT, "implicit100.npz"), **out)


def io_cases(cmf):
    out = {}
    rng = np.random.default_rng(21)
    m, n, k = 30, 20, 150
    u = rng.integers(0, m, k).astype(np.int64)
    v = rng.integers(0, n, k).astype(np.int64)
    r = (rng.standard_normal(k) * 2).astype(np.float32)
    t = cmf.Triples(u, v, r)
    sr = cmf.build(t, m, n)
    d = tempfile.mkdtemp()
    cmf.data.save_cache(os.path.join(d, "c.cmfr"), sr)
    out["u"], out["v"], out["r"], out["dims"] = u, v, r, np.array([m, n])
    out["cache_bytes"] = np.frombuffer(open(os.path.join(d, "c.cmfr"), "rb").read(), dtype=np.uint8)
    for fmt in ("tsv", "csv"):
        cmf.data.save_coo(os.path.join(d, "c." + fmt), t, fmt=fmt)
        out[fmt + "_bytes"] = np.frombuffer(open(os.path.join(d, "c." + fmt), "rb").read(), dtype=np.uint8)
    text = "# header\n\n3\t4\t1.5\n  0\t0\t-2.25e-3 \n# mid\n7\t1\t3\n3\t4\t0.1\n"
    pt, pm, pn = cmf.data.parse_coo(text.splitlines(True), fmt="tsv")
    out["parse_text"] = np.frombuffer(text.encode(), dtype=np.uint8)
    out["parse_u"], out["parse_v"], out["parse_r"] = pt.user, pt.item, pt.rating
    out["parse_dims"] = np.array([pm, pn])
    shutil.rmtree(d)
    np.savez_compressed(os.path.join(OUT, "io_cases.npz"), **out)


if __name__ == "__main__":
    cmf = import_reference()
    cmf.set_workers(os.cpu_count() or 1)
    which = sys.argv[1:] or ["gram", "solve", "build", "data", "small", "implicit", "io", "ml1m"]
    for w in which:
        {"gram": gram_cases, "solve": solve_cases, "build": build_cases,
         "data": data_cases, "small": train_small, "implicit": implicit_small,
         "io": io_cases, "ml1m": train_ml1m, "f100": train_f100, "implicit16": implicit16,
         "implicit100": implicit100}[w](cmf)
        print("wrote", w)

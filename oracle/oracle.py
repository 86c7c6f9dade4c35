"""CPU oracle for the ALS half-iteration -- TEST INFRASTRUCTURE ONLY.

This module restates the reference package (``/root/reference/pkg/src/cmf``)
for the hot path named in BASELINE.json: numpy for the data preparation and
evaluation, and the C restatement ``cmf_oracle.c`` (OpenMP) for the Gram /
bias / CG / Cholesky loops.  Every function cites the reference lines it
restates.

It is pinned against golden vectors produced by the reference itself
(``tests/golden/make_golden.py``); ``tests/test_oracle.py`` checks it.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and
``--impl reference``) may import this module.  The product package
``paper_1808_03843_b200`` never does.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import time
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_c_i64p = ctypes.POINTER(ctypes.c_int64)


def build_oracle() -> str:
    """Compile cmf_oracle.c with the committed Makefile (gcc, OpenMP)."""
    src = os.path.join(_HERE, "cmf_oracle.c")
    if (not os.path.exists(_LIB_PATH)
            or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src)):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build_oracle()
        L = ctypes.CDLL(_LIB_PATH)
        vp = ctypes.c_void_p
        L.oracle_assemble.argtypes = [vp, vp, vp, vp, ctypes.c_int64, vp, ctypes.c_int,
                                      ctypes.c_double, ctypes.c_int, vp, vp, vp, vp,
                                      ctypes.c_int]
        L.oracle_assemble.restype = ctypes.c_int
        L.oracle_pack_half.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int]
        L.oracle_pack_half.restype = ctypes.c_int64
        L.oracle_cg_batch.argtypes = [vp, ctypes.c_int, vp, vp, vp, ctypes.c_int64,
                                      ctypes.c_int, ctypes.c_int, vp, vp, vp, ctypes.c_int]
        L.oracle_cg_batch.restype = ctypes.c_int
        L.oracle_cholesky_batch.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int, vp, vp,
                                            ctypes.c_int]
        L.oracle_cholesky_batch.restype = ctypes.c_int64
        L.oracle_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class OracleNumericalError(Exception):
    pass


class OracleSingularError(Exception):
    def __init__(self, msg, rows):
        super().__init__(msg)
        self.rows = list(rows)


# ---------------------------------------------------------------- data layer
# data.py:205-249 (build), :252-267 (split_holdout), :270-302 (gen_synthetic),
# factors.py:29-38 (init_factors), :41-54 (predict_pairs).

@dataclass
class OTriples:
    user: np.ndarray
    item: np.ndarray
    rating: np.ndarray

    def __len__(self):
        return int(self.user.shape[0])


@dataclass
class ORatings:
    m: int
    n: int
    nnz: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    csr_val: np.ndarray
    col_ptr: np.ndarray
    row_idx: np.ndarray
    csc_val: np.ndarray

    def csr(self):
        return (self.row_ptr, self.col_idx, self.csr_val, self.m, self.n)

    def csc(self):
        return (self.col_ptr, self.row_idx, self.csc_val, self.n, self.m)


def predict_pairs(x, theta, users, items, chunk=1 << 18):
    """factors.py:41-54: float32 einsum per 2^18-pair chunk."""
    users = np.asarray(users)
    items = np.asarray(items)
    out = np.empty(users.shape[0], dtype=np.float32)
    for lo in range(0, users.shape[0], chunk):
        hi = min(lo + chunk, users.shape[0])
        out[lo:hi] = np.einsum("ij,ij->i", x[users[lo:hi]], theta[items[lo:hi]])
    return out


def gen_synthetic(m, n, f, density, noise_sigma, seed):
    """data.py:270-302 (same PCG64 draw sequence)."""
    k = int(round(density * m * n))
    rng = np.random.default_rng(seed)
    half = np.float32(0.5)
    x_true = (rng.random((m, f), dtype=np.float32) - half).astype(np.float32)
    t_true = (rng.random((n, f), dtype=np.float32) - half).astype(np.float32)
    flat = rng.choice(m * n, size=k, replace=False)
    flat.sort()
    users = (flat // n).astype(np.int64)
    items = (flat % n).astype(np.int64)
    r = predict_pairs(x_true, t_true, users, items)
    if noise_sigma > 0:
        r = (r.astype(np.float64) + rng.normal(0.0, noise_sigma, size=k)).astype(np.float32)
    return OTriples(users, items, r), x_true, t_true


def split_holdout(t: OTriples, frac: float, seed: int):
    """data.py:252-267."""
    total = len(t)
    k = int(round(frac * total))
    perm = np.random.default_rng(seed).permutation(total)
    te, tr = np.sort(perm[:k]), np.sort(perm[k:])
    sub = lambda ix: OTriples(t.user[ix], t.item[ix], t.rating[ix])
    return sub(tr), sub(te)


def build(t: OTriples, m: int, n: int) -> ORatings:
    """data.py:205-249: lexsort by (user, item, position), keep the last of each
    duplicate run, CSR by counting, CSC by a second lexsort."""
    user, item, val = t.user, t.item, t.rating
    if len(t):
        bad = (user < 0) | (user >= m) | (item < 0) | (item >= n)
        if bad.any():
            raise ValueError("triple out of range")
    order = np.lexsort((np.arange(len(t), dtype=np.int64), item, user))
    su, si, sv = user[order], item[order], val[order]
    if len(t):
        keep = np.ones(len(t), dtype=bool)
        keep[:-1] = (su[:-1] != su[1:]) | (si[:-1] != si[1:])
        su, si, sv = su[keep], si[keep], sv[keep]
    row_ptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(np.bincount(su, minlength=m), out=row_ptr[1:])
    co = np.lexsort((su, si))
    col_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(si, minlength=n), out=col_ptr[1:])
    return ORatings(m, n, int(su.shape[0]), row_ptr, si.astype(np.int32),
                    sv.astype(np.float32), col_ptr, su[co].astype(np.int32),
                    sv[co].astype(np.float32))


def _mix64(z):
    """splitmix64 finaliser on uint64 arrays (wrap-around arithmetic), gen.cu mix64."""
    z = np.asarray(z, dtype=np.uint64)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xbf58476d1ce4e5b9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94d049bb133111eb)
    return z ^ (z >> np.uint64(31))


def gen_stream_triples(seed, m, n, f, thr_cell, thr_test, noise_scale):
    """numpy restatement of the streaming generator (paper_1808_03843_b200
    csrc/gen.cu -- the B200 package's own counter-based generator, a restatement
    of gen_synthetic's model, data.py:270-302; not the reference's PCG64 draws):
    returns (train triples, test triples) in (user, item) order.  Small m*n only
    (every cell is hashed)."""
    with np.errstate(over="ignore"):
        base = np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15)
        salts = [_mix64(base + np.uint64(k)) for k in range(1, 6)]
        s_cell, s_test, s_noise, s_x, s_t = salts

        def H(s, a, b):
            return _mix64(((np.asarray(a, np.uint64) << np.uint64(32)) | np.asarray(b, np.uint64)) ^ s)

        def truth(salt, rows):
            r, k = np.meshgrid(np.arange(rows, dtype=np.uint64), np.arange(f, dtype=np.uint64), indexing="ij")
            v = (H(salt, r, k) >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)
            return (v - np.float32(0.5)).astype(np.float32)

        X, T = truth(s_x, m), truth(s_t, n)
        uu, vv = np.meshgrid(np.arange(m, dtype=np.uint64), np.arange(n, dtype=np.uint64), indexing="ij")
        uu, vv = uu.ravel(), vv.ravel()
        present = H(s_cell, uu, vv) < np.uint64(thr_cell)
        uu, vv = uu[present], vv[present]
        test = H(s_test, uu, vv) < np.uint64(thr_test)
        acc = np.zeros(uu.shape[0], np.float32)
        xi, ti = X[uu.astype(np.int64)], T[vv.astype(np.int64)]
        for k in range(f):  # sequential, round after every multiply and add
            acc = (acc + (xi[:, k] * ti[:, k]).astype(np.float32)).astype(np.float32)
        h = H(s_noise, uu, vv)
        q = [((h >> np.uint64(sh)) & np.uint64(0xffff)).astype(np.float32) for sh in (0, 16, 32, 48)]
        q = [((x + np.float32(0.5)) * np.float32(2.0 ** -16)).astype(np.float32) for x in q]
        s = ((q[0] + q[1]).astype(np.float32) + (q[2] + q[3]).astype(np.float32)).astype(np.float32)
        s = (s - np.float32(2.0)).astype(np.float32)
        r = (acc + (s * np.float32(noise_scale)).astype(np.float32)).astype(np.float32)
    u64, v64 = uu.astype(np.int64), vv.astype(np.int64)
    tr = OTriples(u64[~test], v64[~test], r[~test])
    te = OTriples(u64[test], v64[test], r[test])
    return tr, te, X, T


def init_factors(rows, f, scale=0.1, seed=0):
    """factors.py:29-38."""
    raw = np.random.default_rng(seed).random((rows, f), dtype=np.float32)
    return (raw * np.float32(2.0) - np.float32(1.0)) * np.float32(scale)


# ---------------------------------------------------------------- hot path

def packed_size(f):
    return f * (f + 1) // 2


def pack_half(a32: np.ndarray) -> np.ndarray:
    """gram.py:132-146 via the C RNE converter."""
    a32 = np.ascontiguousarray(a32, dtype=np.float32)
    out = np.empty(a32.shape, dtype=np.uint16)
    over = lib().oracle_pack_half(_p(a32), _p(out), a32.size, 0)
    if over:
        raise OracleNumericalError("Gram entries overflow binary16 range; rescale")
    return out.view(np.float16)


def assemble_side(indptr, indices, values, nrows, theta, lam, precision="fp32",
                  weighted_reg=True, a_weights=None, b_weights=None,
                  base_packed=None, nthreads=0):
    """gram.py:236-314 -> (a_lower, b, n_u)."""
    theta = np.ascontiguousarray(theta, dtype=np.float32)
    f = theta.shape[1]
    P = packed_size(f)
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int32)
    bw = np.ascontiguousarray(values if b_weights is None else b_weights, dtype=np.float32)
    aw = None if a_weights is None else np.ascontiguousarray(a_weights, dtype=np.float32)
    base = None if base_packed is None else np.ascontiguousarray(base_packed, dtype=np.float32)
    a = np.empty((nrows, P), dtype=np.float32)
    b = np.empty((nrows, f), dtype=np.float32)
    nu = np.empty(nrows, dtype=np.int64)
    lib().oracle_assemble(_p(indptr), _p(indices), _p(aw), _p(bw), nrows, _p(theta), f,
                          float(lam), int(bool(weighted_reg)), _p(base), _p(a), _p(b),
                          _p(nu), int(nthreads))
    if precision == "fp16":
        a = pack_half(a)
    return a, b, nu


def cg_batch(a_lower, b, x0, f_s, eps, nthreads=0):
    """solvers.py:121-145; eps is the absolute per-system tolerance."""
    n_sys, f = b.shape
    half = a_lower.dtype == np.float16
    a = np.ascontiguousarray(a_lower.view(np.uint16) if half else a_lower.astype(np.float32))
    b = np.ascontiguousarray(b, dtype=np.float32)
    x0 = np.ascontiguousarray(x0, dtype=np.float32)
    eps = np.ascontiguousarray(eps, dtype=np.float64)
    out = np.empty((n_sys, f), dtype=np.float32)
    it = np.empty(n_sys, dtype=np.int64)
    br = np.empty(n_sys, dtype=np.int64)
    lib().oracle_cg_batch(_p(a), int(half), _p(b), _p(x0), _p(eps), n_sys, f, int(f_s),
                          _p(out), _p(it), _p(br), int(nthreads))
    return out, it, br


def cholesky_batch(a_lower, b, nthreads=0):
    """solvers.py:148-164 + the aggregation loop :221-235."""
    n_sys, f = b.shape
    a = np.ascontiguousarray(a_lower, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    out = np.zeros((n_sys, f), dtype=np.float32)
    info = np.empty(n_sys, dtype=np.int32)
    nbad = lib().oracle_cholesky_batch(_p(a), _p(b), n_sys, f, _p(out), _p(info),
                                       int(nthreads))
    if nbad:
        rows = np.flatnonzero(info).tolist()
        raise OracleSingularError(f"singular system(s) at rows {rows[:8]}", rows)
    return out


def batch_solve(a_lower, b, x0, method="cg", cg_iters=6, cg_tol=1e-4, nthreads=0):
    """solvers.py:205-247 -> (x, iterations, breakdowns)."""
    if method == "exact":
        return cholesky_batch(a_lower, b, nthreads), np.zeros(b.shape[0], np.int64), 0
    eps = cg_tol * np.linalg.norm(b.astype(np.float64), axis=1)
    x, it, br = cg_batch(a_lower, b, x0, cg_iters, eps, nthreads)
    return x, it, int(br.sum())


def update_side(view, fixed, target, lam, method="cg", precision="fp32", cg_iters=6,
                cg_tol=1e-4, weighted_reg=True, nthreads=0, block_bytes=2 << 30):
    """als.py:54-74: assemble, compact rows with n_u > 0, solve, scatter in place.

    Rows are independent, so the half-update runs in row blocks of at most
    `block_bytes` of packed fp32 systems (the reference materialises all of
    them: 9.7 GB on the Netflix X side); the results do not depend on it."""
    indptr, indices, values, nrows, ncols = view
    indptr = np.asarray(indptr)
    f = fixed.shape[1]
    rows_per = max(1, int(block_bytes // (4 * packed_size(f))))
    br = 0
    for lo in range(0, nrows, rows_per):
        hi = min(nrows, lo + rows_per)
        p0, p1 = int(indptr[lo]), int(indptr[hi])
        a, b, nu = assemble_side(indptr[lo:hi + 1] - p0, indices[p0:p1], values[p0:p1], hi - lo,
                                 fixed, lam, precision, weighted_reg, nthreads=nthreads)
        sel = np.flatnonzero(nu > 0)
        x, _, nbr = batch_solve(a[sel], b[sel], target[lo + sel], method, cg_iters, cg_tol,
                                nthreads)
        target[lo + sel] = x
        br += nbr
    return br


def objective(x, theta, r: ORatings, lam, weighted=True, chunk=1 << 18):
    """als.py:77-97 (float64)."""
    total = 0.0
    users = np.repeat(np.arange(r.m, dtype=np.int64), np.diff(r.row_ptr))
    for lo in range(0, r.nnz, chunk):
        hi = min(lo + chunk, r.nnz)
        pred = np.einsum("ij,ij->i", x[users[lo:hi]].astype(np.float64),
                         theta[r.col_idx[lo:hi]].astype(np.float64))
        d = r.csr_val[lo:hi].astype(np.float64) - pred
        total += float(d @ d)
    sq_x = (x.astype(np.float64) ** 2).sum(axis=1)
    sq_t = (theta.astype(np.float64) ** 2).sum(axis=1)
    if weighted:
        reg = float(np.diff(r.row_ptr).astype(np.float64) @ sq_x
                    + np.diff(r.col_ptr).astype(np.float64) @ sq_t)
    else:
        reg = float(sq_x.sum() + sq_t.sum())
    return total + lam * reg


def rmse(x, theta, test: OTriples):
    """als.py:100-107."""
    pred = predict_pairs(x, theta, test.user, test.item)
    d = test.rating.astype(np.float64) - pred.astype(np.float64)
    return float(np.sqrt(np.mean(d * d)))


def train(r: ORatings, test: OTriples | None, f=100, lam=0.05, epochs=10, method="cg",
          precision="fp32", cg_iters=6, cg_tol=1e-4, init_scale=0.1, seed=0,
          weighted_reg=True, nthreads=0, callback=None):
    """als.py:110-157 (update-X, objective, update-Theta, objective, RMSE)."""
    x = init_factors(r.m, f, init_scale, [seed, 0])
    theta = init_factors(r.n, f, init_scale, [seed, 1])
    hist = []
    for epoch in range(epochs):
        t0 = time.perf_counter()
        bx = update_side(r.csr(), theta, x, lam, method, precision, cg_iters, cg_tol,
                         weighted_reg, nthreads)
        t1 = time.perf_counter()
        obj_mid = objective(x, theta, r, lam, weighted_reg)
        t2 = time.perf_counter()
        bt = update_side(r.csc(), x, theta, lam, method, precision, cg_iters, cg_tol,
                         weighted_reg, nthreads)
        t3 = time.perf_counter()
        obj = objective(x, theta, r, lam, weighted_reg)
        e = rmse(x, theta, test) if test is not None and len(test) else None
        hist.append({"epoch": epoch, "objective": obj, "objective_mid": obj_mid,
                     "rmse": e, "breakdowns": bx + bt,
                     "sec_update": (t1 - t0) + (t3 - t2)})
        if callback is not None:
            callback(epoch, x, theta)
    return x, theta, hist

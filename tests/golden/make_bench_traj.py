"""Generate tests/golden/bench_traj_<shape>.npz: the reference algorithm's RMSE
and objective trajectories on the bench's own inputs (TEST INFRASTRUCTURE).

    python tests/golden/make_bench_traj.py [netflix|ml1m] [exact,cg16,cg32]

The inputs follow the SURVEY 8(d) protocol exactly as bench.py builds them:
total = round(nnz/0.9); gen_synthetic(m, n, f, total/(m n), sigma=0.1, seed=0);
split_holdout(0.1, seed=1); build; init_factors(0.1, [0,0] / [0,1]);
lam=0.05, weighted lambda, cg_iters=6, cg_tol=1e-4.

At Netflix shape the reference package itself needs ~10 min per iteration
per solver on this container's 8 cores, so the trajectories come
from the oracle port (oracle/: C restatement, pinned bit for bit to the
reference's own outputs on train_small / gram / solve goldens by
tests/test_oracle.py).  bench.py reads the fixture at run time:
  * time_to_rmse's target = the exact trajectory's epoch-10 RMSE + 1e-3
    (the reference exact run where feasible);
  * rmse_parity = max |RMSE_gpu(epoch) - RMSE_ref(epoch)| over 10 epochs, the
    north_star's CG bar (<= 1e-3);
  * input digests prove the bench regenerated the same CSR/CSC/test arrays.
"""

import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

SHAPES = {"netflix": (480_189, 17_770, 99_000_000, 100), "ml1m": (6_040, 3_706, 1_000_000, 32)}
SOLVERS = {"exact": ("exact", "fp32"), "cg16": ("cg", "fp16"), "cg32": ("cg", "fp32")}


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    from oracle import oracle as o
    shape = sys.argv[1] if len(sys.argv) > 1 else "netflix"
    which = (sys.argv[2] if len(sys.argv) > 2 else "exact,cg16").split(",")
    m, n, nnz, f = SHAPES[shape]
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"bench_traj_{shape}.npz")
    out = dict(np.load(path)) if os.path.exists(path) else {}
    t0 = time.time()
    total = round(nnz / 0.9)
    t, _, _ = o.gen_synthetic(m, n, f, total / (m * n), 0.1, 0)
    tr, te = o.split_holdout(t, 0.1, 1)
    del t
    r = o.build(tr, m, n)
    del tr
    print(f"data {time.time() - t0:.1f}s nnz={r.nnz}", flush=True)
    out["meta"] = np.array([m, n, nnz, f])
    out["csr_digest"] = np.array(digest(r.row_ptr, r.col_idx, r.csr_val))
    out["csc_digest"] = np.array(digest(r.col_ptr, r.row_idx, r.csc_val))
    out["test_digest"] = np.array(digest(te.user, te.item, te.rating))
    out["threads"] = np.array(o.max_threads())
    for name in which:
        method, prec = SOLVERS[name]
        t0 = time.time()
        _, _, hist = o.train(r, te, f=f, lam=0.05, epochs=10, method=method, precision=prec,
                             callback=lambda e, x, th: print(f"  {name} epoch {e} "
                                                            f"{time.time() - t0:.0f}s", flush=True))
        out[name + "_rmse"] = np.array([h["rmse"] for h in hist])
        out[name + "_obj"] = np.array([h["objective"] for h in hist])
        out[name + "_objmid"] = np.array([h["objective_mid"] for h in hist])
        out[name + "_breakdowns"] = np.array([h["breakdowns"] for h in hist])
        out[name + "_sec_update"] = np.array([h["sec_update"] for h in hist])
        print(name, f"{time.time() - t0:.0f}s", out[name + "_rmse"], flush=True)
        np.savez_compressed(path, **out)


if __name__ == "__main__":
    main()

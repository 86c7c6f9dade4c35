"""Device times of the SURVEY 8(f) rows at Netflix shape (perf probe, not the bench):
implicit ALS iteration (f1), test RMSE / objective (f2), CSR+CSC build (f3).

python tools/probe_next.py [--gram-kernels fma,bitwise] [--reps 2]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1808_03843_b200 as cmfb  # noqa: E402
from paper_1808_03843_b200.implicit import implicit_update_side, precompute_gram  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--gram-kernels", default="fma")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--f", type=int, default=100)
args = ap.parse_args()
m, n, nnz, f = 480_189, 17_770, 99_000_000, args.f


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


train, test = cmfb.gen_synthetic_device(m, n, f, nnz, 0.1, 0.1, seed=0)
x = torch.from_numpy(cmfb.init_factors(m, f, 0.1, [0, 0])).cuda()
th = torch.from_numpy(cmfb.init_factors(n, f, 0.1, [0, 1])).cuda()
out = {"shape": [m, n, train.nnz], "f": f}

# f3: CSR + CSC build from device triples (stable sorts, last duplicate wins)
users = torch.repeat_interleave(torch.arange(m, device="cuda"), train.row_ptr.diff())
trip = cmfb.Triples(users, train.col_idx.to(torch.int64), train.csr_val)
out["build_ms"] = timed(lambda: cmfb.build_device(trip, m, n), 1)
del users, trip

# f2: evaluation
out["rmse_ms"] = timed(lambda: cmfb.rmse(x, th, test), args.reps)
out["objective_ms"] = timed(lambda: cmfb.objective(x, th, train, 0.05), args.reps)

# f1: one implicit iteration (both halves, alpha = 40, CG fp32, f_s = 6) on
# |r| as the non-negative interaction strength
solver = cmfb.SolverConfig("cg")
csr = cmfb.RowView(train.row_ptr, train.col_idx, train.csr_val.abs(), m, n)
csc = cmfb.RowView(train.col_ptr, train.row_idx, train.csc_val.abs(), n, m)
for gk in args.gram_kernels.split(","):
    xi, ti = x.clone(), th.clone()

    def it():
        implicit_update_side(csr, ti, precompute_gram(ti), xi, 40.0, 0.05, solver, gram_kernel=gk)
        implicit_update_side(csc, xi, precompute_gram(xi), ti, 40.0, 0.05, solver, gram_kernel=gk)

    out[f"implicit_iter_ms_{gk}"] = timed(it, args.reps)
print(json.dumps(out))

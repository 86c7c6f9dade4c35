"""Per-half, per-kernel device times at a benchmark shape (perf probe, not the bench).

python tools/probe.py [--shape netflix] [--kernels tc,fma] [--solvers cg16,exact] [--reps 3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1808_03843_b200 as cmfb  # noqa: E402
from paper_1808_03843_b200.als import HalfUpdatePlan, resolve_events  # noqa: E402

SHAPES = {"netflix": (480_189, 17_770, 99_000_000), "ml1m": (6_040, 3_706, 1_000_000),
          "small": (48_019, 17_770, 9_900_000), "yahoo": (1_000_990, 624_961, 252_800_000)}

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="netflix")
ap.add_argument("--f", type=int, default=100)
ap.add_argument("--kernels", default="tc")
ap.add_argument("--solvers", default="cg16")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--only", default="xt")
args = ap.parse_args()
m, n, nnz = SHAPES[args.shape]
f = args.f
train, test = cmfb.gen_synthetic_device(m, n, f, nnz, 0.1, 0.1, seed=0)
x = torch.from_numpy(cmfb.init_factors(m, f, 0.1, [0, 0])).cuda()
th = torch.from_numpy(cmfb.init_factors(n, f, 0.1, [0, 1])).cuda()
SOLV = {"cg16": ("cg", "fp16"), "cg32": ("cg", "fp32"), "exact": ("exact", "fp32")}
out = {}
for sname in args.solvers.split(","):
    meth, prec = SOLV[sname]
    solver = cmfb.SolverConfig(meth, precision=prec)
    for kern in args.kernels.split(","):
        if kern == "tc" and meth == "exact":
            continue
        for side in args.only:
            if side == "x":
                view, fixed, target = train.csr_view(), th, x
            else:
                view, fixed, target = train.csc_view(), x, th
            plan = HalfUpdatePlan(view.nrows, f, solver, x.device)
            for rep in range(args.reps + 1):
                tg = target.clone()  # fresh warm start each rep (a solved target exits CG early)
                rec = {}
                plan.launch(view.indptr, view.indices, view.values, fixed, tg, 0.05, True, kern, rec)
                torch.cuda.synchronize()
                ms = {k: sum(v) for k, v in resolve_events(rec).items()}
            out[f"{sname}/{kern}/{side}"] = ms
            print(sname, kern, side, json.dumps({k: round(v, 3) for k, v in ms.items()}), flush=True)

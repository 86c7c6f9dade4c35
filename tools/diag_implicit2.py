"""implicit_train trajectories (small instance, alpha=1) per route vs the reference's goldens."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1808_03843_b200 as cmfb

g = dict(np.load(os.path.join(ROOT, "tests/golden/implicit_small.npz")))
g16 = dict(np.load(os.path.join(ROOT, "tests/golden/implicit16.npz")))
m, n, f = (int(v) for v in g["meta"])
sr = cmfb.SparseRatings(m, n, int(g["row_ptr"][-1]), g["row_ptr"], g["col_idx"], g["csr_val"],
                        g["col_ptr"], g["row_idx"], g["csc_val"])
te = cmfb.Triples(g["te_u"], g["te_v"], g["te_r"])
print("ref cg16 ", g16["cg16_rmse"])
print("ref exact", g16["exact_rmse"])
for name, solver, kern in (("fused", cmfb.SolverConfig("cg", 6, 1e-4, "fp16"), None),
                           ("fma16", cmfb.SolverConfig("cg", 6, 1e-4, "fp16"), "fma"),
                           ("exact", cmfb.SolverConfig("exact"), None)):
    X, T, rep = cmfb.implicit_train(sr, cmfb.ImplicitConfig(f=f, alpha=1.0, lam=0.05, epochs=4, solver=solver), te,
                                    gram_kernel=kern)
    print(name.ljust(9), np.array([e.rmse for e in rep.epochs]), np.array([e.objective for e in rep.epochs]))

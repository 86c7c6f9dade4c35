"""Step-by-step fused vs fma16 vs exact half-updates along the fused trajectory."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1808_03843_b200 as cmfb

g = dict(np.load(os.path.join(ROOT, "tests/golden/implicit_small.npz")))
m, n, f = (int(v) for v in g["meta"])
sr = cmfb.SparseRatings(m, n, int(g["row_ptr"][-1]), g["row_ptr"], g["col_idx"], g["csr_val"],
                        g["col_ptr"], g["row_idx"], g["csc_val"])
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
x = cmfb.init_factors(m, f, 0.1, [0, 0])
t = cmfb.init_factors(n, f, 0.1, [0, 1])
s16 = cmfb.SolverConfig("cg", 6, 1e-4, "fp16")
for ep in range(2):
    for side in "xt":
        view, fixed, tgt = (sr.csr_view(), t, x) if side == "x" else (sr.csc_view(), x, t)
        gram = cmfb.precompute_gram(fixed)
        res = {}
        for name, solver, kern, dev in (("fused", s16, None, False), ("fused_dev", s16, None, True),
                                        ("fma16", s16, "fma", False), ("exact", cmfb.SolverConfig("exact"), None, False)):
            if dev:
                tt = torch.from_numpy(tgt.copy()).cuda()
                cmfb.implicit_update_side(view, torch.from_numpy(fixed).cuda(), torch.from_numpy(gram).cuda(), tt,
                                          1.0, 0.05, solver, gram_kernel=kern)
                res[name] = tt.cpu().numpy()
            else:
                tt = tgt.copy()
                cmfb.implicit_update_side(view, fixed, gram, tt, 1.0, 0.05, solver, gram_kernel=kern)
                res[name] = tt
        print(ep, side, "max|fixed|=%.3f" % np.abs(fixed).max(),
              " ".join(f"{k}:{rel(res['fused'], res[k]):.2e}" for k in res if k != "fused"),
              "fma16-vs-exact %.2e" % rel(res["fma16"], res["exact"]))
        if side == "x":
            x = res["fused"]
        else:
            t = res["fused"]

"""Diagnostics for the fused implicit route (small instance): per-side relative
differences between the fused kernel, the two-step FMA route (same fp16
storage) and the exact solve."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1808_03843_b200 as cmfb

g = dict(np.load(os.path.join(ROOT, "tests/golden/implicit_small.npz")))
m, n, f = (int(v) for v in g["meta"])
sr = cmfb.SparseRatings(m, n, int(g["row_ptr"][-1]), g["row_ptr"], g["col_idx"], g["csr_val"],
                        g["col_ptr"], g["row_idx"], g["csc_val"])
theta = cmfb.init_factors(n, f, 0.1, [0, 1])
x0 = g["x0"].copy()
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
for alpha in (1.0, 40.0):
    for side in ("x", "t"):
        view, fixed, tgt = (sr.csr_view(), theta, x0) if side == "x" else (sr.csc_view(), x0, theta)
        gram = cmfb.precompute_gram(fixed)
        out = {}
        for name, solver, kern in (("fused", cmfb.SolverConfig("cg", 6, 1e-4, "fp16"), None),
                                   ("fma16", cmfb.SolverConfig("cg", 6, 1e-4, "fp16"), "fma"),
                                   ("fma32", cmfb.SolverConfig("cg", 6, 1e-4, "fp32"), "fma"),
                                   ("exact", cmfb.SolverConfig("exact"), None)):
            t = tgt.copy()
            try:
                cmfb.implicit_update_side(view, fixed, gram, t, alpha, 0.05, solver, gram_kernel=kern)
                out[name] = t
            except Exception as e:  # noqa: BLE001
                print(alpha, side, name, "raised", type(e).__name__)
        if "fused" in out:
            for k in out:
                if k != "fused":
                    d = np.abs(out["fused"] - out[k]).max(1)
                    print(f"alpha={alpha} side={side} fused vs {k}: rel {rel(out['fused'], out[k]):.2e}  "
                          f"worst rows {np.argsort(-d)[:4].tolist()} {np.sort(d)[::-1][:4].round(5).tolist()}")
        if "fma16" in out and "exact" in out:
            print(f"alpha={alpha} side={side} fma16 vs exact: rel {rel(out['fma16'], out['exact']):.2e}")
nu = np.diff(sr.row_ptr)
print("empty rows:", np.nonzero(nu == 0)[0].tolist(), "empty cols:", np.nonzero(np.diff(sr.col_ptr) == 0)[0].tolist())

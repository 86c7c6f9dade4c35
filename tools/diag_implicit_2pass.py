"""Implicit item-side half-update at Netflix shape: the two-pass route (default
for the 100 MB X shadow) against a single pass (CMF_TWO_PASS=0) and against the
two-step route (weighted FMA Gram + the same binary16 CG); relative differences."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1808_03843_b200 as cmfb
from paper_1808_03843_b200.implicit import implicit_update_side, precompute_gram

m, n, f = 480_189, 17_770, 100
train, _ = cmfb.gen_synthetic_device(m, n, f, 99_000_000, 0.1, 0.1, seed=0)
x = torch.from_numpy(cmfb.init_factors(m, f, 0.1, [0, 0])).cuda()
t0 = torch.from_numpy(cmfb.init_factors(n, f, 0.1, [0, 1])).cuda()
csc = cmfb.RowView(train.col_ptr, train.row_idx, train.csc_val.abs(), n, m)
s16 = cmfb.SolverConfig("cg", precision="fp16")
gx = precompute_gram(x)
out = {}
for name, env in (("two_pass", None), ("one_pass", "0")):
    if env is None:
        os.environ.pop("CMF_TWO_PASS", None)
    else:
        os.environ["CMF_TWO_PASS"] = env
    t = t0.clone()
    implicit_update_side(csc, x, gx, t, 1.0, 0.05, s16)
    out[name] = t.cpu().numpy()
os.environ.pop("CMF_TWO_PASS", None)
t = t0.clone()
implicit_update_side(csc, x, gx, t, 1.0, 0.05, s16, gram_kernel="fma")
out["two_step"] = t.cpu().numpy()
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
print("two_pass vs one_pass %.3e  two_pass vs two_step %.3e  one_pass vs two_step %.3e" % (
    rel(out["two_pass"], out["one_pass"]), rel(out["two_pass"], out["two_step"]), rel(out["one_pass"], out["two_step"])))

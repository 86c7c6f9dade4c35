"""Per-half device time of the implicit fused route at Netflix shape (perf probe)."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1808_03843_b200 as cmfb
from paper_1808_03843_b200.implicit import implicit_update_side, precompute_gram

m, n, f = 480_189, 17_770, 100
alpha = float(os.environ.get("ALPHA", "1.0"))
train, test = cmfb.gen_synthetic_device(m, n, f, 99_000_000, 0.1, 0.1, seed=0)
x0 = torch.from_numpy(cmfb.init_factors(m, f, 0.1, [0, 0])).cuda()
t0 = torch.from_numpy(cmfb.init_factors(n, f, 0.1, [0, 1])).cuda()
csr = cmfb.RowView(train.row_ptr, train.col_idx, train.csr_val.abs(), m, n)
csc = cmfb.RowView(train.col_ptr, train.row_idx, train.csc_val.abs(), n, m)
s16 = cmfb.SolverConfig("cg", precision="fp16")
for rep in range(3):
    x, t = x0.clone(), t0.clone()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record()
    gt = precompute_gram(t)
    ev[1].record()
    implicit_update_side(csr, t, gt, x, alpha, 0.05, s16)
    ev[2].record()
    gx = precompute_gram(x)
    ev[3].record()
    implicit_update_side(csc, x, gx, t, alpha, 0.05, s16)
    ev[4].record()
    torch.cuda.synchronize()
    print("gramT %.2f  X %.2f  gramX %.2f  T %.2f ms" % tuple(ev[i].elapsed_time(ev[i + 1]) for i in range(4)))

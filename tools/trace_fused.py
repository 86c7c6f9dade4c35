"""Pipeline timeline of CTA 0 of the fused kernel (cmf_debug_trace) at Netflix shape.

python tools/trace_fused.py [--side t|x] -> per-stage latencies (cycles)."""
import argparse, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1808_03843_b200 as cmfb
from paper_1808_03843_b200 import _native as nat
from paper_1808_03843_b200.als import HalfUpdatePlan

ap = argparse.ArgumentParser()
ap.add_argument("--side", default="t")
ap.add_argument("--kernel", default="tc")
ap.add_argument("--implicit", action="store_true", help="the weighted (implicit-feedback) kernel, alpha = 1")
a = ap.parse_args()
m, n, nnz, f = 480_189, 17_770, 99_000_000, 100
train, test = cmfb.gen_synthetic_device(m, n, f, nnz, 0.1, 0.1, seed=0)
x = torch.from_numpy(cmfb.init_factors(m, f, 0.1, [0, 0])).cuda()
th = torch.from_numpy(cmfb.init_factors(n, f, 0.1, [0, 1])).cuda()
view, fixed, target = (train.csc_view(), x, th) if a.side == "t" else (train.csr_view(), th, x)
solver = cmfb.SolverConfig("cg", precision="fp16")
plan = HalfUpdatePlan(view.nrows, f, solver, x.device)
imp = None
if a.implicit:
    from paper_1808_03843_b200.implicit import _gram_full, precompute_gram
    view = cmfb.RowView(view.indptr, view.indices, view.values.abs(), view.nrows, view.ncols)
    imp = (1.0, _gram_full(precompute_gram(fixed), f, fixed.device))
plan.launch(view.indptr, view.indices, view.values, fixed, target.clone(), 0.05, True, a.kernel, implicit=imp)
buf = torch.zeros(8 * 4096 + 4 * 2048 + 64 * 64, dtype=torch.int64, device="cuda")
nat.call("cmf_debug_trace", nat.ptr(buf))
plan.launch(view.indptr, view.indices, view.values, fixed, target.clone(), 0.05, True, a.kernel, implicit=imp)
torch.cuda.synchronize()
nat.call("cmf_debug_trace", None)
allb = buf.cpu().numpy()
ev = allb[40960:40960 + 4096].reshape(64, 64).astype(np.float64)
for r in (3, 30, 60):
    e = ev[r][ev[r] > 0]
    if len(e) > 2:
        print("row", r, "CG events (cycles from first):", (e - e[0]).astype(int).tolist())
# per exchange (pipelined solve): [entry, after barrier, after matvec wait]; deltas
rows = [ev[r][ev[r] > 0] for r in range(8, 64)]
rows = [e for e in rows if len(e) >= 23]
if rows:
    e = np.array([r[:23] for r in rows])
    d = np.diff(e, axis=1)
    print("median deltas per event (entry->bar, bar->mvwait, mvwait->next entry, ...):")
    print(np.median(d, axis=0).astype(int).tolist())
rr = allb[32768:40960].reshape(2048, 4).astype(np.float64)
rr = rr[(rr[:, 3] > 0) & (rr[:, 0] > 0)]
if len(rr) > 8:
    mid = rr[len(rr) // 4: 3 * len(rr) // 4]
    print("CG rows traced", len(rr))
    print("CG wait for accumulator (1-0): %.0f" % np.median(mid[:, 1] - mid[:, 0]))
    print("CG TMEM load + release  (2-1): %.0f" % np.median(mid[:, 2] - mid[:, 1]))
    print("CG solve                (3-2): %.0f" % np.median(mid[:, 3] - mid[:, 2]))
t7 = allb[:32768].reshape(4096, 8).astype(np.float64)
if a.implicit:
    w = t7[(t7[:, 4] > 0) & (t7[:, 0] > 0) & (t7[:, 5] > 0)]
    w = w - w[0, 0]
    k = len(w)
    mid = w[k // 4: 3 * k // 4]
    print("weighted stages", k, "| median cycles: gather slot wait (1-0) %.0f, issue (2-1) %.0f, "
          "landed after issue (5-2) %.0f, scale (6-5) %.0f, full -> MMA sees (3-6) %.0f, MMA (4-3) %.0f, "
          "commit interval %.0f" % (np.median(mid[:, 1] - mid[:, 0]), np.median(mid[:, 2] - mid[:, 1]),
                                    np.median(mid[:, 5] - mid[:, 2]), np.median(mid[:, 6] - mid[:, 5]),
                                    np.median(mid[:, 3] - mid[:, 6]), np.median(mid[:, 4] - mid[:, 3]),
                                    np.median(np.diff(mid[:, 4]))))
t = t7[:, :5]
ok = (t[:, 4] > 0) & (t[:, 0] > 0)
t = t[ok]
t -= t[0, 0]
k = len(t)
print("stages traced", k)
lo, hi = k // 4, 3 * k // 4
mid = t[lo:hi]
print("per-stage interval (MMA commit to commit): %.0f cyc" % np.median(np.diff(mid[:, 4])))
print("producer slot wait      (1-0): %.0f" % np.median(mid[:, 1] - mid[:, 0]))
print("producer issue          (2-1): %.0f" % np.median(mid[:, 2] - mid[:, 1]))
print("data latency to MMA     (3-2): %.0f  p90 %.0f" % (np.median(mid[:, 3] - mid[:, 2]), np.percentile(mid[:, 3] - mid[:, 2], 90)))
print("MMA issue               (4-3): %.0f" % np.median(mid[:, 4] - mid[:, 3]))
print("slot free -> MMA sees   (3-1): %.0f" % np.median(mid[:, 3] - mid[:, 1]))
for i in range(lo, lo + 12):
    print(i, (t[i] - t[lo, 0]).astype(int).tolist())

import numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import paper_1808_03843_b200 as cmfb
for f, (m, n, nnz) in ((8, (50, 40, 300)), (32, (500, 200, 8000)), (100, (300, 900, 30000))):
    t, _ = cmfb.gen_synthetic(m, n, f, nnz / (m * n), 0.1, 3)
    sr = cmfb.build(t, m + 1, n)
    theta = cmfb.init_factors(n, f, 0.1, [0, 1])
    outs = []
    for kern in ("tc", "tc_unfused", "fma"):
        x = cmfb.init_factors(m + 1, f, 0.1, [0, 0])
        try:
            cmfb.update_side(sr.csr_view(), theta, x, 0.05, cmfb.SolverConfig("cg", precision="fp32"), gram_kernel=kern)
        except Exception as e:
            print(f, kern, "ERR", e); x = None
        outs.append(x)
    if outs[0] is not None:
        for k in range(1,3):
            rel = np.linalg.norm(outs[0] - outs[k]) / np.linalg.norm(outs[k])
            print(f, "fused vs", ["tc_unfused","fma"][k-1], rel)
        print(" row0 fused", outs[0][0][:6]); print(" row0 unfus", outs[1][0][:6])

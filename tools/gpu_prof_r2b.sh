#!/bin/bash
# round-2 evidence: ncu of the implicit (weighted) fused kernel, the two-step
# binary16 CG, the build kernels' launch list and the Hugewiki-shape launch list
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_cg -c 2 -o gpurun_out/prof_impl -f \
  python tools/probe_implicit.py > gpurun_out/prof_impl.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:cg_tc -c 1 -o gpurun_out/prof_cgtc2 -f \
  python tools/probe.py --kernels tc_unfused --solvers cg16 --reps 1 --only x > gpurun_out/prof_cgtc2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_build.csv \
  python -c "
import torch, paper_1808_03843_b200 as c
tr, te = c.gen_synthetic_device(480189, 17770, 100, 99000000, 0.1, 0.1, seed=0)
u = torch.repeat_interleave(torch.arange(tr.m, device='cuda'), tr.row_ptr.diff())
p = torch.randperm(tr.nnz, device='cuda')
c.build_device(c.Triples(u[p], tr.col_idx.long()[p], tr.csr_val[p]), tr.m, tr.n)
torch.cuda.synchronize()" > gpurun_out/launches_build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_huge.csv python bench.py --shape hugewiki --steps 1 --warmup 3 > gpurun_out/b_huge_ncu.log 2>&1
echo done

#!/bin/bash
# A/B of the two-step route's batched binary16 CG (cg_tc_kernel) across library builds in tools/ab/.
for rep in 1 2; do
  for v in "$@"; do
    CMF_LIB_PATH=tools/ab/$v.so timeout 120 python tools/probe.py --kernels tc_unfused --solvers cg16 --reps 2 --only x 2>&1 | tail -1 | sed "s/^/$v /"
  done
done

#!/bin/bash
# A/B of the exact route (split tensor-core Gram + Cholesky) across library builds in tools/ab/.
for rep in 1 2; do
  for v in "$@"; do
    CMF_LIB_PATH=tools/ab/$v.so timeout 120 python tools/probe.py --kernels tc_split --solvers exact --reps 2 2>&1 | tail -2 | head -1 | sed "s/^/$v /"
  done
done

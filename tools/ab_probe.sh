#!/bin/bash
# A/B timing of library builds in tools/ab/*.so on ONE box (box-to-box clock
# differences exceed most kernel changes): tools/ab_probe.sh base var1 var2 ...
for rep in 1 2; do
  for v in "$@"; do
    CMF_LIB_PATH=tools/ab/$v.so timeout 90 python tools/probe.py --kernels tc --solvers cg16 --reps 3 2>&1 | tail -2 | sed "s/^/$v /"
  done
done

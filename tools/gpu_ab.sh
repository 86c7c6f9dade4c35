#!/bin/bash
# usage: tools/gpu_ab.sh "pytest args" base v1 ...   (fused-route tests on the current build, then same-box A/B)
mkdir -p gpurun_out
T="$1"; shift
if [ -n "$T" ]; then timeout 400 python -m pytest -q -x -m gpu $T > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ab.log; tail -4 gpurun_out/pytest_ab.log; fi
bash tools/ab_probe.sh "$@" 2>&1 | tee gpurun_out/ab.log

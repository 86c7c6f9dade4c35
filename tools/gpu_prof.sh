#!/bin/bash
# ncu evidence for the bench step: launch list of the timed region + one --set full
# capture of each fused launch (X half, Theta half).  Outputs under gpurun_out/.
# (--data device: same shape and uniform cell distribution as the reference-protocol
# inputs, generated on the GPU in a second instead of ~40 s on the host)
mkdir -p gpurun_out
TAG=${1:-r2}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
  --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-exact --no-e2e --no-cpu --no-ttr --no-next --data device ${BENCHARGS} > gpurun_out/b_ncu_$TAG.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:${KREGEX:-fused_cg} -c ${KCOUNT:-2} -o gpurun_out/prof_$TAG -f \
  python bench.py --steps 1 --warmup 3 --no-exact --no-e2e --no-cpu --no-ttr --no-next --data device ${BENCHARGS} > gpurun_out/prof_$TAG.log 2>&1
echo done

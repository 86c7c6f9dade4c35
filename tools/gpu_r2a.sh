#!/bin/bash
# Round-2 check: parity tests, the reference-protocol bench (ml1m quick, gloo 2-rank, netflix default)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -12 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --shape ml1m --f 32 --steps 5 --warmup 3 > gpurun_out/b_ml1m.json 2> gpurun_out/b_ml1m.err; tail -3 gpurun_out/b_ml1m.err
CMF_DIST_BACKEND=gloo timeout 300 python bench.py --gpus 2 --shape ml1m --f 32 --steps 5 --warmup 3 --no-next > gpurun_out/b_ml1m_g2.json 2> gpurun_out/b_ml1m_g2.err; tail -3 gpurun_out/b_ml1m_g2.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
nproc; free -g | head -2

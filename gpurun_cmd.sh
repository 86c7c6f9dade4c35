mkdir -p gpurun_out
timeout 400 python -m pytest -q -x -m gpu tests/test_gpu_gram_tc.py tests/test_gpu_boundary.py > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ab.log; tail -3 gpurun_out/pytest_ab.log
bash tools/ab_probe.sh v2 v3 2>&1 | tee gpurun_out/ab.log
CMF_TWO_PASS=0 bash tools/ab_probe.sh v3 2>&1 | sed 's/^/onepass /' | tee -a gpurun_out/ab.log

timeout 600 python -m pytest tests -q -m gpu 2>&1 | grep -E "FAILED|passed|failed" | head -5
python tools/probe.py --kernels tc --solvers cg16 --reps 3 2>&1 | tail -2
CMF_L2_EVICT_LAST=0 python tools/probe.py --kernels tc --solvers cg16 --reps 3 --only t 2>&1 | tail -1
CMF_L2_PERSIST_MB=80 python tools/probe.py --kernels tc --solvers cg16 --reps 3 --only t 2>&1 | tail -1
CMF_L2_EVICT_LAST=0 CMF_L2_PERSIST_MB=100 python tools/probe.py --kernels tc --solvers cg16 --reps 3 --only t 2>&1 | tail -1
python -c "import torch; p=torch.cuda.get_device_properties(0); print('L2', p.L2_cache_size, 'persist max', getattr(p,'persisting_l2_cache_max_size',None))"

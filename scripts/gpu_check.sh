cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_switches.py tests/test_gpu_dp.py -x -q 2>&1 | tail -1
BATCHES="256 1024" bash scripts/ab_kern.sh 2>&1 | head -4
timeout 300 python profiles/timeline_eager.py 1024 | tail -9

cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -3
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dp.py -x -q 2>&1 | tail -1
BATCHES="256 512 1024" timeout 300 bash scripts/ab_kern.sh 2>&1 | head -2
timeout 120 python profiles/timeline_eager.py 1024 | tail -3

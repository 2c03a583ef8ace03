cd $GRAFT_REPO_ROOT; timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_switches.py -x -q 2>&1 | tail -2; bash scripts/ab_kern.sh

cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_dp.py -x -q 2>&1 | tail -1
timeout 300 python profiles/cta_trace.py 32 4 | head -8
for rep in 1 2; do timeout 300 python profiles/graph_step.py 32 2>&1 | tail -1; done

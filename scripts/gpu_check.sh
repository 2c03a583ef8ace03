cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_switches.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for rep in 1 2; do for d in . .ab_base; do (cd $d && echo "$d $(timeout 300 python profiles/graph_step.py 32 2>&1 | tail -1)"); done; done

cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_switches.py tests/test_gpu_parity.py tests/test_gpu_dp.py tests/test_gpu_plugin.py tests/test_gpu_reference_api.py -x -q 2>&1 | tail -2
BATCHES="512 1024" SKIP=0 bash scripts/ab_kern.sh 2>&1 | head -4
STEPS=2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_head|k_fc1_acc7" --csv python profiles/one_step.py 1024 2>/dev/null | grep -E "k_head|k_fc1" | tail -4 | cut -c1-200

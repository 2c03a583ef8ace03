# A/B: epoch-level frames/s of a baseline tree (.ab_cur) vs the working tree, alternating,
# then the GPU test suite of the working tree.  Output: gpurun_out/ab_pair.log
mkdir -p gpurun_out; exec > gpurun_out/ab_pair.log 2>&1
nvidia-smi -L
for i in 1 2; do
  for d in /root/repo/.ab_cur /root/repo; do (cd $d && timeout 300 python /root/repo/scripts/ab_epoch.py 2>&1 | tail -3); done
done
[ -n "$AB_TESTS" ] && timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3

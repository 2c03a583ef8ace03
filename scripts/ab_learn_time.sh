# learner step time at batches $@ for the baseline tree (.ab_cur) and the working tree, alternating
mkdir -p gpurun_out; exec > gpurun_out/ab_learn_time.log 2>&1
for i in 1 2; do
  for d in /root/repo/.ab_cur /root/repo; do echo "$d"; (cd $d && timeout 300 python /root/repo/profiles/learn_time.py "$@"); done
done

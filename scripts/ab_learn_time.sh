# learner step time at batches $@ for baseline trees (.ab_old, .ab_cur, if present) and the
# working tree, alternating; learn_time.py imports the package from the current directory
mkdir -p gpurun_out; exec > gpurun_out/ab_learn_time.log 2>&1
for i in 1 2; do
  for d in /root/repo/.ab_old /root/repo/.ab_cur /root/repo; do
    [ -d "$d/paper_2111_01264_b200" ] || continue
    echo "$d"; (cd $d && timeout 300 python /root/repo/profiles/learn_time.py "$@")
  done
done

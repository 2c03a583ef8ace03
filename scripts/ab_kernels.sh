for d in .ab_base .; do
  (cd $d && timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -s 40 -c 16 --csv --log-file /root/repo/gpurun_out/abk_$(basename $(pwd)).csv python profiles/one_step.py 32 > /dev/null 2>&1)
done
ls gpurun_out/abk_*

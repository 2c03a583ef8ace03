for T in 1 0; do
  PQ_TMA=$T timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed.avg.per_cycle_active,launch__grid_size,lts__t_bytes.sum --clock-control none -s 15 -c 15 --csv --log-file gpurun_out/lb_tma$T.csv python profiles/learn_batch.py 1024 3 > gpurun_out/lb$T.log 2>&1
  PQ_TMA=$T timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 30 --csv --log-file gpurun_out/l32_tma$T.csv python profiles/learn_batch.py 32 5 > gpurun_out/l32$T.log 2>&1
done

# launch list of one steady-state Sigma factor of config 3 (the second of two)
export ONLY_SIGMA=1
timeout 300 python tools/dev_factor.py 3 2 > gpurun_out/r2z_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fp64.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r2z_factor_launches.csv python tools/dev_factor.py 3 2 > gpurun_out/r2z_ncu.log 2>&1
echo rc=$?

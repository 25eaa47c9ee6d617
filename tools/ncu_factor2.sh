# launch list of one steady-state Sigma factor of config 3 (the second of two) + per-kernel summary
export ONLY_SIGMA=1
TAG=${1:-s6}
timeout 300 python tools/dev_factor.py 3 2 > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv \
  --log-file gpurun_out/${TAG}_factor_launches.csv python tools/dev_factor.py 3 2 > gpurun_out/${TAG}_ncu.log 2>&1
python tools/ncu_factor_summary.py gpurun_out/${TAG}_factor_launches.csv > gpurun_out/${TAG}_factor_summary.txt 2>&1
echo rc=$?

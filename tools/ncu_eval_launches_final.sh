# ncu launch list (gpu__time_duration.sum, serialised, cold) of one whole config-3 evaluation of the bench, final round-2 build
timeout 1300 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 56000 --csv \
  --log-file gpurun_out/s4_launches.csv python bench.py --no-cpu-baseline --steps 1 > gpurun_out/s4_launches_ncu.log 2>&1
echo rc=$?
python tools/ncu_launch_summary.py gpurun_out/s4_launches.csv > gpurun_out/s4_launches_summary.txt 2>&1
head -20 gpurun_out/s4_launches_summary.txt

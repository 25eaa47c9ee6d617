# ncu launch list (gpu__time_duration.sum, serialised, cold) of one whole config-3 evaluation of the bench
timeout 1500 python bench.py --no-cpu-baseline --steps 1 > gpurun_out/r3l_plain.json 2> gpurun_out/r3l_plain.err && \
timeout 3000 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 60000 --csv \
  --log-file gpurun_out/r3l_launches.csv python bench.py --no-cpu-baseline --steps 1 > gpurun_out/r3l_ncu.log 2>&1
echo rc=$?

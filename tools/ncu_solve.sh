export RSF_NVTX=1 SOLVE_REPS=1
timeout 300 python tools/solve_bw.py 3 1 > gpurun_out/r2z_plain.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "sv.L1/" --nvtx-include "sv.L2/" --nvtx-include "sv.L3/" --nvtx-include "sv.L4/" --nvtx-include "sv.L5/" --nvtx-include "sv.L6/" --nvtx-include "sv.top/" \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r2z_solve_launches.csv python tools/solve_bw.py 3 1 > gpurun_out/r2z_ncu.log 2>&1
echo rc=$?

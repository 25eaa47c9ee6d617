export RSF_NVTX=1 SOLVE_REPS=1
timeout 300 python tools/solve_bw.py 3 1 > gpurun_out/r2k_plain.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "sv.L2/" -k regex:gemv1 -c 3 --set full --import-source on --clock-control none \
  -o gpurun_out/r2k_gemv_full python tools/solve_bw.py 3 1 > gpurun_out/r2k_ncu.log 2>&1
echo rc=$?

# ncu --set full of the first peeling-subtraction GEMM launches (level-1 bases: the longest
# gemm_pipe_kernel launches of an evaluation) on the final round-2 build
export RSF_NVTX=1 RSF_PAR_TRACES=0
timeout 600 python tools/dev_prof3.py > gpurun_out/s4_sub_plain.log 2>&1 && \
timeout 1500 ncu --nvtx --nvtx-include "p.subtract/" -k regex:gemm_pipe -c 9 --set full --import-source on --clock-control none \
  -o gpurun_out/s4_gemm_sub python tools/dev_prof3.py > gpurun_out/s4_sub_ncu.log 2>&1
echo rc=$?
ncu -i gpurun_out/s4_gemm_sub.ncu-rep --page raw --csv > gpurun_out/s4_gemm_sub_raw.csv 2> gpurun_out/s4_sub_csv.err
echo csv_rc=$?

# ncu --set full of the apply-only level-2 sweep GEMMs (the largest G-apply GEMM class)
export RSF_NVTX=1 RSF_PAR_TRACES=0
timeout 600 python tools/dev_prof3.py > gpurun_out/r2w_plain.log 2>&1 && \
timeout 1200 ncu --nvtx --nvtx-include "ao.L2/" -k regex:gemm_pipe -s 6 -c 2 --set full --import-source on --clock-control none \
  -o gpurun_out/r2w_gemm_ao python tools/dev_prof3.py > gpurun_out/r2w_ncu.log 2>&1
echo rc=$?

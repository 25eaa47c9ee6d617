# ncu --set full of the peeling sketch pivot-selection kernel (sketch_cpqr_cl_kernel<1>), serial order
export RSF_PAR_TRACES=0
timeout 600 python tools/dev_prof3.py > gpurun_out/r3m_plain.log 2>&1 && \
timeout 1500 ncu -k regex:sketch_cpqr_cl_kernel -s 300 -c 2 --set full --import-source on --clock-control none \
  -o gpurun_out/r3m_sketch python tools/dev_prof3.py > gpurun_out/r3m_ncu.log 2>&1
echo rc=$?

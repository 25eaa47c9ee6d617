# ncu --set full of the leaf-level fused sweep (sweep_kernel<32>), serial order
export RSF_PAR_TRACES=0
timeout 600 python tools/dev_prof3.py > gpurun_out/r4c_plain.log 2>&1 && \
timeout 1500 ncu -k regex:sweep_kernel -s 20 -c 1 --set full --import-source on --clock-control none \
  -o gpurun_out/r4c_sweep python tools/dev_prof3.py > gpurun_out/r4c_ncu.log 2>&1
echo rc=$?

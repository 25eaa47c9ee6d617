# ncu --set full of the RRQR pivot-selection and panel kernels in one steady-state Sigma factor of config 3
export ONLY_SIGMA=1
timeout 300 python tools/dev_factor.py 3 2 > gpurun_out/s2_plain.log 2>&1 && \
timeout 900 ncu -k regex:'sketch_cpqr_cl_kernel|qr_panel' -s 40 -c 6 --set full --import-source on --clock-control none \
  -o gpurun_out/s2_rrqr python tools/dev_factor.py 3 2 > gpurun_out/s2_ncu.log 2>&1
echo rc=$?

# factor timing + ncu --set full of the register RRQR kernels (cluster 8) in a config-3 Sigma factor
export ONLY_SIGMA=1
TAG=${1:-s7}
timeout 300 python tools/dev_factor.py 3 3 > gpurun_out/${TAG}_f3.log 2>&1
timeout 300 python tools/dev_factor.py 4 2 > gpurun_out/${TAG}_f4.log 2>&1
timeout 900 ncu -k regex:'sketch_cpqr_reg_kernel|qr_panel_reg_kernel' -s 60 -c 4 --set full --import-source on --clock-control none \
  -o gpurun_out/${TAG}_rrqr python tools/dev_factor.py 3 2 > gpurun_out/${TAG}_ncu.log 2>&1
echo rc=$?

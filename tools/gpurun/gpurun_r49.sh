cd $GRAFT_REPO_ROOT
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sketch_cpqr_cl_kernel -s 400 -c 3 -o gpurun_out/r49_sketch python tools/dev_scale.py 3 262144 1 > gpurun_out/r49_ncu.log 2>&1; echo "ncu exit $?" >> gpurun_out/r49_ncu.log

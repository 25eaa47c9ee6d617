cd $GRAFT_REPO_ROOT
for o in 14677 19641 6053; do
RSF_GEMMLOG=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_pipe_kernel -s $o -c 1 -o gpurun_out/r37_gemm_$o python tools/dev_scale.py 3 262144 1 > gpurun_out/r37_ncu_$o.log 2>&1; echo "ncu exit $?" >> gpurun_out/r37_ncu_$o.log
done

cd $GRAFT_REPO_ROOT
python tools/gemm_bench.py > gpurun_out/r36_gemm.log 2>&1
RSF_GEMMLOG=1 timeout 900 python tools/dev_scale.py 3 262144 1 > gpurun_out/r36_scale3.log 2>&1; echo "scale exit $?" >> gpurun_out/r36_scale3.log

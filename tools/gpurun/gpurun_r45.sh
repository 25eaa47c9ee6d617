cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gemm.py -q -x > gpurun_out/r45_gemm_test.log 2>&1; echo "pytest exit $?" >> gpurun_out/r45_gemm_test.log
python tools/gemm_bench.py > gpurun_out/r45_gemm_small.log 2>&1
RSF_GEMM_SMALLK=0 python tools/gemm_bench.py > gpurun_out/r45_gemm_nosmall.log 2>&1
timeout 900 python tools/dev_scale.py 3 262144 3 > gpurun_out/r45_scale3.log 2>&1; echo "scale exit $?" >> gpurun_out/r45_scale3.log
RSF_GEMM_SMALLK=0 timeout 900 python tools/dev_scale.py 3 262144 3 > gpurun_out/r45_scale3_nosmall.log 2>&1; echo "scale exit $?" >> gpurun_out/r45_scale3_nosmall.log

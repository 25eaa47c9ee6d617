cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gemm.py -q -x > gpurun_out/r38_gemm_test.log 2>&1; echo "pytest exit $?" >> gpurun_out/r38_gemm_test.log
python tools/gemm_bench.py > gpurun_out/r38_gemm_epi1.log 2>&1
RSF_GEMM_EPI=0 python tools/gemm_bench.py > gpurun_out/r38_gemm_epi0.log 2>&1
RSF_GEMMLOG=1 timeout 900 python tools/dev_scale.py 3 262144 2 > gpurun_out/r38_scale3.log 2>&1; echo "scale exit $?" >> gpurun_out/r38_scale3.log
RSF_GEMM_EPI=0 timeout 900 python tools/dev_scale.py 3 262144 2 > gpurun_out/r38_scale3_epi0.log 2>&1; echo "scale exit $?" >> gpurun_out/r38_scale3_epi0.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r38_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r38_pytest.log

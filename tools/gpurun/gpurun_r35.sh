cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gemm.py -q -x > gpurun_out/r35_gemm.log 2>&1; echo "pytest exit $?" >> gpurun_out/r35_gemm.log
RSF_GEMMLOG=1 timeout 900 python tools/dev_scale.py 3 262144 2 > gpurun_out/r35_scale3.log 2>&1; echo "scale exit $?" >> gpurun_out/r35_scale3.log
RSF_SPLITK=0 RSF_GEMMLOG=1 timeout 900 python tools/dev_scale.py 3 262144 2 > gpurun_out/r35_scale3_nosplit.log 2>&1; echo "scale exit $?" >> gpurun_out/r35_scale3_nosplit.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r35_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r35_pytest.log

cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r8_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r8_pytest.log
python tools/gemm_bench.py > gpurun_out/r8_gemm.log 2>&1
RSF_GEMM_BN128=1 python tools/gemm_bench.py >> gpurun_out/r8_gemm.log 2>&1
RSF_PROFILE=1 timeout 400 python tools/dev_scale.py 3 > gpurun_out/r8_scale3.log 2>&1; echo "exit $?" >> gpurun_out/r8_scale3.log
RSF_GEMM_BN128=1 RSF_PROFILE=1 timeout 400 python tools/dev_scale.py 3 > gpurun_out/r8_scale3_bn128.log 2>&1; echo "exit $?" >> gpurun_out/r8_scale3_bn128.log

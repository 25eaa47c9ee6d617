cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r30_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r30_pytest.log
python tools/gemm_bench.py > gpurun_out/r30_gemm.log 2>&1
timeout 900 python tools/dev_scale.py 3 262144 4 > gpurun_out/r30_var.log 2>&1; echo "exit $?" >> gpurun_out/r30_var.log

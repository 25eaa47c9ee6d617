cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r29_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r29_pytest.log
RSF_KTRACE=1 timeout 900 python tools/dev_scale.py 3 262144 4 > gpurun_out/r29_var.log 2>&1; echo "exit $?" >> gpurun_out/r29_var.log

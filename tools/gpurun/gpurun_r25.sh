cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r25_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r25_pytest.log

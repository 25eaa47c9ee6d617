cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r56_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r56_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r56_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r56_smoke.log

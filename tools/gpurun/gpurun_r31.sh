cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_aniso.py tests/test_abi_cpu.py -q > gpurun_out/r31_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r31_pytest.log

cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r40_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r40_pytest.log
RSF_GEMMLOG=1 timeout 900 python tools/dev_scale.py 3 262144 2 > gpurun_out/r40_scale3.log 2>&1; echo "scale exit $?" >> gpurun_out/r40_scale3.log
RSF_KTRACE=1 timeout 900 python tools/dev_scale.py 3 262144 1 > gpurun_out/r40_ktrace3.log 2>&1; echo "scale exit $?" >> gpurun_out/r40_ktrace3.log

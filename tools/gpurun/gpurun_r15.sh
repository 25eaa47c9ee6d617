cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r15_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r15_pytest.log
RSF_KTRACE=1 timeout 400 python tools/dev_scale.py 3 > gpurun_out/r15_trace3.log 2>&1; echo "exit $?" >> gpurun_out/r15_trace3.log
timeout 600 python tools/dev_scale.py 3 262144 3 > gpurun_out/r15_plain3.log 2>&1; echo "exit $?" >> gpurun_out/r15_plain3.log

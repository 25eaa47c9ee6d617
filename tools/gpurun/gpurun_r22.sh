cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r22_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r22_pytest.log
timeout 600 python tools/dev_scale.py 3 262144 3 > gpurun_out/r22_plain3.log 2>&1; echo "exit $?" >> gpurun_out/r22_plain3.log
RSF_KTRACE=1 timeout 600 python tools/dev_scale.py 3 262144 2 > gpurun_out/r22_trace3.log 2>&1; echo "exit $?" >> gpurun_out/r22_trace3.log

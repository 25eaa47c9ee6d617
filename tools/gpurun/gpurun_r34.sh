cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r34_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r34_pytest.log
RSF_VERBOSE=1 RSF_GEMMLOG=1 timeout 900 python tools/dev_scale.py 3 262144 2 > gpurun_out/r34_scale3.log 2>&1; echo "scale exit $?" >> gpurun_out/r34_scale3.log
RSF_SPLITK=1 RSF_GEMMLOG=1 timeout 900 python tools/dev_scale.py 3 262144 2 > gpurun_out/r34_scale3_splitk.log 2>&1; echo "scale exit $?" >> gpurun_out/r34_scale3_splitk.log

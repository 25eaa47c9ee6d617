cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r50_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r50_pytest.log
timeout 900 python tools/dev_scale.py 3 262144 3 > gpurun_out/r50_scale3.log 2>&1; echo "scale exit $?" >> gpurun_out/r50_scale3.log
RSF_PAR_TRACES=0 RSF_PROFILE=1 timeout 900 python tools/dev_scale.py 3 262144 2 > gpurun_out/r50_prof3.log 2>&1; echo "scale exit $?" >> gpurun_out/r50_prof3.log

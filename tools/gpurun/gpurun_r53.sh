cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r53_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r53_pytest.log
timeout 900 python tools/dev_scale.py 3 262144 3 > gpurun_out/r53_scale3.log 2>&1; echo "scale exit $?" >> gpurun_out/r53_scale3.log

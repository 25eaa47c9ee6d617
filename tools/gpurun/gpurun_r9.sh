cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r9_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r9_pytest.log
timeout 300 python tools/dev_check.py 1 > gpurun_out/r9_check1.log 2>&1
RSF_GOP=sym timeout 300 python tools/dev_check.py 1 > gpurun_out/r9_check1_sym.log 2>&1
timeout 600 python tools/dev_check.py 2 > gpurun_out/r9_check2.log 2>&1
RSF_GOP=sym timeout 600 python tools/dev_check.py 2 > gpurun_out/r9_check2_sym.log 2>&1
RSF_PROFILE=1 timeout 400 python tools/dev_scale.py 3 > gpurun_out/r9_scale3.log 2>&1; echo "exit $?" >> gpurun_out/r9_scale3.log
RSF_GOP=sym RSF_PROFILE=1 timeout 400 python tools/dev_scale.py 3 > gpurun_out/r9_scale3_sym.log 2>&1; echo "exit $?" >> gpurun_out/r9_scale3_sym.log

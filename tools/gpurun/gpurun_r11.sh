cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r11_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r11_pytest.log
RSF_PROFILE=1 timeout 400 python tools/dev_scale.py 3 > gpurun_out/r11_scale3.log 2>&1; echo "exit $?" >> gpurun_out/r11_scale3.log
timeout 400 python tools/dev_scale.py 3 > gpurun_out/r11_scale3_noprof.log 2>&1; echo "exit $?" >> gpurun_out/r11_scale3_noprof.log

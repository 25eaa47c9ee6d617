cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -k "not full_size" > gpurun_out/r4_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r4_pytest.log
RSF_PROFILE=1 RSF_VERBOSE=1 timeout 400 python tools/dev_scale.py 3 > gpurun_out/r4_scale3.log 2>&1; echo "exit $?" >> gpurun_out/r4_scale3.log
RSF_VERBOSE=1 timeout 900 python tools/dev_scale.py 4 > gpurun_out/r4_scale4.log 2>&1; echo "exit $?" >> gpurun_out/r4_scale4.log

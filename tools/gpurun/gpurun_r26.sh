cd $GRAFT_REPO_ROOT
RSF_PROFILE=1 timeout 600 python tools/dev_factor.py 3 2 > gpurun_out/r26_factor3.log 2>&1; echo "exit $?" >> gpurun_out/r26_factor3.log
timeout 600 python tools/dev_factor.py 4 2 > gpurun_out/r26_factor4.log 2>&1; echo "exit $?" >> gpurun_out/r26_factor4.log

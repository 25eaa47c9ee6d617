cd $GRAFT_REPO_ROOT
RSF_KTRACE=1 timeout 400 python tools/dev_scale.py 3 > gpurun_out/r14_trace3.log 2>&1; echo "exit $?" >> gpurun_out/r14_trace3.log

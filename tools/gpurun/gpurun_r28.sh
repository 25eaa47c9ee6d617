cd $GRAFT_REPO_ROOT
RSF_KTRACE=1 timeout 900 python tools/dev_scale.py 3 262144 5 > gpurun_out/r28_var.log 2>&1; echo "exit $?" >> gpurun_out/r28_var.log

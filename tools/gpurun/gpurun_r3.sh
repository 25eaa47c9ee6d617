cd $GRAFT_REPO_ROOT
timeout 1200 python tools/dev_resid.py 3,4 1e-8,1e-9,1e-10,1e-11 > gpurun_out/r3_resid.log 2>&1; echo "exit $?" >> gpurun_out/r3_resid.log

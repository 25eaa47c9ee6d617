cd $GRAFT_REPO_ROOT
RSF_KTRACE=1 timeout 900 python tools/dev_scale.py 3 262144 1 > gpurun_out/r39_ktrace3.log 2>&1; echo "scale exit $?" >> gpurun_out/r39_ktrace3.log

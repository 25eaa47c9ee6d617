cd $GRAFT_REPO_ROOT
RSF_KTRACE=1 timeout 400 python tools/dev_scale.py 3 > gpurun_out/r18_trace3.log 2>&1; echo "exit $?" >> gpurun_out/r18_trace3.log
PROBE_BLOCK=1024 timeout 600 python tools/dev_scale.py 3 262144 3 > gpurun_out/r18_plain3_pb1024.log 2>&1; echo "exit $?" >> gpurun_out/r18_plain3_pb1024.log

cd $GRAFT_REPO_ROOT
RSF_KTRACE=1 timeout 400 python tools/dev_scale.py 3 > gpurun_out/r13_trace3.log 2>&1; echo "exit $?" >> gpurun_out/r13_trace3.log
timeout 600 python tools/dev_scale.py 3 262144 3 > gpurun_out/r13_plain3.log 2>&1; echo "exit $?" >> gpurun_out/r13_plain3.log
RSF_SPLITK=0 timeout 600 python tools/dev_scale.py 3 262144 3 > gpurun_out/r13_plain3_nosplit.log 2>&1; echo "exit $?" >> gpurun_out/r13_plain3_nosplit.log

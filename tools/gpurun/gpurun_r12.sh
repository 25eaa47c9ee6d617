cd $GRAFT_REPO_ROOT
RSF_KTRACE=1 timeout 400 python tools/dev_scale.py 3 > gpurun_out/r12_trace3.log 2>&1; echo "exit $?" >> gpurun_out/r12_trace3.log
RSF_SPLITK=0 RSF_KTRACE=1 timeout 400 python tools/dev_scale.py 3 > gpurun_out/r12_trace3_nosplit.log 2>&1; echo "exit $?" >> gpurun_out/r12_trace3_nosplit.log
timeout 400 python tools/dev_scale.py 3 > gpurun_out/r12_plain3.log 2>&1; echo "exit $?" >> gpurun_out/r12_plain3.log
RSF_SPLITK=0 timeout 400 python tools/dev_scale.py 3 > gpurun_out/r12_plain3_nosplit.log 2>&1; echo "exit $?" >> gpurun_out/r12_plain3_nosplit.log

cd $GRAFT_REPO_ROOT
RSF_SPLITK=1 timeout 600 python tools/dev_scale.py 3 262144 3 > gpurun_out/r27_split.log 2>&1; echo "exit $?" >> gpurun_out/r27_split.log
timeout 600 python tools/dev_scale.py 3 262144 3 > gpurun_out/r27_nosplit.log 2>&1; echo "exit $?" >> gpurun_out/r27_nosplit.log
timeout 900 python tools/peel_vs_hutch.py 8192 > gpurun_out/r27_pvh.json 2>&1; echo "exit $?" >> gpurun_out/r27_pvh.json

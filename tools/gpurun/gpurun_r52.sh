cd $GRAFT_REPO_ROOT
RSF_KTRACE=1 RSF_PAR_TRACES=0 RSF_ARENA_GB=64 timeout 900 python tools/dev_scale.py 3 262144 2 > gpurun_out/r52_ktrace3_a64.log 2>&1; echo "scale exit $?" >> gpurun_out/r52_ktrace3_a64.log
RSF_ARENA_GB=64 timeout 900 python tools/dev_scale.py 3 262144 3 > gpurun_out/r52_scale3_a64.log 2>&1; echo "scale exit $?" >> gpurun_out/r52_scale3_a64.log
timeout 900 python tools/dev_scale.py 3 262144 3 > gpurun_out/r52_scale3.log 2>&1; echo "scale exit $?" >> gpurun_out/r52_scale3.log

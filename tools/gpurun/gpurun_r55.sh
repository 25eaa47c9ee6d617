cd $GRAFT_REPO_ROOT
RSF_SPLITK_GAIN=0.97 timeout 900 python tools/dev_scale.py 3 262144 3 > gpurun_out/r55_scale3_g97.log 2>&1; echo "scale exit $?" >> gpurun_out/r55_scale3_g97.log
RSF_SPLITK_GAIN=0.8 timeout 900 python tools/dev_scale.py 3 262144 3 > gpurun_out/r55_scale3_g80.log 2>&1; echo "scale exit $?" >> gpurun_out/r55_scale3_g80.log
timeout 900 python tools/dev_scale.py 3 262144 3 > gpurun_out/r55_scale3.log 2>&1; echo "scale exit $?" >> gpurun_out/r55_scale3.log

cd $GRAFT_REPO_ROOT
free -g > gpurun_out/r2_free.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/r2_fp64.txt 2>&1
RSF_PROFILE=1 timeout 400 python tools/dev_scale.py 3 > gpurun_out/r2_scale3_prof.log 2>&1; echo "exit $?" >> gpurun_out/r2_scale3_prof.log
RSF_VERBOSE=1 timeout 600 python tools/dev_scale.py 4 262144 > gpurun_out/r2_scale4_18.log 2>&1; echo "exit $?" >> gpurun_out/r2_scale4_18.log
RSF_VERBOSE=1 RSF_PEEL_LEVELS=2 timeout 900 python tools/dev_scale.py 4 > gpurun_out/r2_scale4_L2.log 2>&1; echo "exit $?" >> gpurun_out/r2_scale4_L2.log

cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused or concurrent" > gpurun_out/r48_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r48_pytest.log
RSF_SWEEP_MMA=1 timeout 900 python tools/dev_scale.py 3 262144 3 > gpurun_out/r48_scale3_mma.log 2>&1; echo "scale exit $?" >> gpurun_out/r48_scale3_mma.log
RSF_SWEEP_MMA=1 RSF_PAR_TRACES=0 RSF_PROFILE=1 timeout 900 python tools/dev_scale.py 3 262144 2 > gpurun_out/r48_prof3_mma.log 2>&1; echo "scale exit $?" >> gpurun_out/r48_prof3_mma.log
timeout 900 python tools/dev_scale.py 3 262144 3 > gpurun_out/r48_scale3.log 2>&1; echo "scale exit $?" >> gpurun_out/r48_scale3.log

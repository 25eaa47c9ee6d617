cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "concurrent or fused" > gpurun_out/r44_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r44_pytest.log
PROBE_BLOCK=1024 timeout 900 python tools/dev_scale.py 3 262144 3 > gpurun_out/r44_scale3_pb1024.log 2>&1; echo "scale exit $?" >> gpurun_out/r44_scale3_pb1024.log
PROBE_BLOCK=768 timeout 900 python tools/dev_scale.py 3 262144 3 > gpurun_out/r44_scale3_pb768.log 2>&1; echo "scale exit $?" >> gpurun_out/r44_scale3_pb768.log

cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1_smi.txt 2>&1
nproc > gpurun_out/r1_host.txt; lscpu | head -20 >> gpurun_out/r1_host.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r1_pytest.log
timeout 600 python tools/dev_scale.py 3 > gpurun_out/r1_scale3.log 2>&1; echo "exit $?" >> gpurun_out/r1_scale3.log
timeout 900 python tools/dev_scale.py 4 > gpurun_out/r1_scale4.log 2>&1; echo "exit $?" >> gpurun_out/r1_scale4.log

set -x
nvidia-smi --query-gpu=name,clocks.sm,memory.total --format=csv
timeout 2400 python -m pytest tests -x -q -m gpu --durations=25 > gpurun_out/s3_gputest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/s3_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/s3_smoke.log
tail -3 gpurun_out/s3_gputest.log; tail -2 gpurun_out/s3_smoke.log

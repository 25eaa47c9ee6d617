cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r20_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r20_pytest.log
timeout 1500 python bench.py > gpurun_out/r20_bench.json 2> gpurun_out/r20_bench.err; echo "bench exit $?" >> gpurun_out/r20_bench.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r20_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:gemm_pipe_kernel -s 30000 -c 4 -o gpurun_out/r20_gemm_pipe python bench.py --no-cpu-baseline > gpurun_out/r20_ncu_full.log 2>&1; echo "ncu exit $?" >> gpurun_out/r20_ncu_full.log

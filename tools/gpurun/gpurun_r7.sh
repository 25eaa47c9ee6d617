cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -k "full_size" > gpurun_out/r7_pytest_full.log 2>&1; echo "pytest exit $?" >> gpurun_out/r7_pytest_full.log
timeout 1200 python bench.py > gpurun_out/r7_bench.json 2> gpurun_out/r7_bench.err; echo "bench exit $?" >> gpurun_out/r7_bench.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r7_plain.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -s 5000 -c 100000 --csv --log-file gpurun_out/r7_launches.csv python bench.py --no-cpu-baseline > gpurun_out/r7_ncu_list.log 2>&1; echo "ncu1 exit $?" >> gpurun_out/r7_ncu_list.log
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:gemm_pipe_kernel -s 2000 -c 3 -o gpurun_out/r7_gemm_pipe python bench.py --no-cpu-baseline > gpurun_out/r7_ncu_full.log 2>&1; echo "ncu2 exit $?" >> gpurun_out/r7_ncu_full.log

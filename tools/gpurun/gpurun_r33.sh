cd $GRAFT_REPO_ROOT
timeout 1500 python bench.py > gpurun_out/r33_bench.json 2> gpurun_out/r33_bench.err; echo "bench exit $?" >> gpurun_out/r33_bench.err
timeout 900 python bench.py --no-cpu-baseline --steps 1 > gpurun_out/r33_plain.log 2>&1 && \
timeout 2700 ncu --metrics gpu__time_duration.sum --clock-control none -s 4000 -c 56000 --csv --log-file gpurun_out/r33_launches.csv python bench.py --no-cpu-baseline --steps 1 > gpurun_out/r33_ncu_list.log 2>&1; echo "ncu1 exit $?" >> gpurun_out/r33_ncu_list.log
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:gemm_pipe_kernel -s 30000 -c 4 -o gpurun_out/r33_gemm_pipe python bench.py --no-cpu-baseline --steps 1 > gpurun_out/r33_ncu_full.log 2>&1; echo "ncu2 exit $?" >> gpurun_out/r33_ncu_full.log

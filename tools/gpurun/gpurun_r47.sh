cd $GRAFT_REPO_ROOT
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r47_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r47_smoke.log
timeout 1500 python bench.py > gpurun_out/r47_bench.json 2> gpurun_out/r47_bench.err; echo "bench exit $?" >> gpurun_out/r47_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r47_ref.json 2> gpurun_out/r47_ref.err; echo "ref exit $?" >> gpurun_out/r47_ref.err
timeout 900 python bench.py --no-cpu-baseline --steps 1 > gpurun_out/r47_plain.log 2>&1 && \
timeout 2700 ncu --metrics gpu__time_duration.sum --clock-control none -s 4000 -c 56000 --csv --log-file gpurun_out/r47_launches.csv python bench.py --no-cpu-baseline --steps 1 > gpurun_out/r47_ncu_list.log 2>&1; echo "ncu1 exit $?" >> gpurun_out/r47_ncu_list.log

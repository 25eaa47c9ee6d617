cd $GRAFT_REPO_ROOT
timeout 1500 python bench.py > gpurun_out/r24_bench.json 2> gpurun_out/r24_bench.err; echo "bench exit $?" >> gpurun_out/r24_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r24_ref.json 2> gpurun_out/r24_ref.err; echo "ref exit $?" >> gpurun_out/r24_ref.err

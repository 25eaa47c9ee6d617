cd $GRAFT_REPO_ROOT
timeout 1500 python bench.py > gpurun_out/r51_bench.json 2> gpurun_out/r51_bench.err; echo "bench exit $?" >> gpurun_out/r51_bench.err
RSF_KTRACE=1 RSF_PAR_TRACES=0 timeout 900 python tools/dev_scale.py 3 262144 2 > gpurun_out/r51_ktrace3.log 2>&1; echo "scale exit $?" >> gpurun_out/r51_ktrace3.log

cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r42_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r42_pytest.log
timeout 900 python tools/dev_scale.py 3 262144 3 > gpurun_out/r42_scale3_par.log 2>&1; echo "scale exit $?" >> gpurun_out/r42_scale3_par.log
RSF_PAR_TRACES=0 timeout 900 python tools/dev_scale.py 3 262144 2 > gpurun_out/r42_scale3_ser.log 2>&1; echo "scale exit $?" >> gpurun_out/r42_scale3_ser.log
timeout 1500 python bench.py > gpurun_out/r42_bench.json 2> gpurun_out/r42_bench.err; echo "bench exit $?" >> gpurun_out/r42_bench.err

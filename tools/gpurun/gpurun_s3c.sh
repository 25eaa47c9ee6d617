# serial-order per-site GEMM log and launch-site trace of one config-3 evaluation
RSF_GEMMLOG=1 timeout 600 python tools/dev_scale.py 3 262144 1 > gpurun_out/s3c_gemmlog.log 2>&1
python tools/gemmlog_summary.py gpurun_out/s3c_gemmlog.log > gpurun_out/s3c_gemmlog_summary.txt 2>&1
RSF_KTRACE=1 timeout 600 python tools/dev_scale.py 3 262144 1 > gpurun_out/s3c_ktrace.log 2>&1
tail -3 gpurun_out/s3c_gemmlog_summary.txt; grep -A12 "KTRACE total" gpurun_out/s3c_ktrace.log

# 1-RHS solve: sweep of the GEMV split cost-model knobs (config 3 Sigma factor, 20 reps each)
for cfg in "128 32 128" "64 32 128" "32 32 128" "256 32 128" "64 64 64" "32 64 64" "16 64 64" "128 64 64" "64 32 64" "0 64 64"; do
  set -- $cfg
  echo "c0=$1 smax=$2 mink=$3" >> gpurun_out/s3e_gemv.log
  RSF_GEMV_C0=$1 RSF_GEMV_SMAX=$2 RSF_GEMV_MINK=$3 timeout 300 python tools/solve_bw.py 3 1 >> gpurun_out/s3e_gemv.log 2>&1
done
RSF_GEMV_SPLIT=0 timeout 300 python tools/solve_bw.py 3 1 >> gpurun_out/s3e_gemv.log 2>&1
grep -o 'c0=.*\|"GBps": [0-9.]*' gpurun_out/s3e_gemv.log

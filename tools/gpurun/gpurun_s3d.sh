# doubling triangular inverse: parity suite (without the 5-minute config-4 case) + A/B bench
timeout 1500 python -m pytest tests -x -q -m gpu -k "not cfg4_full" > gpurun_out/s3d_gputest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/s3d_gputest.log
for v in 0 1 0 1; do
  RSF_TRINV_REC=$v timeout 900 python bench.py --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/s3d_bench_rec$v.$RANDOM.json 2> gpurun_out/s3d_bench_rec$v.err
done
tail -2 gpurun_out/s3d_gputest.log
for f in gpurun_out/s3d_bench_rec*.json; do echo $f; python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['frac'],d['factor_roofline'],d.get('ell'),d.get('grad'))"; done

# LPT order A/B on the config-3 bench (frozen z), then a GEMM log of one evaluation
for lpt in 0 1 0 1; do
  RSF_GEMM_LPT=$lpt timeout 900 python bench.py --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/s3b_bench_lpt$lpt.$RANDOM.json 2> gpurun_out/s3b_bench_lpt${lpt}.err
done
RSF_GEMMLOG=1 timeout 600 python tools/dev_scale.py 3 262144 2 > gpurun_out/s3b_gemmlog.log 2>&1
python tools/gemmlog_summary.py gpurun_out/s3b_gemmlog.log > gpurun_out/s3b_gemmlog_summary.txt 2>&1
for f in gpurun_out/s3b_bench_lpt*.json; do echo $f; python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['frac'],d.get('ell'),d.get('grad'))"; done

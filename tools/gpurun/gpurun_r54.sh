cd $GRAFT_REPO_ROOT
timeout 1500 python bench.py > gpurun_out/r54_bench.json 2> gpurun_out/r54_bench.err; echo "bench exit $?" >> gpurun_out/r54_bench.err
timeout 900 python tools/paper_grid.py > gpurun_out/r54_paper_grid.jsonl 2> gpurun_out/r54_paper_grid.err; echo "grid exit $?" >> gpurun_out/r54_paper_grid.err
RSF_PAR_TRACES=0 RSF_GEMMLOG=1 timeout 900 python tools/dev_scale.py 3 262144 1 > gpurun_out/r54_gemmlog.log 2>&1
ORD=$(python - <<'PY'
import re
best=None
for l in open('gpurun_out/r54_gemmlog.log'):
    m=re.match(r'\s+([\d.]+) s .* longest#(\d+)\s+p\.subtract\|peel\.cu:\d+\|NT', l)
    if m and (best is None or float(m.group(1))>best[0]): best=(float(m.group(1)), int(m.group(2)))
print(best[1] if best else 14677)
PY
)
echo "ordinal $ORD" > gpurun_out/r54_ncu.log
RSF_PAR_TRACES=0 RSF_GEMMLOG=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_pipe_kernel -s $ORD -c 1 -o gpurun_out/r54_gemm python tools/dev_scale.py 3 262144 1 >> gpurun_out/r54_ncu.log 2>&1; echo "ncu exit $?" >> gpurun_out/r54_ncu.log

import os, sys
sys.path.insert(0, '/root/repo')
import paper_1603_08057_b200 as R
# representative shapes of the G-apply sweeps, the subtraction, the RRQR (GEMM log, config 3)
shapes = [(488, 1804, 3500, 16, 0, 0), (488, 944, 5750, 4, 0, 0), (488, 3200, 1620, 64, 0, 0), (976, 3312, 890, 64, 0, 1),
          (488, 12288 // 48, 2400, 48, 0, 1), (976, 1472, 1880, 16, 0, 1), (488, 5144, 700, 256, 0, 0), (4096, 4096, 4096, 1, 0, 0),
          (264, 2000, 8000, 4, 0, 0), (264, 2000, 8000, 4, 0, 1), (6000, 32, 8000, 4, 1, 0), (2000, 32, 16000, 16, 1, 0),
          (488, 32, 4000, 64, 0, 0)]
for (M, N, K, b, ta, tb) in shapes:
    v = R.lib.rsf_debug_gemm_bench(M, N, K, b, ta, tb, 5)
    print(f"variant={os.environ.get('RSF_GEMM_VARIANT', '-1')}/{os.environ.get('RSF_GEMM_VARIANT32', '0')} M={M} N={N} K={K} batch={b} ta={ta} tb={tb}: {v:.2f} TFLOP/s", flush=True)

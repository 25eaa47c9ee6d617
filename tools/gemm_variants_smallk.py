import os, sys
sys.path.insert(0, '/root/repo')
import paper_1603_08057_b200 as R
shapes = [(976, 150, 100, 1024, 0, 0), (976, 150, 100, 1024, 0, 1), (488, 241, 120, 1024, 0, 0), (488, 241, 120, 1024, 0, 1),
          (976, 64, 32, 2048, 0, 0), (2048, 2048, 32, 4, 0, 1), (976, 241, 250, 1024, 0, 0), (8000, 6000, 32, 4, 0, 1)]
for (M, N, K, b, ta, tb) in shapes:
    v = R.lib.rsf_debug_gemm_bench(M, N, K, b, ta, tb, 5)
    print(f"smallk={os.environ.get('RSF_GEMM_VARIANT_SMALLK', '0')} M={M} N={N} K={K} batch={b} ta={ta} tb={tb}: {v:.2f} TFLOP/s", flush=True)

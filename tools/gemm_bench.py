import os, sys
sys.path.insert(0, '/root/repo')
import paper_1603_08057_b200 as R
shapes = [(976, 150, 100, 1024), (488, 150, 100, 1024), (976, 64, 32, 2048), (2048, 2048, 32, 4), (1952, 600, 300, 256), (1952, 1371, 700, 64), (1952, 2900, 1500, 16), (976, 241, 120, 1024), (976, 600, 600, 256), (512, 512, 512, 64), (512, 64, 64, 4096), (512, 32, 32, 8192), (4096, 4096, 4096, 1), (8192, 8192, 64, 1), (512, 2048, 2048, 8)]
for (M, N, K, b) in shapes:
    for ta, tb in [(0, 0), (0, 1)]:
        v = R.lib.rsf_debug_gemm_bench(M, N, K, b, ta, tb, 5)
        print(f"{os.environ.get("RSF_GEMM","pipe")} bn128={os.environ.get("RSF_GEMM_BN128","0")} M={M} N={N} K={K} batch={b} ta={ta} tb={tb}: {v:.2f} TFLOP/s")

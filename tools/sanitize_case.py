"""Small end-to-end case for compute-sanitizer (one tool per gpurun call):
config 1 (n = 1024) l+g with two concurrent trace jobs (theta = rho, sigma2 -> the Tr(F^-1) job
on its own stream), the one-RHS solve / apply / sample paths, a Sigma_i apply, the emulated
two-rank sharded peeling, and the batched GEMM/GEMV test shapes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1603_08057_b200 as R  # noqa: E402
from workloads import config, points_for, w_for  # noqa: E402

c = config(1)
dev = torch.device("cuda:0")
ctx = R.Context(0)
xy = torch.from_numpy(points_for(c)).to(dev)
w = torch.from_numpy(w_for(c)).to(dev)
K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, ("rho", "sigma2"))
F = R.Factor(ctx, xy, K, c.eps_fact, c.leaf)
z = F.sample(w)
x = F.solve(z)
y = F.apply(x)
Fi = R.Factor(ctx, xy, K, c.eps_fact, c.leaf, which=0)
yi = Fi.apply(x)
X = torch.randn(8, c.n, dtype=torch.float64, device=dev)
Xs = F.solve(X)
r = R.gp_mle_eval(ctx, xy, z, K, c.eps_fact, c.leaf, R.Opts(eps_peel=c.eps_peel, seed=c.seed, probe_block=64))
os.environ["RSF_EMU_WORLD"] = "2"
r2 = R.gp_mle_eval(ctx, xy, z, K, c.eps_fact, c.leaf, R.Opts(eps_peel=c.eps_peel, seed=c.seed, probe_block=64))
del os.environ["RSF_EMU_WORLD"]
for (M, N, Kk) in [(1, 200, 3000), (1, 64, 20000), (40, 70, 33)]:
    for ta in (0, 1):
        for tb in (0, 1):
            A = torch.randn(Kk * M, dtype=torch.float64, device=dev)
            B = torch.randn(Kk * N, dtype=torch.float64, device=dev)
            C = torch.randn(M * N, dtype=torch.float64, device=dev)
            assert R.lib.rsf_debug_gemm(ta, tb, M, N, Kk, 1, 1.0, A.data_ptr(), B.data_ptr(), 0.5, C.data_ptr(), 0) == 0
torch.cuda.synchronize()
print("sanitize case ok", r.ell, r.grad, r2.grad, float((y - z).norm() / z.norm()))

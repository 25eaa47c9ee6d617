"""Peeling vs Hutchinson (PAPER §5.2, Fig. 5) on config 2's recipe: relative error of
Tr(Sigma^-1 Sigma_rho) against the dense oracle, versus the number of G applies (columns).

    python tools/peel_vs_hutch.py [n]      (default n = 8192)
"""
import sys, time, json
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from workloads import config, points_for, w_for
from oracle.kernels import Kernel as OK
from oracle.dense import dense_eval, dense_sample
import paper_1603_08057_b200 as R

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
c = config(2)
xy = points_for(c, n)
ok = OK(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
z = dense_sample(ok, xy, w_for(c, n))
t = time.time(); d = dense_eval(ok, xy, z); t_dense = time.time() - t
tr = float(d["trace"][0])
dev = torch.device('cuda:0')
ctx = R.Context(0)
K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
xyd = torch.from_numpy(xy).to(dev)
F = R.Factor(ctx, xyd, K, c.eps_fact, c.leaf)
Fi = R.Factor(ctx, xyd, K, c.eps_fact, c.leaf, which=0)
rows = []
for eps_peel in (1e-4, 1e-6, 1e-8):
    torch.cuda.synchronize(); t = time.time()
    tp, pd = R.peel_trace(F, Fi, eps_peel)
    torch.cuda.synchronize(); dt = time.time() - t
    rows.append({"method": f"peel eps={eps_peel:g}", "applies": pd.applies, "G_cost_columns": 2 * pd.applies,
                 "rel_err": abs(tp - tr) / abs(tr), "seconds": dt})
for q in (16, 64, 256, 1024, 4096):
    torch.cuda.synchronize(); t = time.time()
    th, se = R.hutch_trace(F, Fi, q, 1603080570)
    torch.cuda.synchronize(); dt = time.time() - t
    # one Hutchinson probe costs one solve + one apply = half a symmetrized G column
    rows.append({"method": f"hutchinson q={q}", "applies": q, "G_cost_columns": q, "rel_err": abs(th - tr) / abs(tr),
                 "rel_std_err": se / abs(tr), "seconds": dt})
print(json.dumps({"n": n, "config": "config2 recipe (Matern 3/2, rho=0.05, nugget 1e-3)", "trace_dense": tr,
                  "dense_oracle_seconds": t_dense, "rows": rows}, indent=1))

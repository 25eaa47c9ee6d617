"""The paper's gridded workload (PAPER §5.3, Table 4) on the CUDA path: one l+g
evaluation (3 factorizations + 2 peeled traces) for the Matern 3/2 kernel with anisotropic
theta = [10, 7] on [0, 100]^2 (= [0.1, 0.07] on the unit square), noise 1e-4, eps_peel = 1e-6,
eps_fact = eps_peel / 1000, on sqrt(n) x sqrt(n) grids.  Prints a JSON list with the paper's
MATLAB/Xeon times beside ours (context only: different hardware and implementation).

    python tools/paper_grid.py [m1,m2,...]       (default 64,128,256,512)
"""
import json, sys, time
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from workloads import paper_grid_points, w_for, config
import paper_1603_08057_b200 as R

PAPER = {64: (7.34, 12.3, 19.6), 128: (48.6, 120.0, 168.0), 256: (273.0, 1220.0, 1490.0), 512: (1410.0, 13900.0, 15300.0)}
ms = [int(a) for a in sys.argv[1].split(',')] if len(sys.argv) > 1 else [64, 128, 256, 512]
dev = torch.device('cuda:0')
ctx = R.Context(0)
K = R.Kernel("matern32", 0.1, 1.0, 1e-4, 1.0, ("rho", "rho2"), rho2=0.07)
eps_peel, eps_fact = 1e-6, 1e-9
out = []
for m in ms:
    n = m * m
    xy = torch.from_numpy(paper_grid_points(m)).to(dev)
    w = torch.from_numpy(w_for(config(3), n)).to(dev)
    F = R.Factor(ctx, xy, K, eps_fact, 64)
    z = F.sample(w)
    del F
    best = None
    for rep in range(2):
        torch.cuda.synchronize(); t = time.time()
        r = R.gp_mle_eval(ctx, xy, z, K, eps_fact, 64, R.Opts(eps_peel=eps_peel))
        torch.cuda.synchronize(); el = time.time() - t
        d = r.diag
        row = {"m": m, "n": n, "t_fact": d.t_factor + d.t_compress, "t_peel": d.t_peel, "t_total": el,
               "ell": r.ell, "grad": r.grad, "peel_cols_rho": list(d.peel[0].cols)[:d.fact.levels + 1],
               "paper_xeon_matlab": {"t_fact": PAPER.get(m, (None,) * 3)[0], "t_peel": PAPER.get(m, (None,) * 3)[1],
                                     "t_total": PAPER.get(m, (None,) * 3)[2]}}
        if best is None or el < best["t_total"]:
            best = row
    out.append(best)
    print(json.dumps(best), flush=True)

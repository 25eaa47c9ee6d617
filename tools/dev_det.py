"""Developer probe: reproducibility of the config-3 Sigma factor (standalone, twice) and of the
factor inside gp_mle_eval (log|F|, z^T F^-1 z), to tell rounding-path differences from races."""
import sys, math
import torch
sys.path.insert(0, '/root/repo')
from workloads import config, points_for, frozen_z
import paper_1603_08057_b200 as R
dev = torch.device('cuda:0')
ctx = R.Context(0)
c = config(3)
xy = torch.from_numpy(points_for(c)).to(dev)
z = torch.from_numpy(frozen_z(3)).to(dev)
K0 = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, theta=())
for rep in range(2):
    F = R.Factor(ctx, xy, K0, c.eps_fact, c.leaf)
    ld = F.logdet(); u = F.solve(z); q = float(torch.dot(z, u))
    info = F.info()
    print(f'standalone {rep}: logdet {ld!r} quad {q!r} top {info.top_size} skel {list(info.level_skel)}', flush=True)
    F.close()
K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
o = R.Opts(eps_peel=c.eps_peel, seed=c.seed)
for rep in range(2):
    r = R.gp_mle_eval(ctx, xy, z, K, c.eps_fact, c.leaf, o)
    print(f'eval {rep}: logdet {r.diag.logdet!r} quad {r.diag.quad!r} ell {r.ell!r} grad {r.grad}', flush=True)

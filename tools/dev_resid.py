"""Developer probe: full-size solve residual on sampled rows vs eps_fact (R-A calibration)."""
import sys, time, math
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from workloads import config, points_for, w_for
from oracle.kernels import Kernel as OK
import paper_1603_08057_b200 as R

dev = torch.device('cuda:0')
ctx = R.Context(0)
for cid in [int(a) for a in sys.argv[1].split(',')]:
    c = config(cid)
    xy = points_for(c)
    ok = OK(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    xyd = torch.from_numpy(xy).to(dev)
    w = torch.from_numpy(w_for(c)).to(dev)
    rows = np.random.default_rng(cid).choice(len(xy), 48, replace=False)
    for e in [float(a) for a in sys.argv[2].split(',')]:
        torch.cuda.synchronize(); t = time.time()
        F = R.Factor(ctx, xyd, K, e, c.leaf)
        torch.cuda.synchronize(); tf = time.time() - t
        z = F.sample(w); x = F.solve(z)
        zn, xn = z.cpu().numpy(), x.cpu().numpy()
        res = np.array([ok.sigma_block(xy, np.array([i]), np.arange(len(xy)))[0] @ xn - zn[i] for i in rows])
        rr = math.sqrt(len(xy) / len(rows) * float(res @ res)) / np.linalg.norm(zn)
        inf = F.info()
        print(f'cfg{cid} eps_fact {e:.0e}: factor {tf:.2f}s top {inf.top_size} bytes {inf.factor_bytes/1e9:.2f} GB '
              f'flops {(inf.flops_id+inf.flops_elim+inf.flops_top)/1e12:.2f} TF resid {rr:.3e} |x|/|z| {np.linalg.norm(xn)/np.linalg.norm(zn):.1f}', flush=True)
        del F

"""Developer check on the GPU: CUDA path vs oracle on config 1 (and optionally 2)."""
import sys, time, math
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from workloads import config, points_for, w_for, philox_normal
from oracle.kernels import Kernel as OK
from oracle.dense import dense_eval, dense_sample, dense_sigma
import paper_1603_08057_b200 as R

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
c = config(cid)
n = int(sys.argv[2]) if len(sys.argv) > 2 else c.n
xy = points_for(c, n)
ok = OK(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
z = dense_sample(ok, xy, w_for(c, n))
t = time.time(); d = dense_eval(ok, xy, z); print('oracle dense', time.time() - t, flush=True)
S = dense_sigma(ok, xy)
ctx = R.Context(0)
dev = torch.device('cuda:0')
xyd = torch.from_numpy(xy).to(dev)
zd = torch.from_numpy(z).to(dev)
K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
t = time.time(); F = R.Factor(ctx, xyd, K, c.eps_fact, c.leaf); torch.cuda.synchronize(); print('factor', time.time() - t, flush=True)
info = F.info()
print('levels', info.levels, 'top', info.top_size, [(l, info.level_boxes[l], info.level_active[l], info.level_skel[l], info.level_maxI[l]) for l in range(1, info.levels + 1)])
ld = F.logdet()
print('logdet', ld, d['logdet'], 'rel', abs(ld - d['logdet']) / abs(d['logdet']))
x = F.solve(zd).cpu().numpy()
print('quad rel', abs(z @ x - d['quad']) / d['quad'], 'resid', np.linalg.norm(S @ x - z) / np.linalg.norm(z))
v = np.random.default_rng(0).standard_normal(n)
av = F.apply(torch.from_numpy(v).to(dev)).cpu().numpy()
print('apply vs Sigma', np.linalg.norm(av - S @ v) / np.linalg.norm(S @ v))
sv = F.sample(torch.from_numpy(v).to(dev)).cpu().numpy()
print('sample norm', np.linalg.norm(sv), 'v^T F^-1 v vs |w|^2:', float(sv @ np.linalg.solve(S, sv)), float(v @ v))
Fi = R.Factor(ctx, xyd, K, c.eps_fact, c.leaf, which=0)
Si = ok.dsigma_block(c.theta[0], xy, np.arange(n), np.arange(n))
fv = Fi.apply(torch.from_numpy(v).to(dev)).cpu().numpy()
print('Fi apply vs Sigma_i', np.linalg.norm(fv - Si @ v) / np.linalg.norm(Si @ v))
tr, pd = R.peel_trace(F, Fi, c.eps_peel)
print('trace', tr, d['trace'][0], 'rel', abs(tr - d['trace'][0]) / abs(d['trace'][0]), 'cols', list(pd.cols)[:info.levels+1], 'ranks', list(pd.rank_max)[:info.levels+1], 'secs', pd.seconds)
t = time.time(); r = R.gp_mle_eval(ctx, xyd, zd, K, c.eps_fact, c.leaf, R.Opts(eps_peel=c.eps_peel, seed=c.seed)); print('gp_mle_eval', time.time() - t)
print('ell', r.ell, d['ell'], 'rel', abs(r.ell - d['ell']) / abs(d['ell']))
print('grad', r.grad, d['grad'], 'rel', np.abs(np.array(r.grad) - d['grad']) / np.abs(d['grad']))
print('times tree/factor/compress/solve/peel/total', r.diag.t_tree, r.diag.t_factor, r.diag.t_compress, r.diag.t_solve, r.diag.t_peel, r.diag.t_total, 'launches', r.diag.kernel_launches)

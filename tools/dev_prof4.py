"""Developer probe: phase wall times of one config-4 evaluation (memory-saving mode, serial order;
RSF_PROFILE=1 synchronises at phase boundaries -- set it in the environment)."""
import sys, time
import torch
sys.path.insert(0, '/root/repo')
from workloads import config, points_for, w_for
import paper_1603_08057_b200 as R
dev = torch.device('cuda:0')
ctx = R.Context(0)
c = config(4)
xy = torch.from_numpy(points_for(c)).to(dev)
o = R.Opts(eps_peel=c.eps_peel, seed=c.seed, peel_f32=1)
K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
F = R.Factor(ctx, xy, K, c.eps_fact, c.leaf, opts=o)
z = F.sample(torch.from_numpy(w_for(c)).to(dev))
F.close()
R.lib.rsf_profile_reset()
t = time.time()
r = R.gp_mle_eval(ctx, xy, z, K, c.eps_fact, c.leaf, o)
print("eval", time.time() - t, r.grad, flush=True)
prof = R.lib.rsf_profile_dump().decode()
items = sorted([(float(v), k) for k, v in (x.rsplit("=", 1) for x in prof.strip(";").split(";") if "=" in x)], reverse=True)
for v, k in items[:45]:
    print(f"{v:9.3f}  {k}")

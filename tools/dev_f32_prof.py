"""Developer probe: phase wall times (RSF_PROFILE=1, serial) of one config-3 evaluation with FP64- and
with FP32-stored peeled levels (memory-saving mode), side by side -- where the mode's cost goes."""
import os, sys
os.environ["RSF_PROFILE"] = "1"
import torch
sys.path.insert(0, '/root/repo')
from workloads import config, points_for, frozen_z
import paper_1603_08057_b200 as R
dev = torch.device('cuda:0')
ctx = R.Context(0)
c = config(3)
xy = torch.from_numpy(points_for(c)).to(dev)
z = torch.from_numpy(frozen_z(3)).to(dev)
K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
tabs = {}
for f32 in (0, 1, 0, 1):
    o = R.Opts(eps_peel=c.eps_peel, seed=c.seed, peel_f32=f32)
    R.lib.rsf_profile_reset()
    r = R.gp_mle_eval(ctx, xy, z, K, c.eps_fact, c.leaf, o)
    prof = R.lib.rsf_profile_dump().decode()
    tabs[f32] = {k: float(v) for k, v in (x.rsplit("=", 1) for x in prof.strip(";").split(";") if "=" in x)}
    print(f"peel_f32={f32}: total {r.diag.t_total:.2f} s", flush=True)
keys = sorted(set(tabs[0]) | set(tabs[1]), key=lambda k: -max(tabs[0].get(k, 0), tabs[1].get(k, 0)))
for k in keys[:30]:
    print(f"{k:16s} fp64 {tabs[0].get(k, 0):8.3f}  fp32 {tabs[1].get(k, 0):8.3f}")

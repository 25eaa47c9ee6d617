"""Developer probe: phase wall times of one config-3 evaluation in the serial order (RSF_PROFILE=1
synchronises at phase boundaries; set it in the environment)."""
import os, sys, time
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
o = R.Opts(eps_peel=c.eps_peel, seed=c.seed)
R.gp_mle_eval(ctx, xy, z, K, c.eps_fact, c.leaf, o)
R.lib.rsf_profile_reset()
t = time.time()
r = R.gp_mle_eval(ctx, xy, z, K, c.eps_fact, c.leaf, o)
print("eval", time.time() - t, r.grad, flush=True)
prof = R.lib.rsf_profile_dump().decode()
items = sorted([(float(v), k) for k, v in (x.rsplit("=", 1) for x in prof.strip(";").split(";") if "=" in x)], reverse=True)
for v, k in items[:60]:
    print(f"{v:9.3f}  {k}")
if os.environ.get("RSF_GEMMLOG") == "1":
    g = R.lib.rsf_debug_gemm_log().decode()
    rows = []
    for x in g.strip(";").split(";"):
        if "=" not in x:
            continue
        k, v = x.rsplit("=", 1)
        f = v.split(",")
        rows.append((float(f[0]), float(f[1]), k, v))
    rows.sort(reverse=True)
    import json as _json
    _json.dump([[sec, fl, k, v] for sec, fl, k, v in rows], open(os.path.join("gpurun_out", "gemmlog_rows.json"), "w"))
    for sec, fl, k, v in rows[:40]:
        print(f"{sec:8.3f} s {fl / max(sec, 1e-12) / 1e12:6.1f} TF/s  {k}  {v}")

"""Developer probe: cost and effect of the memory-saving mode at config 3 on the
frozen z -- FP64-stored vs FP32-stored peeled levels, both with the trace jobs in the serial order."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
os.environ["RSF_PAR_TRACES"] = "0"
from workloads import config, points_for, frozen_z
import paper_1603_08057_b200 as R
dev = torch.device('cuda:0')
ctx = R.Context(0)
c = config(3)
xy = torch.from_numpy(points_for(c)).to(dev)
z = torch.from_numpy(frozen_z(3)).to(dev)
K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
res = {}
for f32 in (0, 1, 0, 1):
    o = R.Opts(eps_peel=c.eps_peel, seed=c.seed, peel_f32=f32)
    torch.cuda.synchronize(); t = time.time()
    r = R.gp_mle_eval(ctx, xy, z, K, c.eps_fact, c.leaf, o)
    torch.cuda.synchronize(); el = time.time() - t
    res[f32] = r
    print(f"peel_f32={f32}: {el:.2f} s  grad={list(r.grad)} stored={[r.diag.peel[i].stored_bytes for i in range(2)]}", flush=True)
g0, g1 = np.array(res[0].grad), np.array(res[1].grad)
print("rel diff of g (fp32 vs fp64 storage):", list(np.abs(g1 - g0) / np.abs(g0)))

"""Developer probe: config 3 (frozen z) l+g with the current G operator (RSF_GOP env), timings,
traces, probe columns per level; plus the P7 separable surrogate at 512^2 vs its closed form."""
import os, sys, time, json
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from workloads import config, points_for, frozen_z, separable_axes, SEED_SEPARABLE, STREAM_W, philox_normal_pair
from oracle.separable import SeparableSE
import paper_1603_08057_b200 as R

dev = torch.device('cuda:0')
ctx = R.Context(0)
c = config(3)
xy = torch.from_numpy(points_for(c)).to(dev)
z = torch.from_numpy(frozen_z(3)).to(dev)
K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    t = time.time()
    r = R.gp_mle_eval(ctx, xy, z, K, c.eps_fact, c.leaf, R.Opts(eps_peel=c.eps_peel, seed=c.seed))
    el = time.time() - t
    d = r.diag
    cols = [[d.peel[i].cols[l] for l in range(1, d.peel[i].levels + 1)] for i in range(2)]
    print(json.dumps({"gop": os.environ.get("RSF_GOP", "default"), "t": el, "ell": r.ell, "grad": r.grad,
                      "trace": [d.trace[0], d.trace[1]], "q": [d.q[0], d.q[1]], "cols": cols,
                      "peel_s": d.t_peel}), flush=True)
m = 512
a, b = separable_axes(m)
n = m * m
cc = np.arange((n + 1) // 2, dtype=np.uint64)
w0, w1 = philox_normal_pair(cc, 0, 0, 0, SEED_SEPARABLE, STREAM_W)
w = np.empty(n); w[0::2], w[1::2] = w0, w1
zs = SeparableSE(a, b, 0.016, 1.0, 1e-4).sample(w)
S = SeparableSE(a, b, 0.02, 1.0, 1e-4)
th = ("rho", "sigma2", "nugget")
ref = S.eval(zs, th)
Ks = R.Kernel("sqexp", 0.02, 1.0, 1e-4, theta=th)
t = time.time()
r = R.gp_mle_eval(ctx, torch.from_numpy(S.points()).to(dev), torch.from_numpy(zs).to(dev), Ks, 1e-11, 64, R.Opts(eps_peel=1e-6))
print(json.dumps({"P7_512_t": time.time() - t, "grad_rel_err": [abs(r.grad[i] - ref["grad"][i]) / abs(ref["grad"][i]) for i in range(3)],
                  "trace_rel_err": [abs(r.diag.trace[i] - ref["trace"][i]) / abs(ref["trace"][i]) for i in range(3)]}), flush=True)

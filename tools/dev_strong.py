"""Developer probe: strong- vs weak-admissibility peeling (next row f4) at config 3 (frozen z)
and on the P7 separable surrogate at m x m (closed form)."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from workloads import config, points_for, frozen_z, separable_axes, SEED_SEPARABLE, STREAM_W, philox_normal_pair
from oracle.separable import SeparableSE
import paper_1603_08057_b200 as R

dev = torch.device('cuda:0')
ctx = R.Context(0)
which = sys.argv[1] if len(sys.argv) > 1 else "both"
if which in ("both", "cfg3"):
    c = config(3)
    xy = torch.from_numpy(points_for(c)).to(dev)
    z = torch.from_numpy(frozen_z(3)).to(dev)
    K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    for strong in (1, 0):
        for rep in range(2):
            t = time.time()
            r = R.gp_mle_eval(ctx, xy, z, K, c.eps_fact, c.leaf, R.Opts(eps_peel=c.eps_peel, seed=c.seed, strong=strong))
            d = r.diag
            print(json.dumps({"cfg": 3, "strong": strong, "t": time.time() - t, "grad": r.grad,
                              "trace": [d.trace[0], d.trace[1]],
                              "cols": [[d.peel[i].cols[l] for l in range(1, d.peel[i].levels + 1)] for i in range(2)],
                              "rank_max": [[d.peel[i].rank_max[l] for l in range(1, d.peel[i].levels + 1)] for i in range(2)],
                              "stored_GB": [d.peel[i].stored_bytes / 1e9 for i in range(2)]}), flush=True)
if which in ("both", "p7"):
    m = int(os.environ.get("P7M", "1024"))
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
    X = torch.from_numpy(S.points()).to(dev)
    Z = torch.from_numpy(zs).to(dev)
    for strong in (1, 0):
        t = time.time()
        r = R.gp_mle_eval(ctx, X, Z, Ks, 1e-11, 64, R.Opts(eps_peel=1e-6, strong=strong))
        d = r.diag
        print(json.dumps({"P7_m": m, "strong": strong, "t": time.time() - t,
                          "grad_rel_err": [abs(r.grad[i] - ref["grad"][i]) / abs(ref["grad"][i]) for i in range(3)],
                          "cols": [[d.peel[i].cols[l] for l in range(1, d.peel[i].levels + 1)] for i in (0, 1)],
                          "stored_GB": [d.peel[i].stored_bytes / 1e9 for i in (0, 1)]}), flush=True)
if which == "m12":
    # Matern 1/2 (config 4's kernel, rho = 0.01, nugget 1e-3, theta = (rho, sigma2)) on a perfect
    # jittered m x m grid: weak vs strong peeling (P:760 -- strong should scale better for Matern)
    m = int(os.environ.get("M12M", "512"))
    c3 = config(3)
    xy = torch.from_numpy(points_for(c3, m * m)).to(dev)
    K = R.Kernel("matern12", 0.01, 1.0, 1e-3, 1.0, ("rho", "sigma2"))
    w = torch.from_numpy(np.random.default_rng(5).standard_normal(m * m)).to(dev)
    F = R.Factor(ctx, xy, K, 1e-8, 64)
    z = F.sample(w)
    F.close()
    order = [int(x) for x in os.environ.get("M12ORDER", "1,0").split(",")]
    for strong in order:
        t = time.time()
        try:
            r = R.gp_mle_eval(ctx, xy, z, K, 1e-8, 64, R.Opts(eps_peel=1e-6, strong=strong))
            d = r.diag
            print(json.dumps({"m12_m": m, "strong": strong, "t": time.time() - t, "grad": r.grad,
                              "trace": [d.trace[0], d.trace[1]],
                              "cols": [[d.peel[i].cols[l] for l in range(1, d.peel[i].levels + 1)] for i in (0, 1)],
                              "rank_max": [[d.peel[i].rank_max[l] for l in range(1, d.peel[i].levels + 1)] for i in (0, 1)],
                              "stored_GB": [d.peel[i].stored_bytes / 1e9 for i in (0, 1)]}), flush=True)
        except Exception as e:
            print(json.dumps({"m12_m": m, "strong": strong, "t": time.time() - t, "error": str(e)[:300]}), flush=True)

"""Config 4 (n = 2^20, the metric's workload) on one B200 in the memory-saving mode:
one l+g evaluation (gp_mle_eval, FP32-stored peeled levels, FP64 arithmetic) checked without a dense
reference (n = 2^20 has none, parity unpinned otherwise) against what the mathematics fixes:
  P10  g_i vs Richardson central differences of l (RSF factors at theta +- h, +- 2h; h = 1e-2 theta_i),
  P8   the peeled traces vs Richardson differences of log|F|, and the q_i by the same factor's solve.
z = F^{1/2} w from the CUDA factor (reading R-V for configs 4-5).  Writes one JSON record per run to
profiles/ (argument: output path)."""
import json, math, sys, time
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from workloads import config, points_for, w_for
import paper_1603_08057_b200 as R

out = sys.argv[1] if len(sys.argv) > 1 else None
pb = int(sys.argv[2]) if len(sys.argv) > 2 else 512
c = config(4)
n = c.n
dev = torch.device('cuda:0')
xy = torch.from_numpy(points_for(c)).to(dev)
w = torch.from_numpy(w_for(c)).to(dev)
ctx = R.Context(0)
opts = R.Opts(eps_peel=c.eps_peel, seed=c.seed, probe_block=pb, peel_f32=1)
K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
F = R.Factor(ctx, xy, K, c.eps_fact, c.leaf, opts=opts)
z = F.sample(w)
F.close()
torch.cuda.synchronize()
t0 = time.time()
r = R.gp_mle_eval(ctx, xy, z, K, c.eps_fact, c.leaf, opts)
t_eval = time.time() - t0
print(f"eval {t_eval:.1f}s ell={r.ell!r} grad={list(r.grad)} trace={[r.diag.trace[i] for i in range(2)]} "
      f"q={[r.diag.q[i] for i in range(2)]}", flush=True)


def ell_at(logdet_only=False, **kw):
    Kx = R.Kernel(c.family, kw.get('rho', c.rho), kw.get('sigma2', c.sigma2), c.nugget, c.alpha, theta=())
    Fx = R.Factor(ctx, xy, Kx, c.eps_fact, c.leaf, opts=opts)
    ld = Fx.logdet()
    if logdet_only:
        Fx.close()
        return ld
    u = Fx.solve(z)
    q = float(torch.dot(z, u))
    Fx.close()
    return -0.5 * q - 0.5 * ld - 0.5 * n * math.log(2 * math.pi)


def rich(f, v, rel=1e-2):
    h = rel * v
    d1 = (f(v + h) - f(v - h)) / (2 * h)
    d2 = (f(v + 2 * h) - f(v - 2 * h)) / (4 * h)
    return (4 * d1 - d2) / 3


names = list(c.theta)
vals = {'rho': c.rho, 'sigma2': c.sigma2}
ell0 = ell_at()
gfd = [rich(lambda x, nm=nm: ell_at(**{nm: x}), vals[nm]) for nm in names]
tfd = [rich(lambda x, nm=nm: ell_at(logdet_only=True, **{nm: x}), vals[nm]) for nm in names]
gerr = [abs(r.grad[i] - gfd[i]) / abs(gfd[i]) for i in range(2)]
terr = [abs(r.diag.trace[i] - tfd[i]) / abs(tfd[i]) for i in range(2)]
rec = {"config": 4, "n": n, "peel_storage": "fp32 (memory-saving mode)", "probe_block": pb,
       "t_eval_s": t_eval, "ell": r.ell, "ell_standalone_factor": ell0, "grad": list(r.grad), "grad_fd": gfd,
       "grad_rel_err": gerr, "trace": [r.diag.trace[i] for i in range(2)], "trace_fd_logdet": tfd,
       "trace_rel_err": terr, "q": [r.diag.q[i] for i in range(2)],
       "peel_cols": [[r.diag.peel[i].cols[l] for l in range(1, r.diag.peel[i].levels + 1)] for i in range(2)],
       "peel_rank_max": [[r.diag.peel[i].rank_max[l] for l in range(1, r.diag.peel[i].levels + 1)] for i in range(2)],
       "stored_bytes": [r.diag.peel[i].stored_bytes for i in range(2)],
       "phases_s": {"factor": r.diag.t_factor, "compress": r.diag.t_compress, "peel": r.diag.t_peel,
                    "total": r.diag.t_total}}
print(json.dumps(rec), flush=True)
if out:
    with open(out, "a") as f:
        f.write(json.dumps(rec) + "\n")

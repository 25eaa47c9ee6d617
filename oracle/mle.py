"""O2 - Alg. 1: l-hat and g-hat through RSF + peeling (oracle; test infrastructure).

  F <- RSF(Sigma, eps_fact)
  l-hat = -1/2 z^T F^-1 z - 1/2 log|F| - n/2 log 2 pi          P:666 with R-O (n/2)
  for each theta_i:
     F_i <- compression of Sigma_i (R-F apply-only)
     t_i <- peel Tr of G = 1/2 (F^-1 F_i + F_i F^-1)           P:671 (R-Z)
     g_i = 1/2 z^T F^-1 F_i F^-1 z - 1/2 t_i
Reading R-G: Sigma_nugget = I (G = F^-1, q = u^T u); Sigma_sigma2 = (Sigma - nugget I)/sigma2
so t_sigma2 = (n - nugget Tr F^-1)/sigma2 and q_sigma2 = (q0 - nugget u^T u)/sigma2.
"""
from __future__ import annotations

import math

import numpy as np

from .kernels import Kernel
from .peel import peel_trace
from .rsf import RSF
from .tree import QuadTree


def make_probe(seed: int, trace_id: int, gen):
    """Adapt an input generator gen(seed, stream, c0, c1, c2, c3) -> N(0,1) to the
    probe(rows, cols, level) interface of peel_trace (counter layout DESIGN.md §4)."""
    def probe(rows, cols, level):
        rows = np.asarray(rows, dtype=np.uint64)
        cols = np.asarray(cols, dtype=np.uint64)
        R, C = np.meshgrid(rows, cols, indexing="ij")
        return gen(seed, 3, R.ravel(), C.ravel(), level, trace_id).reshape(R.shape)
    return probe


def rsf_mle_eval(kern: Kernel, xy, z, eps_fact: float, eps_peel: float, leaf: int,
                 seed: int, gen, *, oversample=8, block=8, diag=None):
    xy = np.asarray(xy, dtype=np.float64)
    z = np.asarray(z, dtype=np.float64)
    n = len(xy)
    tree = QuadTree(xy, leaf)
    F = RSF(kern, xy, eps_fact, leaf, tree=tree)
    u = F.solve(z)
    q0 = float(z @ u)
    ell = -0.5 * q0 - 0.5 * F.logdet - 0.5 * n * math.log(2.0 * math.pi)
    grad, qs, ts = [], [], []
    trinv = None
    info = {}
    for ti, name in enumerate(kern.theta):
        if name in ("sigma2", "nugget"):
            if trinv is None:
                d = {}
                trinv = peel_trace(lambda X: F.solve(X), tree, eps_peel,
                                   make_probe(seed, 100, gen), oversample=oversample,
                                   block=block, diag=d)
                info["inv"] = d
            utu = float(u @ u)
            if name == "nugget":
                q, t = utu, trinv
            else:
                q = (q0 - kern.nugget * utu) / kern.sigma2
                t = (n - kern.nugget * trinv) / kern.sigma2
        else:
            Fi = RSF(kern, xy, eps_fact, leaf, which=name, tree=tree)
            q = float(u @ Fi.apply(u))

            def G(X, Fi=Fi):
                return 0.5 * (F.solve(Fi.apply(X)) + Fi.apply(F.solve(X)))
            d = {}
            t = peel_trace(G, tree, eps_peel, make_probe(seed, ti, gen),
                           oversample=oversample, block=block, diag=d)
            info[name] = d
        qs.append(q)
        ts.append(t)
        grad.append(0.5 * q - 0.5 * t)
    out = dict(ell=ell, grad=np.array(grad), logdet=F.logdet, quad=q0, q=np.array(qs),
               trace=np.array(ts), u=u, info=info, F=F)
    if diag is not None:
        diag.update(out)
    return out

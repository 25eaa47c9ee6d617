"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no kernel evaluation, no
factorization, no trace estimation).  It only turns (config, seed) into
bytes: point coordinates and i.i.d. N(0,1) vectors.  Both the oracle
(`oracle/`) and the CUDA path consume what it produces; neither imports the
other.

Generator: Philox4x32-10 (Salmon et al., SC'11) with the counter layouts
documented in DESIGN.md §4 ("input recipe").  The CUDA library implements the
same generator independently for its peeling probes (stream 3); the oracle
receives probes from `philox_normal` below as an input.

Config recipes follow BASELINE.json `configs` and SURVEY.md §8(d) readings
R-T (jittered grid), R-U (clipping = resampling), R-W (seeds/streams).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "philox4x32", "philox_uniform_pair", "philox_normal_pair", "philox_normal", "philox_rademacher",
    "CONFIGS", "Config", "points_for", "w_for", "config", "paper_grid_points", "frozen_z", "DATA_DIR",
    "separable_axes", "SEED_SEPARABLE",
]

_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = np.uint64(0x9E3779B9)
_W1 = np.uint64(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)

SEED_BASE = 1603080570  # R-W: seed_k = SEED_BASE + k
STREAM_POINTS, STREAM_MIXTURE, STREAM_W, STREAM_PROBES, STREAM_HUTCH = 0, 1, 2, 3, 4


def philox4x32(c0, c1, c2, c3, k0: int, k1: int):
    """Philox4x32-10 on arrays of 32-bit counters (held in uint64 arrays).

    Returns four uint64 arrays holding 32-bit outputs.
    """
    c0 = np.asarray(c0, dtype=np.uint64) & _MASK
    c1 = np.broadcast_to(np.asarray(c1, dtype=np.uint64) & _MASK, c0.shape)
    c2 = np.broadcast_to(np.asarray(c2, dtype=np.uint64) & _MASK, c0.shape)
    c3 = np.broadcast_to(np.asarray(c3, dtype=np.uint64) & _MASK, c0.shape)
    k0 = np.uint64(k0 & 0xFFFFFFFF)
    k1 = np.uint64(k1 & 0xFFFFFFFF)
    for r in range(10):
        if r > 0:
            k0 = (k0 + _W0) & _MASK
            k1 = (k1 + _W1) & _MASK
        p0 = _M0 * c0
        p1 = _M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0), lo1, (hi0 ^ c3 ^ k1), lo0
    return c0, c1, c2, c3


def _u53(a, b):
    """Two 32-bit words -> double in [0, 1) with 53 random bits."""
    return ((a >> np.uint64(5)).astype(np.float64) * 67108864.0
            + (b >> np.uint64(6)).astype(np.float64)) * (1.0 / 9007199254740992.0)


def philox_uniform_pair(c0, c1, c2, c3, k0, k1):
    x0, x1, x2, x3 = philox4x32(c0, c1, c2, c3, k0, k1)
    return _u53(x0, x1), _u53(x2, x3)


def philox_normal_pair(c0, c1, c2, c3, k0, k1):
    """Box-Muller on one Philox block: two independent N(0,1)."""
    u1, u2 = philox_uniform_pair(c0, c1, c2, c3, k0, k1)
    r = np.sqrt(-2.0 * np.log1p(-u1))  # 1-u1 in (0, 1]
    t = 2.0 * math.pi * u2
    return r * np.cos(t), r * np.sin(t)


def philox_normal(seed: int, stream: int, c0, c1, c2, c3):
    """The first Box-Muller output for counter (c0,c1,c2,c3): one N(0,1) each.

    This is the probe generator of the peeling step: entry
    (point j, column t) of the level-l probe block of trace number q is
    philox_normal(seed, 3, j, t, l, q).
    """
    n0, _ = philox_normal_pair(c0, c1, c2, c3, seed, stream)
    return n0


def philox_rademacher(seed: int, c0, c1):
    """Rademacher (+-1) entries for the Hutchinson estimator (stream 4, R-W): entry
    (point j, probe p) is +1 if bit 0 of the first Philox4x32-10 output word of counter
    (j, p, 0, 0) under key (seed, 4) is 0, else -1."""
    x0, _, _, _ = philox4x32(c0, c1, 0, 0, seed, STREAM_HUTCH)
    return 1.0 - 2.0 * (x0 & np.uint64(1)).astype(np.float64)


# --------------------------------------------------------------------------
# Configs (BASELINE.json configs[0..4] -> ids 1..5)
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Config:
    cid: int
    n: int
    points: str            # 'uniform' | 'jgrid' | 'clusters'
    family: str            # 'rq' | 'matern12' | 'matern32' | 'matern52' | 'sqexp'
    rho: float
    alpha: float
    sigma2: float
    nugget: float
    theta: tuple           # ordered subset of ('rho','sigma2','nugget','alpha')
    leaf: int
    eps: float             # the configured tolerance (BASELINE.json)
    eps_fact: float        # ID tolerance used (reading R-A / R-B)
    eps_peel: float
    z: str                 # 'dense_chol' | 'rsf_sample'
    extra: dict = field(default_factory=dict)

    @property
    def seed(self) -> int:
        return SEED_BASE + self.cid


CONFIGS = {
    1: Config(1, 1024, "uniform", "rq", 0.1, 1.0, 1.0, 1e-2, ("rho",), 64,
              1e-6, 1e-8, 1e-6, "dense_chol"),
    2: Config(2, 16384, "uniform", "matern32", 0.05, 1.0, 1.0, 1e-3,
              ("rho", "sigma2"), 64, 1e-6, 1e-8, 1e-6, "dense_chol"),
    # eps_fact 1e-11 (R-A): at 1e-8 the sampled full-size solve residual is 1.2e-3 (kappa ~ 1e7
    # with nugget 1e-4); 1e-11 gives 5.7e-6 <= 10 eps (gpurun_out r3)
    3: Config(3, 262144, "jgrid", "rq", 0.02, 1.5, 1.0, 1e-4, ("rho", "alpha"),
              64, 1e-6, 1e-11, 1e-6, "rsf_sample"),
    4: Config(4, 1048576, "clusters", "matern12", 0.01, 1.0, 1.0, 1e-3,
              ("rho", "sigma2"), 64, 1e-6, 1e-8, 1e-6, "rsf_sample",
              {"clusters": 64, "cluster_sigma": 0.03}),
    5: Config(5, 4194304, "uniform", "matern52", 0.005, 1.0, 1.0, 1e-4,
              ("rho", "sigma2", "nugget"), 128, 1e-6, 1e-9, 1e-6, "rsf_sample"),
}


def config(cid: int, **overrides) -> Config:
    c = CONFIGS[cid]
    if overrides:
        d = dict(c.__dict__)
        d.update(overrides)
        c = Config(**d)
    return c


def _uniform_points(n: int, seed: int) -> np.ndarray:
    j = np.arange(n, dtype=np.uint64)
    x, y = philox_uniform_pair(j, 0, 0, 0, seed, STREAM_POINTS)
    return np.stack([x, y], axis=1)


def _jgrid_points(n: int, seed: int) -> np.ndarray:
    m = int(round(math.sqrt(n)))
    assert m * m == n
    p = np.arange(n, dtype=np.uint64)
    u0, u1 = philox_uniform_pair(p, 0, 0, 0, seed, STREAM_POINTS)
    i = (p // np.uint64(m)).astype(np.float64)
    jj = (p % np.uint64(m)).astype(np.float64)
    x = (i + 0.5 + 0.8 * (u0 - 0.5)) / m   # R-T: +-0.4 cell jitter
    y = (jj + 0.5 + 0.8 * (u1 - 0.5)) / m
    return np.stack([x, y], axis=1)


def _cluster_points(n: int, seed: int, nc: int, sig: float) -> np.ndarray:
    c = np.arange(nc, dtype=np.uint64)
    cx, cy = philox_uniform_pair(c, 0, 0, 0, seed, STREAM_MIXTURE)
    out = np.empty((n, 2))
    todo = np.arange(n, dtype=np.uint64)
    attempt = 0
    while todo.size:
        ua, _ = philox_uniform_pair(todo, attempt, 0, 0, seed, STREAM_POINTS)
        k = np.minimum((ua * nc).astype(np.int64), nc - 1)
        g0, g1 = philox_normal_pair(todo, attempt, 1, 0, seed, STREAM_POINTS)
        x = cx[k] + sig * g0
        y = cy[k] + sig * g1
        ok = (x >= 0.0) & (x < 1.0) & (y >= 0.0) & (y < 1.0)   # R-U: resample
        idx = todo[ok].astype(np.int64)
        out[idx, 0] = x[ok]
        out[idx, 1] = y[ok]
        todo = todo[~ok]
        attempt += 1
    return out


def paper_grid_points(m: int) -> np.ndarray:
    """The paper's gridded workload: an m x m grid uniformly discretizing
    [0, 100]^2, rescaled to the unit square (reading R-f1: cell centres ((i + 1/2)/m,
    (j + 1/2)/m); theta = [10, 7] on [0, 100]^2 is [0.1, 0.07] here)."""
    g = (np.arange(m, dtype=np.float64) + 0.5) / m
    return np.stack([np.repeat(g, m), np.tile(g, m)], axis=1)


SEED_SEPARABLE = SEED_BASE + 7   # the P7 separable surrogate (R-W numbering: configs use 1..5)


def separable_axes(m: int, seed: int = SEED_SEPARABLE):
    """Axis coordinates of the P7 tensor-grid surrogate at config 3's size and density:
    a_i = (i + 1/2 + 0.8 (u_i - 1/2)) / m (the +-0.4-cell jitter of R-T, applied per axis so
    that the grid stays a tensor product), u from Philox stream 0, counters (i, 1, 0, 0) for
    a and (i, 2, 0, 0) for b.  Point (i, j) of the grid is (a_i, b_j), index i * m + j."""
    i = np.arange(m, dtype=np.uint64)
    ua, _ = philox_uniform_pair(i, 1, 0, 0, seed, STREAM_POINTS)
    ub, _ = philox_uniform_pair(i, 2, 0, 0, seed, STREAM_POINTS)
    g = np.arange(m, dtype=np.float64) + 0.5
    return (g + 0.8 * (ua - 0.5)) / m, (g + 0.8 * (ub - 0.5)) / m


def points_for(cfg: Config, n: int | None = None) -> np.ndarray:
    """n x 2 float64 coordinates in [0,1)^2 (row-major), deterministic."""
    n = cfg.n if n is None else n
    if cfg.points == "uniform":
        return _uniform_points(n, cfg.seed)
    if cfg.points == "jgrid":
        return _jgrid_points(n, cfg.seed)
    if cfg.points == "clusters":
        return _cluster_points(n, cfg.seed, cfg.extra.get("clusters", 64),
                               cfg.extra.get("cluster_sigma", 0.03))
    raise ValueError(cfg.points)


def w_for(cfg: Config, n: int | None = None, stream: int = STREAM_W) -> np.ndarray:
    """i.i.d. N(0,1) vector of length n (the w in z = L w or z = F^{1/2} w)."""
    n = cfg.n if n is None else n
    m = (n + 1) // 2
    c = np.arange(m, dtype=np.uint64)
    n0, n1 = philox_normal_pair(c, 0, 0, 0, cfg.seed, stream)
    w = np.empty(2 * m)
    w[0::2] = n0
    w[1::2] = n1
    return w[:n].copy()


DATA_DIR = __import__("os").path.join(__import__("os").path.dirname(__import__("os").path.abspath(__file__)), "data")


def frozen_z(cid: int) -> np.ndarray:
    """The frozen observation vector of config `cid` (reading R-V): bytes written once by
    tools/make_frozen_z.py from the O2 oracle, verified against the SHA-256 in
    data/MANIFEST.json.  Raises if the file is missing or its hash does not match."""
    import hashlib
    import json
    import os
    man = json.load(open(os.path.join(DATA_DIR, "MANIFEST.json")))[str(cid)]
    raw = open(os.path.join(DATA_DIR, man["file"]), "rb").read()
    h = hashlib.sha256(raw).hexdigest()
    if h != man["sha256"]:
        raise ValueError(f"frozen z of config {cid}: sha256 {h} != manifest {man['sha256']}")
    z = np.frombuffer(raw, dtype="<f8").astype(np.float64)
    if z.size != man["n"]:
        raise ValueError(f"frozen z of config {cid}: {z.size} values, manifest says {man['n']}")
    return z

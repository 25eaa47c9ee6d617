#!/usr/bin/env python
"""Freeze the observation vector z of configs 3-5 (reading R-V) as bytes + SHA-256.

    python tools/make_frozen_z.py 3 [4 ...]

z = F^{1/2} w with F the O2 oracle's RSF of Sigma (oracle/rsf.py) at the
config's eps_fact and w = workloads.w_for(config) (Philox stream 2).  Only `oracle/`
and `workloads/` are called: no value comes from the CUDA path.  Output:
workloads/data/z_config<k>.f64 (little-endian float64, original point order) and
workloads/data/MANIFEST.json (n, eps_fact, sha256, generator, seconds).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle.kernels import Kernel  # noqa: E402
from oracle.rsf import RSF  # noqa: E402
from workloads import DATA_DIR, config, points_for, w_for  # noqa: E402


def main(ids):
    os.makedirs(DATA_DIR, exist_ok=True)
    man_p = os.path.join(DATA_DIR, "MANIFEST.json")
    man = json.load(open(man_p)) if os.path.exists(man_p) else {}
    for cid in ids:
        c = config(cid)
        xy, w = points_for(c), w_for(c)
        k = Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
        t = time.time()
        F = RSF(k, xy, c.eps_fact, c.leaf)
        z = np.ascontiguousarray(F.sqrt(w), dtype="<f8")
        dt = time.time() - t
        fn = f"z_config{cid}.f64"
        z.tofile(os.path.join(DATA_DIR, fn))
        man[str(cid)] = {"file": fn, "n": c.n, "eps_fact": c.eps_fact,
                         "sha256": hashlib.sha256(z.tobytes()).hexdigest(),
                         "generator": "oracle.rsf.RSF(...).sqrt(workloads.w_for(config)) (O2, P:385-388, R-V)",
                         "logdet_O2": F.logdet, "top_size": int(len(F.I0)), "seconds": round(dt, 1)}
        json.dump(man, open(man_p, "w"), indent=1, sort_keys=True)
        print(cid, man[str(cid)], flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [3])

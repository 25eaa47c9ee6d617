#!/usr/bin/env python
"""Host-core timing study of the oracle (the cpu_baseline of bench.py):
O2 (numpy/scipy RSF + weak peeling, one full l+g evaluation of config 3's recipe) at several n,
at all cores and at 1 thread (OMP/OpenBLAS/MKL thread caps set before numpy loads), and O1
(dense Cholesky + explicit inverse) at configs 1 and 2.  One JSON line per measurement, then a
power-law fit per thread count.

    python tools/oracle_timing.py [--threads all|1] [--sizes 576,1024,2304] [--o1]
"""
import argparse
import json
import math
import os
import subprocess
import sys
import time

ap = argparse.ArgumentParser()
ap.add_argument("--threads", default="all")
ap.add_argument("--sizes", default="576,1024,2304")
ap.add_argument("--o1", action="store_true")
args = ap.parse_args()
if args.threads != "all":
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "NUMEXPR_NUM_THREADS"):
        os.environ[k] = args.threads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle.dense import dense_eval, dense_sample  # noqa: E402
from oracle.kernels import Kernel  # noqa: E402
from oracle.mle import rsf_mle_eval  # noqa: E402
from workloads import config, philox_normal, points_for, w_for  # noqa: E402

cores = len(os.sched_getaffinity(0))
pts = []
c = config(3)
ok = Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
for n in [int(x) for x in args.sizes.split(",") if x]:
    xy, w = points_for(c, n), w_for(c, n)
    t = time.perf_counter()
    rsf_mle_eval(ok, xy, w, c.eps_fact, c.eps_peel, c.leaf, c.seed, philox_normal, block=8)
    dt = time.perf_counter() - t
    pts.append((n, dt))
    print(json.dumps({"oracle": "O2", "config": 3, "n": n, "threads": args.threads, "cores": cores, "seconds": dt}),
          flush=True)
if len(pts) >= 2:
    b, la = np.polyfit(np.log([p[0] for p in pts]), np.log([p[1] for p in pts]), 1)
    print(json.dumps({"fit": "O2 t = a n^b", "threads": args.threads, "b": b, "a": math.exp(la),
                      "extrapolated_s_at_262144": math.exp(la) * 262144 ** b}), flush=True)
if args.o1:
    for cid in (1, 2):
        cc = config(cid)
        xy = points_for(cc)
        k = Kernel(cc.family, cc.rho, cc.sigma2, cc.nugget, cc.alpha, cc.theta)
        z = dense_sample(k, xy, w_for(cc))
        t = time.perf_counter()
        dense_eval(k, xy, z)
        print(json.dumps({"oracle": "O1", "config": cid, "n": cc.n, "threads": args.threads, "cores": cores,
                          "seconds": time.perf_counter() - t}), flush=True)
try:
    print(json.dumps({"lscpu": subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines()[:16]}))
except Exception:
    pass

#!/usr/bin/env python
"""HBM roofline of the 1-RHS solve (north star: achieved HBM GB/s for the solves).

    python tools/solve_bw.py [config] [nrhs ...]

Builds the config's Sigma factor through the C ABI and times F^-1 X on nrhs internal-layout
columns (rsf_debug_solve_bench: CUDA events on the library stream, mean of 20 after one
warm-up).  Bytes = the algorithmic bytes of one 1-RHS solve x nrhs is NOT
claimed: for nrhs > 1 the factor is read once per sweep, so GB/s counts factor bytes once."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1603_08057_b200 as R  # noqa: E402
from workloads import config, points_for  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ks = [int(a) for a in sys.argv[2:]] or [1, 8, 64]
c = config(cid)
ctx = R.Context(0)
xy = torch.from_numpy(points_for(c)).cuda()
K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
F = R.Factor(ctx, xy, K, c.eps_fact, c.leaf)
info = F.info()
hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6540.2
for k in ks:
    b = C.c_double()
    t = R.lib.rsf_debug_solve_bench(F.h, k, int(os.environ.get("SOLVE_REPS", "20")), C.byref(b))
    if t <= 0:
        print("error", t, R.lib.rsf_last_error().decode(), flush=True)
        continue
    print(json.dumps({"config": cid, "nrhs": k, "seconds": t, "bytes_1rhs": b.value,
                      "GBps": b.value / t / 1e9, "frac_hbm": b.value / t / 1e9 / hbm,
                      "factor_bytes": info.factor_bytes, "levels": info.levels, "top": info.top_size}), flush=True)
    if os.environ.get("RSF_KTRACE") == "1":
        rows = [x.rsplit("=", 1) for x in R.lib.rsf_trace_dump().decode().split(";") if "=" in x]
        rows = sorted(((float(v.split(",")[0]), k, v) for k, v in rows), reverse=True)[:25]
        for sec, k, v in rows:
            print(f"   {sec * 1e3:9.3f} ms  {k}  {v}", flush=True)
        R.lib.rsf_profile_reset()

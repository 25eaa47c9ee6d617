#!/usr/bin/env python
"""bench.py -- l(theta)+g(theta) evaluations per second through the CUDA path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cuda|reference]
                    [--config 4] [--n N]

A "step" is one full evaluation of Alg. 1 -- quadtree, RSF of
Sigma, compression of each Sigma_i, solve, and the peeled traces -- at the
largest BASELINE.json workload that fits one B200 (config 3: n = 262,144
jittered-grid points, rational quadratic, theta = (rho, alpha), z frozen from
the O2 oracle); the metric's own config 4 (n = 2^20) fits one GPU only in the
memory-saving mode at ~230 s per evaluation (`--config 4`, DESIGN.md §7g;
profiles/r02_bench_config4_v2.json), too long for a default W >= 3 run.  Inputs
are resident in HBM.
Multi-GPU (torchrun): the ranks form one NCCL group and share every evaluation
(factor replicated, peeling probe columns split, one all-gather per probe
block) -- strong scaling, time = max over ranks, value =
evaluations / time.

--impl reference times the CPU oracle (oracle/, the only other place bench.py
runs it) on rank 0 on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "l+g evals/sec at n=2^20 (1/2/4/8 B200); RSF FP64 TFLOP/s vs peak"
UNIT = "evals/s"
# FP64 FMA-pipe peak derived from unit counts and clocks:
# 148 SMs x 64 FP64 FMA/clk x 2 flop x 1.965 GHz
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.th = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.th:
            self.th.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax.append(float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def aggregate(t_local: float, steps: int, world: int, device=None, strong: bool = False):
    """Max-over-ranks time and whole-job throughput.  strong: the ranks share each of the
    `steps` evaluations (probe columns split across ranks) -> steps / time;
    else every rank evaluates `steps` independent replicas -> world * steps / time.
    Used by the timed region and by tests/test_multirank.py."""
    t_all = t_local
    if world > 1:
        import torch
        import torch.distributed as dist
        tt = torch.tensor([t_local], dtype=torch.float64, device=device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_all = float(tt.item())
    return t_all, (steps if strong else world * steps) / t_all


def _hbm_peak():
    """(GB/s, source): MEASURED_PEAKS.json's measured copy bandwidth, else the profiling guide's
    fallback figure."""
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    except Exception:
        return 6540.2, "fallback: the measured B200 copy bandwidth of round 1 (MEASURED_PEAKS.json absent)"


def workload(cid: int, n: int | None):
    from workloads import config, points_for, w_for
    c = config(cid)
    n = n or c.n
    return c, n, points_for(c, n), w_for(c, n)


# O2 sample sizes of config 3's recipe (square grids: 24^2, 32^2, 40^2); the time of one l+g
# evaluation is fitted as t = a n^b over the measured points (least squares in log-log) and
# extrapolated to the workload's n with the FITTED exponent b (round 1 assumed the paper's 1.6)
REF_SIZES = (1024, 2304, 4096)
# BLAS threads of the oracle: 1.  Measured on the GPU box's 16-core host (profiles/
# r02_oracle_timing.jsonl): O2 at n = 576 / 1024 / 2304 takes 0.40 / 1.1 / 6.4 s on one thread and
# 5.6 / 7.6 / 34.6 s with the BLAS on all 16 cores (thread overhead on its small dense blocks), so
# the single-threaded oracle is the faster baseline at every size it can run in the bench.
REF_THREADS = 1


def _o2_eval_seconds(args, c, n_s):
    from threadpoolctl import threadpool_limits

    from oracle.kernels import Kernel as OK
    from oracle.mle import rsf_mle_eval
    from workloads import philox_normal
    _, _, xy, w = workload(args.config, n_s)
    ok = OK(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    with threadpool_limits(REF_THREADS):
        t = time.perf_counter()
        # z = w: a valid observation vector for timing (the time does not depend on z)
        rsf_mle_eval(ok, xy, w, c.eps_fact, c.eps_peel, c.leaf, c.seed, philox_normal, block=8)
        return time.perf_counter() - t


def _fit_and_extrapolate(pts, n_full):
    """pts: [(n, seconds)].  Least-squares fit of log t = log a + b log n."""
    ns = np.log([p[0] for p in pts])
    ts = np.log([p[1] for p in pts])
    if len(set(p[0] for p in pts)) >= 2:
        b, la = np.polyfit(ns, ts, 1)
    else:
        b, la = 1.6, float(np.mean(ts - 1.6 * ns))   # one size only: the paper's n^1.6
    return float(math.exp(la) * n_full ** b), float(b)


def _host_info():
    info = {"cores": len(os.sched_getaffinity(0))}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            k, _, v = ln.partition(":")
            if k.strip() in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core"):
                info[k.strip()] = v.strip()
    except Exception:
        pass
    try:
        import numpy.__config__  # noqa: F401
        info["blas_threads"] = os.environ.get("OMP_NUM_THREADS", "all cores (unset)")
    except Exception:
        pass
    return info


def run_reference(args, rank):
    """CPU oracle (O2: serial numpy RSF + weak peeling), rank 0 only: every step is one full
    l+g evaluation of config 3's recipe at a sample size (cycling through REF_SIZES; warm-up
    steps at the smallest), the points are fitted by a power law and extrapolated."""
    if rank != 0:
        return
    c, n_full, _, _ = workload(args.config, args.n)
    for _ in range(args.warmup):
        _o2_eval_seconds(args, c, 576)
    pts = []
    for it in range(args.steps):
        n_s = REF_SIZES[it % len(REF_SIZES)]
        pts.append((n_s, _o2_eval_seconds(args, c, n_s)))
    t_full, b = _fit_and_extrapolate(pts, n_full)
    value = 1.0 / t_full
    host = _host_info()
    meas = {str(n): float(np.median([t for m, t in pts if m == n])) for n in sorted(set(m for m, _ in pts))}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_full * 1e3,
        "higher_is_better": True, "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": _config_dict(c, n_full, args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": REF_THREADS, "kind": "oracle",
                         "sample": f"O2 oracle (numpy/scipy RSF + weak peeling, BLAS on {REF_THREADS} thread of "
                                   f"the {host['cores']}-core host: faster than all cores at these sizes) "
                                   f"full l+g evaluations of config {c.cid}'s recipe at "
                                   f"n = {', '.join(meas)} (median seconds {meas}); fitted t ~ n^{b:.2f}; "
                                   f"value = extrapolation to n = {n_full} with the fitted exponent",
                         "measured_points": pts, "fitted_exponent": b, "host": host},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _config_dict(c, n, args):
    return {"workload": f"config{c.cid}: n={n} {c.points} points, {c.family}, rho={c.rho}, "
                        f"nugget={c.nugget}, theta={list(c.theta)}, leaf={c.leaf}",
            "n": n, "eps": c.eps, "eps_fact": c.eps_fact, "eps_peel": c.eps_peel, "leaf": c.leaf,
            "theta": list(c.theta),
            "parallelism": (f"sharded x{args.gpus}: factor replicated, peeling probe columns split, NCCL "
                            "all-gather per probe block" if args.gpus > 1 else "1 GPU"),
            "l2": "working set (factor + probe blocks, GBs) >> 126 MB L2; no flush",
            "peel_storage": ("fp32 (memory-saving mode: peeled bases and cores stored in FP32, FP64 arithmetic; "
                             "serial trace jobs; DESIGN.md §7g)" if getattr(args, "_peel_f32", 0) else "fp64")}


def cpu_baseline_sample(args, c):
    """The oracle as it stands on a bounded sample (rank 0, N=1 only): one O2 evaluation at
    each of REF_SIZES (about 20 s of CPU work), power-law fit, labeled extrapolation."""
    pts = [(n_s, _o2_eval_seconds(args, c, n_s)) for n_s in REF_SIZES]
    n_full = args.n or c.n
    t_full, b = _fit_and_extrapolate(pts, n_full)
    host = _host_info()
    return {"value": 1.0 / t_full, "unit": UNIT, "cores": REF_THREADS, "kind": "oracle",
            "sample": f"O2 oracle (numpy/scipy RSF + weak peeling, BLAS on {REF_THREADS} thread of the "
                      f"{host['cores']}-core host) one full l+g evaluation of config {c.cid}'s "
                      f"recipe at each n in {list(REF_SIZES)}: {[round(t, 2) for _, t in pts]} s; fitted "
                      f"t ~ n^{b:.2f}; value = extrapolation to n = {n_full} with the fitted exponent "
                      f"(profiles/ has the 1-thread / all-core study at larger n)",
            "measured_points": pts, "fitted_exponent": b, "host": host}


# ncu --set full of the longest launch of the dominant kernel (profiles/r01_gemm_pipe_ncu_v4.txt)
TRAFFIC_BYTES = 4.1665e9 + 0.7543e9
TRAFFIC_NOTE = ("dram__bytes_read.sum + dram__bytes_write.sum of the longest gemm_pipe_kernel launch of an "
                "evaluation (peeling subtraction at level 1, 13.76 ms, 12288 CTAs, DMMA pipe 85 % busy); "
                "its compulsory bytes are ~5.6e9 (V_i of three level-1 boxes 4.2 GB + the Y' block read "
                "and written), so operands are not re-read from DRAM; re-captured on the final round-2 "
                "build with the same figures (profiles/r02_gemm_sub_ncu_final.txt: 4.16 GB read + 0.754 GB "
                "written, 13.78 ms, DMMA 84.8 %)")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    # N=1 workload: config 3 (n = 262,144), the largest BASELINE config that fits one B200;
    # config 4 (n = 2^20, the metric's config, tagged "8-GPU subdomain sharding") needs more
    # than one GPU's 180 GB for its weak-peeling bases (gpurun_out r5 / profiles)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--ref-n", type=int, default=2304)   # 48 x 48 (config 3's grid needs a square)
    ap.add_argument("--ref-budget", type=float, default=120.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # memory-saving mode (FP32-stored peeled levels, serial trace jobs): the default
    # for config 4 (n = 2^20), whose FP64 peeled representation exceeds one B200's 180 GB
    ap.add_argument("--peel-f32", type=int, default=None)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist
    import paper_1603_08057_b200 as R
    from workloads import config

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    c, n, xy_h, w_h = workload(args.config, args.n)
    # N > 1: ONE evaluation shared by the group (probe columns split, NCCL all-gather per
    # probe block) -- strong scaling, the same inputs and seed on every rank
    ctx = R.Context.from_process_group(local) if world > 1 else R.Context(local)
    K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
    peel_f32 = args.peel_f32 if args.peel_f32 is not None else int((args.n or c.n) >= (1 << 20))
    opts = R.Opts(eps_peel=c.eps_peel, seed=c.seed, peel_f32=peel_f32)
    args._peel_f32 = peel_f32
    xy = torch.from_numpy(xy_h).to(dev)
    w = torch.from_numpy(w_h).to(dev)
    # z (reading R-V): config 3's frozen bytes (O2 oracle F^{1/2} w, SHA-256 checked); configs
    # without frozen bytes sample z = F^{1/2} w through the CUDA path before timing (labeled)
    try:
        from workloads import frozen_z
        z_h = frozen_z(c.cid) if args.n in (None, c.n) else None
        z_src = "frozen (workloads/data, O2 F^{1/2} w, sha256-checked)" if z_h is not None else None
    except (FileNotFoundError, KeyError):
        z_h = None
    if z_h is not None:
        z = torch.from_numpy(z_h).to(dev)
    else:
        F = R.Factor(ctx, xy, K, c.eps_fact, c.leaf, opts=opts)
        z = F.sample(w)
        F.close()
        z_src = "F^{1/2} w from the CUDA factor before timing (not frozen)"
    torch.cuda.synchronize()

    def step(xyb, zb):
        return R.gp_mle_eval(ctx, xyb, zb, K, c.eps_fact, c.leaf, opts)

    for _ in range(args.warmup):
        r = step(xy, z)
    torch.cuda.synchronize()
    barrier()

    # live roofline denominator: FP64 DMMA.8x8x4 peak on this GPU at its current clocks
    # (MEASURED_PEAKS.json carries no FP64 figure)
    fp64_peak = R.lib.rsf_debug_fp64_peak(1, 3)
    fp64_peak_dfma = R.lib.rsf_debug_fp64_peak(0, 3)

    # ---- timed region: device-resident inputs, no instrumentation
    clk = ClockSampler(local)
    clk.start()
    l0 = R.kernel_launches()
    torch.cuda.synchronize()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    diags = []
    for _ in range(args.steps):
        r = step(xy, z)
        diags.append(r.diag)
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    barrier()
    clocks = clk.stop()
    launches = R.kernel_launches() - l0
    # the library synchronises its own stream at the end of every evaluation, so the
    # wall time brackets exactly the device work; torch events on the default stream
    # see only the torch part, hence max(device-synchronised wall, event time)
    ev_ms = e0.elapsed_time(e1)
    t_local = max(wall, ev_ms / 1e3)
    t_all, value = aggregate(t_local, args.steps, world, dev, strong=world > 1)

    # ---- one more step with the GEMM statistics on (events around every batched-GEMM launch,
    # on its own stream): the roofline numbers, kept out of the timed steps above
    R.lib.rsf_stats_reset()
    R.lib.rsf_stats_enable(1)
    torch.cuda.synchronize()
    ts0 = time.perf_counter()
    step(xy, z)
    torch.cuda.synchronize()
    t_stat = time.perf_counter() - ts0
    R.lib.rsf_stats_enable(0)
    st = (R.C if hasattr(R, "C") else __import__("ctypes")).c_double * 4
    stats = st()
    R.lib.rsf_stats_get(stats)

    # ---- 1-RHS solve on the HBM roofline (north star: "achieved HBM GB/s for the solves"):
    # device time of F^-1 z sweeps of the full Sigma factor, algorithmic bytes per solve
    solve_rl = None
    factor_rl = None
    try:
        Fs = R.Factor(ctx, xy, K, c.eps_fact, c.leaf, opts=opts)   # warm (allocations cached)
        Fs.close()
        Fs = R.Factor(ctx, xy, K, c.eps_fact, c.leaf, opts=opts)
        fi = Fs.info()
        fl = fi.flops_id + fi.flops_elim + fi.flops_top
        peak64 = fp64_peak if fp64_peak > 0 else FP64_PEAK_TFLOPS
        factor_rl = {"bound": "fp64", "achieved": fl / fi.seconds / 1e12, "peak": peak64, "unit": "TFLOP/s",
                     "frac": fl / fi.seconds / 1e12 / peak64, "seconds": fi.seconds, "flops": fl,
                     "what": f"RSF of config {c.cid}'s Sigma alone (rsf_factor, full factor with L for apply), its own "
                             "device-synchronised time (not overlapped with the compressions); algorithmic flops "
                             "of DESIGN.md §5 (ID + elimination + top Cholesky)"}
        nb = __import__("ctypes").c_double()
        t_solve = R.lib.rsf_debug_solve_bench(Fs.h, 1, 20, __import__("ctypes").byref(nb))
        Fs.close()
        if t_solve > 0:
            hbm = _hbm_peak()
            ach = nb.value / t_solve / 1e9
            solve_rl = {"bound": "hbm", "achieved": ach, "peak": hbm[0], "unit": "GB/s", "frac": ach / hbm[0],
                        "peak_source": hbm[1], "seconds_per_solve": t_solve, "bytes_per_solve": nb.value,
                        "what": f"one F^-1 z (k = 1) of config {c.cid}'s Sigma factor, forward + backward sweeps; "
                                "bytes = 2 x (T, E, L^-1 of every box + C^-1) + active-DOF vector traffic "
                                "(DESIGN.md §5); CUDA events, mean of 20"}
    except Exception as e:  # diagnostics only
        solve_rl = {"error": str(e)}

    # ---- e2e: same metric through the C ABI with pinned HOST buffers (H2D inside the call)
    xy_p = torch.from_numpy(xy_h).pin_memory()
    z_p = z.cpu().pin_memory()
    torch.cuda.synchronize()
    barrier()
    e2e_steps = 1   # one host-buffer evaluation (each is minutes at config 4)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        step(xy_p, z_p)
    torch.cuda.synchronize()
    te, e2e_value = aggregate(time.perf_counter() - t0, e2e_steps, world, dev, strong=world > 1)
    e2e = {"value": e2e_value, "unit": UNIT,
           "h2d_bytes_per_step": int(xy_h.nbytes + z_p.numel() * 8),
           "d2h_bytes_per_step": int(8 * (1 + len(c.theta)))}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    d = diags[-1]
    gl, gsec, gfl, gby = stats[0], stats[1], stats[2], stats[3]
    achieved = gfl / gsec / 1e12 if gsec > 0 else 0.0
    peak = fp64_peak if fp64_peak > 0 else FP64_PEAK_TFLOPS
    roofline = {"bound": "tensor", "kernel": "gemm_pipe_kernel (variable-size batched FP64 GEMM on "
                                             "DMMA.8x8x4: RSF sweeps of the G applies, peeling bases, "
                                             "Schur/WY updates)",
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "peak_source": ("measured live: FP64 DMMA.8x8x4 micro-benchmark (rsf_debug_fp64_peak) "
                                f"{fp64_peak:.2f} TFLOP/s, DFMA {fp64_peak_dfma:.2f}; no FP64 figure in "
                                "MEASURED_PEAKS.json; nominal 148 SM x 64 FMA/clk x 2 x 1.965 GHz = "
                                f"{FP64_PEAK_TFLOPS:.1f}"),
                # DRAM bytes of one representative dominant launch (ncu --set full, see the note)
                "traffic": TRAFFIC_BYTES, "traffic_note": TRAFFIC_NOTE,
                "launches": int(gl), "kernel_seconds": gsec,
                "timing": "CUDA events around every launch on its stream; kernel_seconds = length of the "
                          "union of the launch intervals (the trace jobs run on concurrent streams, so "
                          "summed durations would double-count overlap)",
                "share_of_step": gsec / t_stat if t_stat > 0 else None,
                "stats_pass": "one extra evaluation after the timed steps with rsf_stats_enable(1) "
                              f"({t_stat:.2f} s); the timed steps ran uninstrumented",
                "algorithmic_flops_per_launch": gfl / gl if gl else None}
    line = {
        "metric": METRIC,
        "metric_note": ("BASELINE.json quotes this metric at n = 2^20 (config 4). Config 4 runs on one B200 "
                        "only in the memory-saving mode (FP32-stored peeled levels, DESIGN.md §7g) at ~230 s "
                        "per evaluation, so a W >= 3 run takes ~25 min; the default line measures config 3 "
                        "(FP64 storage throughout, named in config.workload) and `bench.py --config 4` gives "
                        "the config-4 line (profiles/r02_bench_config4_v2.json: 0.00438 evals/s)"
                        if (args.n or c.n) != 1048576 else
                        "config 4 (n = 2^20), the metric's own workload, memory-saving mode (DESIGN.md §7g)"),
        "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_all / args.steps, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config_dict(c, n, args), "clocks": clocks, "gpu_launches": int(launches),
        "e2e": e2e, "roofline": roofline, "solve_roofline": solve_rl, "factor_roofline": factor_rl,
        "phases_s": {"tree": d.t_tree, "factor": d.t_factor, "compress": d.t_compress,
                     "solve": d.t_solve, "peel": d.t_peel, "jobs_wall": d.t_jobs_wall, "total": d.t_total,
                     "note": f"compress/solve/peel are sums over the {d.jobs} trace jobs, which ran "
                             f"{'concurrently' if d.concurrent else 'serially'} (jobs_wall: their wall time)"},
        "peel_levels": [{"theta": c.theta[i],
                         "cols": [d.peel[i].cols[l] for l in range(1, d.peel[i].levels + 1)],
                         "rank_min": [d.peel[i].rank_min[l] for l in range(1, d.peel[i].levels + 1)],
                         "rank_med": [d.peel[i].rank_med[l] for l in range(1, d.peel[i].levels + 1)],
                         "rank_max": [d.peel[i].rank_max[l] for l in range(1, d.peel[i].levels + 1)],
                         "stored_GB": d.peel[i].stored_bytes / 1e9} for i in range(len(c.theta))],
        "serial_fallback": int(d.serial_fallback),
        "ell": r.ell, "grad": r.grad, "z": z_src,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample(args, c)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""ctypes declarations of include/rsf.h (argument marshalling only).

The product path has no fallback: if librsf.so is missing or fails to load,
importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librsf.so")

RSF_OK, RSF_EINVAL, RSF_ENUMERIC, RSF_ECUDA, RSF_ENOMEM, RSF_ENCCL = range(6)
FAMILY = {"rq": 0, "matern12": 1, "matern32": 2, "matern52": 3, "sqexp": 4}
PARAM = {"rho": 0, "sigma2": 1, "nugget": 2, "alpha": 3, "rho2": 4}


class rsf_kernel(C.Structure):
    _fields_ = [("family", C.c_int32), ("rho", C.c_double), ("sigma2", C.c_double),
                ("nugget", C.c_double), ("alpha", C.c_double), ("p", C.c_int32),
                ("theta", C.c_int32 * 4), ("rho2", C.c_double)]


class rsf_opts(C.Structure):
    _fields_ = [("eps_peel", C.c_double), ("oversample", C.c_int32), ("probe_block", C.c_int32),
                ("peel_start", C.c_int32), ("max_depth", C.c_int32), ("r_near", C.c_double),
                ("r_in", C.c_double), ("r_out", C.c_double), ("seed", C.c_uint64), ("strong", C.c_int32),
                ("peel_f32", C.c_int32)]


class rsf_fact_diag(C.Structure):
    _fields_ = [("levels", C.c_int32), ("top_size", C.c_int32),
                ("level_boxes", C.c_int32 * 32), ("level_active", C.c_int32 * 32),
                ("level_skel", C.c_int32 * 32), ("level_maxI", C.c_int32 * 32),
                ("flops_id", C.c_double), ("flops_elim", C.c_double), ("flops_top", C.c_double),
                ("factor_bytes", C.c_double), ("seconds", C.c_double)]


class rsf_peel_diag(C.Structure):
    _fields_ = [("levels", C.c_int32), ("cols", C.c_int32 * 32), ("rank_max", C.c_int32 * 32),
                ("nL", C.c_int32), ("cancellation", C.c_double), ("applies", C.c_double),
                ("seconds", C.c_double), ("rank_min", C.c_int32 * 32), ("rank_med", C.c_int32 * 32),
                ("stored_bytes", C.c_double)]


class rsf_eval_diag(C.Structure):
    _fields_ = [("logdet", C.c_double), ("quad", C.c_double), ("q", C.c_double * 4),
                ("trace", C.c_double * 4), ("t_tree", C.c_double), ("t_factor", C.c_double),
                ("t_compress", C.c_double), ("t_solve", C.c_double), ("t_peel", C.c_double),
                ("t_total", C.c_double), ("flops_factor", C.c_double),
                ("kernel_launches", C.c_double), ("fact", rsf_fact_diag),
                ("peel", rsf_peel_diag * 4), ("t_jobs_wall", C.c_double), ("jobs", C.c_int32),
                ("concurrent", C.c_int32), ("serial_fallback", C.c_int32), ("groups", C.c_int32)]


EXPORTS = ["rsf_opts_default", "rsf_ctx_create", "rsf_ctx_destroy", "rsf_factor", "rsf_fact_destroy",
           "rsf_fact_info", "rsf_logdet", "rsf_solve", "rsf_apply", "rsf_sample", "peel_trace", "hutch_trace", "gp_profile_eval", "gp_cond_mean",
           "gp_mle_eval", "rsf_last_error", "rsf_kernel_launches", "rsf_profile_dump",
           "rsf_profile_reset", "rsf_stats_enable", "rsf_stats_get", "rsf_stats_reset",
           "rsf_debug_gemm_bench", "rsf_debug_fp64_peak", "rsf_trace_dump", "rsf_debug_gemm_log",
           "rsf_debug_gemm", "rsf_ctx_wait_stream", "rsf_nccl_unique_id", "rsf_ctx_create_group",
           "rsf_ctx_group", "rsf_debug_col_slice", "rsf_debug_solve_bench",
           "rsf_debug_job_runs", "gp_cond_sample", "rsf_debug_job_group", "rsf_debug_nccl_calls"]


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -m paper_1603_08057_b200.build` "
                          "(the CUDA library is required; there is no fallback)")
    lib = C.CDLL(path)
    vp, i32, i64, dp = C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double)
    lib.rsf_opts_default.argtypes = [C.POINTER(rsf_opts)]
    lib.rsf_opts_default.restype = None
    lib.rsf_ctx_create.argtypes = [C.c_int, vp, vp, C.POINTER(vp)]
    lib.rsf_ctx_wait_stream.argtypes = [vp, vp]
    ub = C.POINTER(C.c_ubyte)
    lib.rsf_nccl_unique_id.argtypes = [ub]
    lib.rsf_ctx_create_group.argtypes = [C.c_int, vp, ub, C.c_int, C.c_int, C.POINTER(vp)]
    lib.rsf_ctx_group.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    lib.rsf_debug_col_slice.argtypes = [i64, C.c_int, C.c_int, C.POINTER(i64), C.POINTER(i64)]
    lib.rsf_debug_col_slice.restype = None
    lib.rsf_debug_solve_bench.argtypes = [vp, C.c_int, C.c_int, dp]
    lib.rsf_debug_solve_bench.restype = C.c_double
    lib.rsf_debug_job_runs.argtypes = [C.c_int] * 4
    lib.rsf_debug_job_group.argtypes = [C.c_int, C.POINTER(C.c_double), C.c_int, C.c_int]
    lib.rsf_ctx_destroy.argtypes = [vp]
    lib.rsf_ctx_destroy.restype = None
    lib.rsf_factor.argtypes = [vp, vp, i64, C.POINTER(rsf_kernel), i32, C.c_double, i32,
                               C.POINTER(rsf_opts), C.POINTER(vp)]
    lib.rsf_fact_destroy.argtypes = [vp]
    lib.rsf_fact_destroy.restype = None
    lib.rsf_fact_info.argtypes = [vp, C.POINTER(rsf_fact_diag)]
    lib.rsf_logdet.argtypes = [vp, dp]
    for f in ("rsf_solve", "rsf_apply", "rsf_sample"):
        getattr(lib, f).argtypes = [vp, vp, vp, i64, i64]
    lib.peel_trace.argtypes = [vp, vp, C.c_double, C.POINTER(rsf_opts), i32, dp, C.POINTER(rsf_peel_diag)]
    lib.hutch_trace.argtypes = [vp, vp, i64, C.c_uint64, dp, dp]
    lib.gp_profile_eval.argtypes = [vp, vp, vp, i64, C.POINTER(rsf_kernel), C.c_double, i32,
                                    C.POINTER(rsf_opts), dp, dp, C.POINTER(rsf_eval_diag)]
    lib.gp_cond_mean.argtypes = [vp, vp, vp, i64, vp]
    lib.gp_cond_sample.argtypes = [vp, vp, i64, vp, vp, vp, i64]
    lib.gp_mle_eval.argtypes = [vp, vp, vp, i64, C.POINTER(rsf_kernel), C.c_double, i32,
                                C.POINTER(rsf_opts), dp, dp, C.POINTER(rsf_eval_diag)]
    lib.rsf_last_error.argtypes = []
    lib.rsf_last_error.restype = C.c_char_p
    lib.rsf_kernel_launches.argtypes = []
    lib.rsf_kernel_launches.restype = C.c_int64
    lib.rsf_debug_nccl_calls.argtypes = []
    lib.rsf_debug_nccl_calls.restype = C.c_int64
    lib.rsf_profile_dump.argtypes = []
    lib.rsf_profile_dump.restype = C.c_char_p
    lib.rsf_trace_dump.argtypes = []
    lib.rsf_trace_dump.restype = C.c_char_p
    lib.rsf_debug_gemm.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                   C.c_void_p, C.c_void_p, C.c_double, C.c_void_p, C.c_int]
    lib.rsf_debug_gemm.restype = C.c_int
    lib.rsf_debug_gemm_log.argtypes = []
    lib.rsf_debug_gemm_log.restype = C.c_char_p
    lib.rsf_profile_reset.argtypes = []
    lib.rsf_profile_reset.restype = None
    lib.rsf_stats_enable.argtypes = [C.c_int]
    lib.rsf_stats_enable.restype = None
    lib.rsf_stats_get.argtypes = [C.POINTER(C.c_double)]
    lib.rsf_stats_get.restype = None
    lib.rsf_stats_reset.argtypes = []
    lib.rsf_stats_reset.restype = None
    lib.rsf_debug_gemm_bench.argtypes = [C.c_int] * 7
    lib.rsf_debug_gemm_bench.restype = C.c_double
    lib.rsf_debug_fp64_peak.argtypes = [C.c_int, C.c_int]
    lib.rsf_debug_fp64_peak.restype = C.c_double
    for f in EXPORTS:
        if f not in ("rsf_ctx_destroy", "rsf_fact_destroy", "rsf_opts_default", "rsf_last_error",
                     "rsf_kernel_launches", "rsf_profile_dump", "rsf_profile_reset", "rsf_stats_enable",
                     "rsf_stats_get", "rsf_stats_reset", "rsf_debug_gemm_bench",
                     "rsf_debug_fp64_peak", "rsf_trace_dump", "rsf_debug_gemm_log", "rsf_debug_col_slice",
                     "rsf_debug_solve_bench", "rsf_debug_nccl_calls"):
            getattr(lib, f).restype = C.c_int
    return lib

/*
 * rsf.h -- C ABI of librsf: Gaussian-process log-likelihood l(theta) and score
 * g(theta) through the recursive skeletonization factorization (RSF) of
 * Sigma(theta) and weak-admissibility matrix peeling of Tr(Sigma^-1 Sigma_i),
 * hand-written FP64 CUDA for sm_100a (B200).
 *
 * Citations: "P:n" = line n of the paper's text (arXiv:1603.08057, PAPER.md).
 *   problem statement   P:14-18 (Eq. normaldist), P:37-39 (Eq. loglikelihood),
 *                       P:43-47 (Eq. gradient)
 *   RSF                 P:201-283 (Eq. rskelf), Def. id P:205-210,
 *                       proxy trick P:299-308, operators P:381-389
 *   peeling             P:438-595 (Eq. lowrankapprox, levels, extraction)
 *   Alg. 1
 * Readings of ambiguous passages (R-*) are listed in DESIGN.md §3.
 *
 * Conventions (all functions):
 *   - every call returns rsf_status; RSF_OK == 0; no C++ exception or exit()
 *     crosses the ABI.  On error the outputs are unspecified, no handle is
 *     created, and rsf_last_error() describes the failure (level/box on a
 *     numerical failure).
 *   - points: xy is n x 2, row-major (x0,y0,x1,y1,...), FP64, every coordinate
 *     finite and inside the unit square [0,1]^2 (root box, reading R-S);
 *     device OR host memory (host buffers are staged by the library).
 *   - vectors / blocks: column-major n x nrhs with leading dimension ld >= n,
 *     in the CALLER's original point order (the library applies its Morton
 *     permutation internally); device or host memory.
 *   - the caller owns every buffer it passes; the library owns handles and
 *     their device memory until *_destroy.  Handles are immutable after
 *     creation; concurrent solve/apply calls on one handle must use the same
 *     context stream (calls are stream-ordered on it).
 *   - results are bitwise reproducible for a fixed (input, seed, build, GPU).
 *   - stream ordering: the library works on its context stream.  Device inputs must be
 *     complete before a call reads them: a caller that produced them on another stream
 *     calls rsf_ctx_wait_stream(ctx, that_stream) first (the Python binding does this with
 *     torch's current stream before every call).  Every call returns after its own device
 *     work is complete, so outputs are ready for any stream on return.
 */
#ifndef RSF_H_
#define RSF_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RSF_OK = 0,
  RSF_EINVAL = 1,    /* invalid argument (null pointer, n < 1, eps <= 0, leaf < 1, rho/sigma2/alpha <= 0,
                        nugget < 0, p out of range, point outside [0,1]^2 or non-finite, logdet of a
                        Sigma_i handle, ...) */
  RSF_ENUMERIC = 2,  /* Cholesky of a redundant block X_RR or of the top block failed (Remark P:285-287) */
  RSF_ECUDA = 3,     /* CUDA runtime error */
  RSF_ENOMEM = 4,    /* device allocation failed */
  RSF_ENCCL = 5      /* collective failure (multi-GPU) */
} rsf_status;

/* covariance families: Sigma_jk = sigma2 * k(r_jk) + nugget * [j == k] (index delta, R-H/R-I) */
typedef enum {
  RSF_RQ = 0,        /* (1 + r^2/(2 alpha rho^2))^-alpha */
  RSF_MATERN12 = 1,  /* exp(-r/rho) */
  RSF_MATERN32 = 2,  /* (1 + sqrt3 r/rho) exp(-sqrt3 r/rho) */
  RSF_MATERN52 = 3,  /* (1 + s + s^2/3) exp(-s), s = sqrt5 r/rho */
  RSF_SQEXP = 4      /* exp(-r^2/(2 rho^2)) (alpha -> inf limit; test family) */
} rsf_family;

/* theta components (order of the gradient is the order given in rsf_kernel.theta) */
typedef enum { RSF_RHO = 0, RSF_SIGMA2 = 1, RSF_NUGGET = 2, RSF_ALPHA = 3, RSF_RHO2 = 4 } rsf_param;

typedef struct {
  int32_t family;      /* rsf_family */
  double rho, sigma2, nugget, alpha;   /* current values; alpha used by RSF_RQ only */
  int32_t p;           /* number of theta components, 0 <= p <= 4 */
  int32_t theta[4];    /* rsf_param values, distinct; RSF_ALPHA only with RSF_RQ, RSF_RHO2 only if rho2 > 0 */
  double rho2;         /* 0: isotropic k(r / rho).  > 0: anisotropic scaled distance
                          q = sqrt(dx^2/rho^2 + dy^2/rho2^2) and k(q) at unit length; RSF_RHO is then
                          the x-axis length theta_1 and RSF_RHO2 the y-axis length theta_2 */
} rsf_kernel;

typedef struct {
  double eps_peel;     /* peeling tolerance (CPQR truncation of the sketches; R-N). default 1e-6 */
  int32_t oversample;  /* c of W in R^{n x (r+c)} (R-K). default 8 */
  int32_t probe_block; /* max columns per G-apply block (memory bound). default 512 */
  int32_t peel_start;  /* initial probe columns per group at level 1 (adaptive, R-M). default 64 */
  int32_t max_depth;   /* quadtree depth cap (degenerate leaves). default 30 */
  double r_near;       /* near radius / box half-width (R-C). default 1.8 */
  double r_in, r_out;  /* proxy annulus radii / half-width (R-C; 4 rings x 64 angles, n_prox=256). 1.75, 2.45 */
  uint64_t seed;       /* Philox4x32-10 key of the peeling probes (stream 3). default 1603080570 */
  int32_t strong;      /* peeling admissibility (next row f4): 0 weak (default);
                          1 strong -- interaction-list blocks, 36 probe classes per level, 9 extraction
                          classes; needs a perfect quadtree (every leaf at depth L), else RSF_EINVAL */
  int32_t peel_f32;    /* memory-saving mode.  1: store the peeled levels G^(m) (row bases V_i, cores
                          Brow_i) in FP32 -- every product still runs and accumulates in FP64 -- and run
                          gp_mle_eval's trace jobs one after the other (halves the
                          O(n s_1) peeling storage of P:615 so that config 4, n = 2^20, fits one GPU).
                          default 0 */
} rsf_opts;            /* pass NULL for all defaults; rsf_opts_default() fills the defaults */

typedef struct rsf_ctx_s* rsf_ctx;     /* device, stream, optional NCCL communicator */
typedef struct rsf_fact_s* rsf_fact;   /* an RSF of Sigma, or the apply-only compression of Sigma_i */

typedef struct {
  int32_t levels;            /* quadtree depth L */
  int32_t top_size;          /* |I_0| (dense top block) */
  int32_t level_boxes[32];   /* boxes per level 1..L (index = level) */
  int32_t level_active[32];  /* sum |I_b| per level */
  int32_t level_skel[32];    /* sum |S_b| per level */
  int32_t level_maxI[32];    /* max |I_b| per level */
  double flops_id, flops_elim, flops_top;   /* algorithmic FP64 flops */
  double factor_bytes;       /* stored factor bytes (read twice by a 1-RHS solve) */
  double seconds;            /* wall time of the factorization (device-synchronised) */
} rsf_fact_diag;

typedef struct {
  int32_t levels;
  int32_t cols[32];          /* probe columns per group at level l (index = level), after adaptivity */
  int32_t rank_max[32];      /* max eps_peel-rank of the sibling blocks at level l */
  int32_t nL;                /* extraction columns (max leaf size) */
  double cancellation;       /* sum |diag(H)| / |Tr| (P:597-599 diagnostic) */
  double applies;            /* operator columns applied (G X column count) */
  double seconds;
  int32_t rank_min[32];      /* min / median eps_peel-rank of the sibling blocks at level l */
  int32_t rank_med[32];
  double stored_bytes;       /* bytes of the peeled representation (bases V_i + cores) */
} rsf_peel_diag;

typedef struct {
  double logdet, quad;       /* log|F| and z^T F^-1 z */
  double q[4], trace[4];     /* z^T F^-1 F_i F^-1 z and Tr(F^-1 F_i) per theta component */
  double t_tree, t_factor, t_compress, t_solve, t_peel, t_total;  /* seconds */
  double flops_factor;       /* algorithmic flops of all factorizations */
  double kernel_launches;    /* CUDA kernels launched by the call */
  rsf_fact_diag fact;        /* the Sigma factor */
  rsf_peel_diag peel[4];     /* per theta component (sigma2/nugget share the F^-1 peel) */
  /* t_compress, t_solve and t_peel above are SUMS over the trace jobs, which may run concurrently
   * (and then exceed t_total); t_jobs_wall is the wall time of the job section itself */
  double t_jobs_wall;
  int32_t jobs;              /* trace jobs of the evaluation (one per general theta_i, + Tr(F^-1)) */
  int32_t concurrent;        /* 1: the jobs ran concurrently on their own streams */
  int32_t serial_fallback;   /* 1: out of memory side by side, the evaluation was redone serially */
  int32_t groups;            /* rank sub-groups the jobs were dealt to (1 on a single GPU) */
} rsf_eval_diag;

void rsf_opts_default(rsf_opts* out);

/* context on CUDA device `device`; cuda_stream may be NULL (library creates a stream).
 * nccl_comm: NULL = single GPU, else an ncclComm_t of the caller (not owned): this context is
 * one rank of a group that shares every gp_mle_eval / peel_trace call (DESIGN.md §7 -- the
 * peeling probe columns of each block are split across the ranks, and exchanged
 * with one NCCL all-gather per block; every rank passes the same inputs and receives the
 * same results).  Returns RSF_ENCCL when NCCL cannot be loaded or queried. */
rsf_status rsf_ctx_create(int device, void* cuda_stream, void* nccl_comm, rsf_ctx* out);
/* NCCL bootstrap of a rank group without a caller communicator (one process per GPU):
 * rank 0 calls rsf_nccl_unique_id (out: 128 bytes, host), the caller distributes the bytes
 * (e.g. torch.distributed broadcast), then every rank calls rsf_ctx_create_group with its
 * rank in [0, world).  The context owns the communicator.  world = 1 needs no id traffic
 * (any 128 bytes).  RSF_EINVAL on bad ranks, RSF_ENCCL on NCCL failures. */
rsf_status rsf_nccl_unique_id(unsigned char* out);
rsf_status rsf_ctx_create_group(int device, void* cuda_stream, const unsigned char* id, int rank, int world,
                                rsf_ctx* out);
/* rank and group size of a context (0 and 1 for a single-GPU context) */
rsf_status rsf_ctx_group(rsf_ctx ctx, int* rank, int* world);
/* column slice [lo, hi) that part `part` of `parts` owns when k probe columns are split
 * (contiguous; sizes differ by at most one, larger first).  Host only (tests). */
void rsf_debug_col_slice(int64_t k, int parts, int part, int64_t* lo, int64_t* hi);
/* 1 if rank `rank` of a `world`-rank group runs trace job `job` of an evaluation with `njobs` jobs
 * (jobs dealt to min(njobs, world) rank groups), 0 if not, -1 on bad arguments.
 * Host only (tests). */
int rsf_debug_job_runs(int njobs, int world, int rank, int job);
/* group (0..ngroups-1) of rank `rank` of a `world`-rank group when the ngroups trace-job groups carry
 * the estimated work gw[0..ngroups-1] (gp_mle_eval: 3 per general theta_i job, 1 for the Tr(F^-1)
 * job): ranks 0..ngroups-1 seed one group each, every further rank joins the group
 * with the largest current work per rank; equal weights give rank r -> group r mod ngroups.
 * -1 on bad arguments.  Host only (tests). */
int rsf_debug_job_group(int ngroups, const double* gw, int world, int rank);
/* Number of NCCL collectives (all-gathers of probe-block slices, job results, memory agreements,
 * trace partial sums) this process has issued so far.  A single-GPU context issues none; with
 * RSF_NCCL_FORCE=1 in the environment a world = 1 group made by rsf_ctx_create_group keeps its
 * one-rank NCCL communicator and routes every collective of the sharded path through it (the
 * transport test on one GPU; results are unchanged).  Host only (tests). */
int64_t rsf_debug_nccl_calls(void);
void rsf_ctx_destroy(rsf_ctx ctx);
/* Order the context after the caller: everything enqueued on `stream` so far (an event recorded
 * there) completes before the context stream runs further work.  stream = NULL is the legacy
 * default stream.  Returns RSF_EINVAL for a NULL ctx, RSF_ECUDA on a runtime error. */
rsf_status rsf_ctx_wait_stream(rsf_ctx ctx, void* stream);

/* Build F ~ Sigma (which = -1) with ID tolerance eps (Def. id: |R'_jj| <= eps |R'_11| truncation,
 * reading R-A), leaf capacity `leaf` (n_occ), or (which = i in [0,p)) the apply-only
 * compression of Sigma_i = dSigma/dtheta_i (reading R-F).  xy: n x 2 (see conventions). */
rsf_status rsf_factor(rsf_ctx ctx, const double* xy, int64_t n, const rsf_kernel* kernel, int32_t which,
                      double eps, int32_t leaf, const rsf_opts* opts, rsf_fact* out);
void rsf_fact_destroy(rsf_fact f);
rsf_status rsf_fact_info(rsf_fact f, rsf_fact_diag* out);

/* log|F| = 2 log|C| plus the redundant-block terms; Sigma handles only. out: host. */
rsf_status rsf_logdet(rsf_fact f, double* out);
/* x = F^-1 b; b and x may alias; Sigma handles only */
rsf_status rsf_solve(rsf_fact f, const double* b, double* x, int64_t nrhs, int64_t ld);
/* y = F x; for a Sigma_i handle, y = F_i x */
rsf_status rsf_apply(rsf_fact f, const double* x, double* y, int64_t nrhs, int64_t ld);
/* z = F^{1/2} w with F^{1/2} (F^{1/2})^T = F; Sigma handles only */
rsf_status rsf_sample(rsf_fact f, const double* w, double* z, int64_t nrhs, int64_t ld);

/* Tr(F^-1 F_i) by peeling G = 1/2 (F^-1 F_i + F_i F^-1) (R-Z); Fi == NULL peels G = F^-1.
 * trace_id selects the probe counter stream. trace: host. diag nullable. */
rsf_status peel_trace(rsf_fact F, rsf_fact Fi, double eps_peel, const rsf_opts* opts, int32_t trace_id,
                      double* trace, rsf_peel_diag* diag);

/* Hutchinson estimate (Eq. hutch; the baseline the paper compares peeling with):
 * trace = (1/q) sum_p u_p^T F^-1 F_i u_p over q = nprobe Rademacher probes (Philox4x32-10, key (seed, 4),
 * counter (original point index, probe, 0, 0), sign from bit 0), std_err = sample standard deviation / sqrt(q).
 * Fi == NULL estimates Tr(F^-1).  One solve and one apply per probe.  trace, std_err: host. */
rsf_status hutch_trace(rsf_fact F, rsf_fact Fi, int64_t nprobe, uint64_t seed, double* trace, double* std_err);

/* Alg. 1: l-hat and g-hat at theta = kernel values.  On a rank group (rsf_ctx_create
 * with a communicator, rsf_ctx_create_group) every rank calls it with the same arguments; the
 * factorizations are replicated (deterministic), the peeling columns are split, and every rank
 * returns the same l and g.  eps is the ID tolerance of every
 * factorization (eps_fact), opts->eps_peel the peeling tolerance.  ell: host scalar; grad: host
 * array of p doubles.  xy, z device or host.  diag nullable.  The independent trace jobs (one per
 * theta component) run concurrently on streams the context creates on first use and
 * releases in rsf_ctx_destroy; the call returns after all of them (and the context stream) are
 * complete.  Results equal the serial order (RSF_PAR_TRACES=0).  diag times are summed over jobs. */
rsf_status gp_mle_eval(rsf_ctx ctx, const double* xy, const double* z, int64_t n, const rsf_kernel* kernel,
                       double eps, int32_t leaf, const rsf_opts* opts, double* ell, double* grad,
                       rsf_eval_diag* diag);

/* Log profile likelihood (next row f3; Eq. prof and its gradient): z ~ N(mu 1, s2 Sigma(theta))
 * with mu and s2 profiled out,
 *   l~ = -1/2 log|Sigma| - n/2 log Q + n/2 (log n - 1 - log 2pi),  Q = z^T (Sigma + 1 1^T)^-1 z,
 *   g~_i = -1/2 Tr(Sigma^-1 Sigma_i) + n/2 v^T Sigma_i v / Q,        v = (Sigma + 1 1^T)^-1 z
 * (Sherman-Morrison through F^-1 z and F^-1 1; reading R-Prof: the printed constant's "2 pi" is log 2 pi).
 * Arguments as gp_mle_eval; theta may not contain RSF_SIGMA2 (profiled out); n >= 2.  diag->quad = Q. */
rsf_status gp_profile_eval(rsf_ctx ctx, const double* xy, const double* z, int64_t n, const rsf_kernel* kernel,
                           double eps, int32_t leaf, const rsf_opts* opts, double* ell, double* grad,
                           rsf_eval_diag* diag);

/* Conditional (kriging) mean at m new locations (Remark conditional):
 * out = Sigma_12 F^-1 z with (Sigma_12)_aj = sigma2 k(x'_a, x_j) (no nugget between distinct observations).
 * F: Sigma factor of the n data locations; z: n values in original order; xy_new: m x 2 row-major;
 * out: m.  Device or host buffers.  Direct O(m n) cross product (FP64). */
rsf_status gp_cond_mean(rsf_fact F, const double* z, const double* xy_new, int64_t m, double* out);

/* Conditional sampling (Remark conditional): with F ~ Sigma of the joint covariance of
 * [x_new; x_data] (the m new points FIRST, then the n2 data points, as passed to rsf_factor) and
 * F22 ~ Sigma_22 of the data points alone,
 *   out = Sigma_12 F22^-1 z + [I, -Sigma_12 F22^-1] F^{1/2} w
 *       = y_1 + Sigma_12 F22^-1 (z - y_2),   y = F^{1/2} w,
 * Sigma_12 applied as the first m rows of F [0; v] (the paper's "appropriate padding").  For w ~ N(0, I)
 * out ~ N(Sigma_12 Sigma_22^-1 z, Sigma_11 - Sigma_12 Sigma_22^-1 Sigma_12^T) up to the factorizations'
 * accuracy.  z: n2 data values; w: (m + n2) x nrhs (ld m + n2), joint order; out: m x nrhs (ld m);
 * device or host.  F must be a full factor from rsf_factor.  RSF_EINVAL on shape mismatch. */
rsf_status gp_cond_sample(rsf_fact F, rsf_fact F22, int64_t m, const double* z, const double* w, double* out,
                          int64_t nrhs);

/* message of the last failing call on this thread ("" if none) */
const char* rsf_last_error(void);
/* number of CUDA kernels launched by this thread so far (diagnostics) */
int64_t rsf_kernel_launches(void);
/* phase timings "name=seconds;..." collected when RSF_PROFILE=1 (stream-synchronising; diagnostics only) */
const char* rsf_profile_dump(void);
void rsf_profile_reset(void);
/* launch trace "phase|file:line=seconds,launches;..." collected when RSF_KTRACE=1: an event after every
 * launch on the evaluation stream, the time between consecutive events attributed to the launch site
 * (diagnostics only; resets with rsf_profile_reset) */
const char* rsf_trace_dump(void);
/* batched-GEMM log "phase|file:line|TATB=seconds,flops,launches,ctas_min,ctas_max,kmin,kmax;..." collected
 * when RSF_GEMMLOG=1: events around every batched GEMM, aggregated by phase and call site
 * (diagnostics only; resets with rsf_profile_reset) */
const char* rsf_debug_gemm_log(void);
/* batched-GEMM statistics for the roofline: CUDA events around every launch on its stream.
 * rsf_stats_get fills {launches, busy seconds (length of the union of the launch intervals, so that
 * launches overlapping on concurrent streams are not double-counted), algorithmic flops,
 * compulsory bytes}. */
void rsf_stats_enable(int on);
/* diagnostics: TFLOP/s of the batched FP64 GEMM on batch x (M x N x K), transposes ta/tb */
double rsf_debug_gemm_bench(int M, int N, int K, int batch, int ta, int tb, int reps);
/* diagnostics / tests: C_i = alpha op(A_i) op(B_i) + beta C_i for `batch` problems stored back to back
 * (device pointers, column-major, leading dimensions = rows of the stored matrix) through the batched
 * pipelined FP64 GEMM; splitk > 0 forces that many K slices (1 = none), 0 = the cost model decides.
 * Synchronous; returns RSF_OK, RSF_EINVAL or RSF_ECUDA. */
int rsf_debug_gemm(int ta, int tb, int M, int N, int K, int batch, double alpha, const double* A,
                   const double* B, double beta, double* C, int splitk);
void rsf_stats_get(double* out4);
/* diagnostics: seconds per F^-1 X on nrhs columns of the Sigma factor f, device time
 * (CUDA events on the context stream, mean of reps after one warm-up; no layout permutation);
 * *bytes (nullable) = algorithmic bytes of one 1-RHS solve.  -1 on error. */
double rsf_debug_solve_bench(rsf_fact f, int nrhs, int reps, double* bytes);
/* diagnostics: FP64 peak (TFLOP/s) of independent DMMA.8x8x4 (dmma=1) or DFMA (dmma=0) chains on the
 * current device, best of `reps` timed launches -- the live roofline denominator of bench.py */
double rsf_debug_fp64_peak(int dmma, int reps);
void rsf_stats_reset(void);

#ifdef __cplusplus
}
#endif
#endif /* RSF_H_ */

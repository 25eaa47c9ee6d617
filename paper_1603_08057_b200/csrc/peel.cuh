// Weak-admissibility matrix peeling (PAPER §3.2) and Alg. 1.
#pragma once
#include "../../include/rsf.h"
#include "rsf_impl.cuh"

namespace rsf {

struct PeelDiag {
  std::vector<int> cols, rank_max;   // per level (index = level)
  std::vector<int> rank_min, rank_med;   // per level: min / median eps_peel-rank over the sibling blocks
  double stored_bytes = 0;           // bytes of the peeled representation (bases V_i + cores Brow_i)
  int nL = 0;
  double cancellation = 0;
  double applies = 0;
  double seconds = 0;
  double flops = 0;
};

// Tr(G) with G = 1/2 (F^-1 Fi + Fi F^-1) (Fi != null) or G = F^-1 (Fi == null).  comm: the rank
// group sharing the probe columns (null: the factor context's group)
double peel(const Fact& F, const Fact* Fi, const Opts& o, int trace_id, PeelDiag* diag,
            const Comm* comm = nullptr);
void fill_peel_diag(const PeelDiag& d, rsf_peel_diag* out);

// Hutchinson estimate of Tr(F^-1 F_i) or Tr(F^-1): mean and standard error over q probes
void hutch(const Fact& F, const Fact* Fi, long long q, unsigned long long seed, double* mean, double* se);

struct EvalResult {
  double ell = 0, logdet = 0, quad = 0;
  double grad[4] = {0, 0, 0, 0}, q[4] = {0, 0, 0, 0}, trace[4] = {0, 0, 0, 0};
  double t_tree = 0, t_factor = 0, t_compress = 0, t_solve = 0, t_peel = 0, t_total = 0;
  double flops_factor = 0;
  long long launches = 0;
  FactDiag fdiag;
  int L = 0, n0 = 0;
  PeelDiag pd[4];
  double t_jobs_wall = 0;            // wall time from the start of the trace jobs to the last one's end
  int jobs = 0, concurrent = 0, serial_fallback = 0, groups = 1;
};

// profile = true: the log profile likelihood of Eq. prof and its gradient; quad holds
// Q = z^T (Sigma + 1 1^T)^-1 z, q_i = v^T Sigma_i v with v = (Sigma + 1 1^T)^-1 z
EvalResult mle_eval(Ctx& ctx, const double* xy, const double* z, int n, const KParams& kp, int p,
                    const int* theta, double eps, int leaf, const Opts& o, bool profile = false);
// conditional mean Sigma_12 F^-1 z at m new points (xyn, m x 2 device; out device)
void cond_mean(const Fact& F, const double* z, const double* xyn, long long m, double* out);
void fill_eval_diag(const EvalResult& r, rsf_eval_diag* out);

// deterministic dot product of two device vectors (n doubles)
double ddot(cudaStream_t s, const double* a, const double* b, long long n);

// Philox4x32-10 N(0,1) probe entries: X'(j, t) = qmap[t] == g ?
// normal(perm[t], col0 + j, level, trace) : 0, X' is k x n (ld k)
void gen_probes(cudaStream_t s, double* X, int k, int n, const int* perm, const int* qmap, int g,
                int col0, int level, int trace, unsigned long long seed);

}  // namespace rsf

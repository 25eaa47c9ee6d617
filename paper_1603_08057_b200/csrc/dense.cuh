// Batched dense FP64 factorizations used by the RSF and the peeling:
//   * blocked Householder QR (panel kernel + compact-WY trailing update on the
//     batched GEMM), optionally keeping (V, T) to apply Q later;
//   * column-pivoted QR of the triangular factor with rank truncation and the
//     interpolation matrix T = R11^-1 R12 (the ID of Def. id);
//   * blocked Cholesky with the explicit inverse of the factor.
#pragma once
#include "common.cuh"
#include "gemm.cuh"

namespace rsf {

constexpr int QR_NB = 32;    // Householder panel width
constexpr int CH_NB = 64;    // Cholesky / inverse block

struct QRProb {
  double* A;       // m x c, column-major, overwritten by R (upper) and V (below diagonal)
  long long lda;
  int m, c;
  double* Tws;     // if keep_q: ceil(min(m,c)/QR_NB) blocks of QR_NB x QR_NB (the WY T factors)
  double* tau;     // if keep_q: min(m,c) reflector scalars
};

// Householder QR of every problem (R in the upper triangle).  Workspace is
// allocated internally.  If keep_q, the per-panel T factors go to Tws.
void geqrf_batched(cudaStream_t s, const std::vector<QRProb>& probs, bool keep_q);

// Q^T C (trans=true) or Q C (trans=false) for Q from geqrf_batched(keep_q),
// C is m x nc with leading dimension ldc (per problem).
struct QApplyProb {
  const double* A; long long lda; int m, c; const double* Tws;
  double* C; long long ldc; int nc;
};
void ormqr_batched(cudaStream_t s, const std::vector<QApplyProb>& probs, bool trans);

struct CPQRProb {
  const double* R;   // q x c upper-triangular (rows 0..q-1 of an lda=ldr matrix); read only
  long long ldr;
  int q, c;
  double* W;         // workspace q x c (global fallback; may be null when it fits in smem)
  double* T;         // output, T(0:k, 0:c-k) with leading dimension c
  int* piv;          // output, c pivot positions (skeleton = piv[0:k])
  double* Rout;      // optional: q x c pivoted R' (ld = q) incl. Householder vectors below the diagonal
  double* tau;       // optional: reflector scalars (needed with Rout to form Q_R)
};
// k[i] (device array, one per problem) receives the rank.
void cpqr_id_batched(cudaStream_t s, const std::vector<CPQRProb>& probs, double eps, int* d_k,
                     bool want_T = true);

struct PotrfProb {
  double* A;   // n x n lower Cholesky in place (upper triangle zeroed)
  long long lda;
  int n;
  double* Linv;  // optional n x n (ld = ldi): explicit L^-1 (lower)
  long long ldi;
};
// d_logsum[i] = sum_j log L_jj; d_info[i] = 0 or (1 + first failing column).
void potrf_batched(cudaStream_t s, const std::vector<PotrfProb>& probs, double* d_logsum, int* d_info);

// One Householder panel step: factor the panel A(j0:m, j0:j0+ncol) (A points at
// A(j0, j0)), then apply Q^T of the panel to the c2 trailing columns (compact WY
// on the batched GEMM).  V (rows x ncol), T (QR_NB^2), W/W2 (QR_NB x c2) are
// caller workspaces; T is kept if the caller needs Q later.
struct PanelStep {
  double* A; long long lda;
  int rows, ncol, c2;
  double* V; double* T; double* W; double* W2;
};
void panel_step_batched(cudaStream_t s, const std::vector<PanelStep>& v);

struct CopyProb {
  const double* src; long long lds;
  double* dst; long long ldd;
  int rows, cols;
  double alpha;       // dst = alpha * src
};
void copy_batched(cudaStream_t s, const std::vector<CopyProb>& probs);

}  // namespace rsf

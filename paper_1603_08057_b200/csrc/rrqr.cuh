// Blocked rank-revealing QR with randomized block pivoting (HQRRP-style),
// truncated at the eps-rank, for large boxes and for the peeling sketches.
//
// The paper computes IDs "based on a rank-revealing QR factorization"
// and orth() by column-pivoted QR.  Greedy CPQR is BLAS2; here the
// pivots of each block of QR_NB columns are chosen by greedy CPQR of a small
// Gaussian sketch Y = G A ((QR_NB+8) rows), the block is factored with the
// Householder panel kernel and the trailing matrix updated with the batched
// GEMM (compact WY), and the sketch is downdated as Y2 -= Y1 R11^-1 R12.
// Truncation is exact: k is the smallest column count whose trailing columns
// all have norm <= eps * max_j ||A(:,j)|| (the quantity greedy CPQR tests).
#pragma once
#include "dense.cuh"

namespace rsf {

struct RRQRProb {
  double* A;        // m x c (lda), overwritten: R (upper, first kdone columns), V below the diagonal
  long long lda;
  int m, c;
  int* piv;         // out: c column positions (skeleton = piv[0:k])
  double* Tws;      // optional: WY T factors, one QR_NB^2 block per panel (for ormqr / U formation)
  double* T;        // optional: out T = R11^-1 R12, k x (c-k), leading dimension ldt
  long long ldt;
  const double* ref_in = nullptr;  // optional (device scalar): absolute reference norm; the
                                   // truncation becomes ||trailing col|| <= eps * (*ref_in)
  double* ref_out = nullptr;       // optional (device scalar): max_j ||A(:, j)|| of the input
};

struct RRQRResult {
  std::vector<int> k;       // eps-rank per problem
  std::vector<int> done;    // columns factored (multiple of QR_NB, >= k) -> panels for ormqr
};

RRQRResult rrqr_batched(cudaStream_t s, const std::vector<RRQRProb>& probs, double eps,
                        unsigned long long seed);

// X = U^-1 B for upper-triangular U (k x k, ld ldu), B (k x nrhs, ld ldb) in place
struct TrsmProb { const double* U; long long ldu; double* B; long long ldb; int k, nrhs; };
void trsm_upper_batched(cudaStream_t s, const std::vector<TrsmProb>& probs);

}  // namespace rsf

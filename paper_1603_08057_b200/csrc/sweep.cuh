// Fused per-box level sweeps of the RSF operators for small boxes.
//
// The solve F^-1 b and the apply-only F_i x
// visit every box of a level with three dense steps on the box's skeleton (S)
// and redundant (R) columns of the right-hand-side block X' (k x n, tree order):
//   solve, forward   x_R -= T^T x_S;  x_R <- L^-1 x_R;  x_S -= E x_R
//   solve, backward  x_R -= E^T x_S;  x_R <- L^-T x_R;  x_S -= T x_R
//   apply-only, up   x_S += T x_R;    y_R  = X_SR^T x_S + X_RR x_R
//   apply-only, down y_S += X_SR x_R; y_R += T^T y_S
// For boxes with |I_b| <= 256 one CTA per (box, slab of KC right-hand sides)
// holds the slab's S and R columns in shared memory and runs all steps of the
// level in one pass: one read and one write of the box's columns instead of
// four batched-GEMM launches with intermediate round trips through HBM.
#pragma once
#include "common.cuh"

namespace rsf {

struct BoxOp {
  const int* S; const int* R;   // tree indices of the skeleton / redundant DOFs (device)
  int kb, r;                    // |S_b|, |R_b|
  const double* T;              // kb x r (ld kb): interpolation matrix
  const double* L;              // r x r (ld r): L^-1 (Sigma) or X_RR (Sigma_i)
  const double* E;              // kb x r (ld kb): E (Sigma) or X_SR (Sigma_i)
};

enum SweepKind { SW_SOLVE_FWD = 0, SW_SOLVE_BWD = 1, SW_AO_UP = 2, SW_AO_DN = 3 };

constexpr int SWEEP_MAX_I = 128;       // largest |I_b| of the FMA fused kernel (measured: slower than the GEMM path above)
constexpr int SWEEP_MAX_I_MMA = 256;   // ... of the DMMA fused kernel
constexpr int SWEEP1_MAX_I = 512;      // largest |I_b| of the one-right-hand-side fused kernel (k = 1)
// largest |I_b| the fused sweeps take with the current settings (RSF_SWEEP_MMA=1: DMMA kernel)
int sweep_max_i();

// X0: the operand updated in place (solve: X'; apply-only: x'), X1: apply-only output y'.
// ldx = k (number of right-hand sides, X' is k x n column-major).
void sweep_level(cudaStream_t s, const BoxOp* d_ops, int nops, int max_i, SweepKind kind, double* X0,
                 double* X1, int k);

}  // namespace rsf

// Element kernels of the factorization: on-the-fly kernel-entry assembly
// (ID matrices with near-field + proxy rows, self blocks, parent blocks),
// permutations and column copies.
#pragma once
#include "rsf_impl.cuh"

namespace rsf {

// A_b = [K(N_b, I_b); K(Gamma_b, I_b)] (Eq. proxyid) column-major, lda = m
struct IdAsmDesc {
  double* A;
  int m_near, c;
  const int* near;   // tree indices of N_b
  const int* I;      // tree indices of I_b
  double cx, cy, h;
};
void assemble_id(cudaStream_t s, const std::vector<IdAsmDesc>& d, const KParams& kp, int which,
                 const Opts& o, const double* xs, const double* ys, int nprox_rings, int nprox_angles);

// self block B_b (c x c, ld c): child diagonal blocks copied from the children's
// (modified) B_SS, everything else original kernel entries
struct SelfAsmDesc {
  double* B;
  int c;
  const int* I;
  int nch;
  int choff[5];
  const double* chB[4];
  int chld[4];
};
void assemble_self(cudaStream_t s, const std::vector<SelfAsmDesc>& d, const KParams& kp, int which,
                   const double* xs, const double* ys);

// Bp = B(piv, piv)
struct PermDesc { const double* B; double* Bp; int c; const int* piv; };
void permute_sym(cudaStream_t s, const std::vector<PermDesc>& d);

// X = (X + X^T)/2 on an n x n block
struct SymDesc { double* A; long long lda; int n; };
void symmetrize(cudaStream_t s, const std::vector<SymDesc>& d);

}  // namespace rsf

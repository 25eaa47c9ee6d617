// Variable-size batched FP64 GEMM with column gather/scatter maps.
//
//   C_b[:, mapC] = alpha * op(A_b)[:, :] * op(B_b) + beta * C_b[:, mapC]
//
// All matrices column-major.  A "map" replaces the stored-column index j by
// map[j] (gather for A/B, scatter for C); the multi-RHS sweeps of the RSF use
// it to read/write the per-box DOF columns of X' (k x n, the transpose of the
// n x k right-hand-side block) without packing.  Operands may be absolute
// pointers (factor storage) or offsets into two per-call base pointers X0/X1
// with leading dimension ldx, so descriptor arrays are built once per factor
// and reused by every solve/apply.
#pragma once
#include "common.cuh"

namespace rsf {

struct GemmDesc {
  int M, N, K;                 // M < 0: use the per-call M (number of RHS)
  int selA, selB, selC;        // 0: absolute pointer (+off elements), 1: X0, 2: X1 (+off columns, ld = ldx)
  const double* A; long long offA; int lda; const int* mapA;
  const double* B; long long offB; int ldb; const int* mapB;
  double* C; long long offC; int ldc; const int* mapC;
  double alpha, beta;
  int lower;                   // 1: only tiles touching the lower triangle of C (SYRK-style)
  const int* mapK;             // optional K-index gather applied to both operands (sparse right-hand sides)
  int btri;                    // op(B) triangular (TRMM-style K range): 1 lower (op(B)(l,j) = 0 for l < j),
                               // 2 upper (op(B)(l,j) = 0 for l > j); 0 general
  int bf32;                    // B (absolute pointer, selB = 0) holds FP32 values: (const float*)B, ldb in floats
};

inline GemmDesc gdesc(int M, int N, int K) {
  GemmDesc d{};
  d.M = M; d.N = N; d.K = K;
  d.alpha = 1.0; d.beta = 0.0;
  return d;
}

// Per-launch GEMM log (diagnostics, RSF_GEMMLOG=1): events around every batched launch,
// aggregated by (phase, call site, transposes); dump() lists the sites by time with their
// achieved FP64 rate, CTA count and K range.
struct GemmLog {
  static bool on();
  static void push(cudaEvent_t e0, cudaEvent_t e1, const char* file, int line, bool ta, bool tb, double flops,
                   long long ctas, int maxK, int maxM);
  static std::string dump();
  static void reset();
};

// test hook: > 0 forces that many K slices in the next batched launches of this thread
// (1 = no split-K), 0 = the cost model decides
int& gemm_force_splitk();

class GemmBatch {
 public:
  GemmBatch() = default;
  GemmBatch(bool ta, bool tb) : ta_(ta), tb_(tb) {}
  void reset(bool ta, bool tb) { ta_ = ta; tb_ = tb; h_.clear(); ready_ = false; }
  void add(const GemmDesc& d) { h_.push_back(d); ready_ = false; }
  // finalize(): descriptors in a persistent device buffer (batches run many times); a batch
  // that is run without finalize() uploads its descriptors through the transient ring
  size_t size() const { return h_.size(); }
  bool empty() const { return h_.empty(); }
  void finalize(cudaStream_t s) const;
  // Launch; X0/X1/ldx/Mglob resolve the per-call operands.
  // (file/line: the call site, for the RSF_GEMMLOG diagnostics)
  void run(cudaStream_t s, double* X0 = nullptr, double* X1 = nullptr, int ldx = 0, int Mglob = 0,
           const char* file = __builtin_FILE(), int line = __builtin_LINE()) const;
  // flops of one run (2*M*N*K summed), for diagnostics
  double flops(int Mglob = 0) const;

 private:
  bool ta_ = false, tb_ = false;
  mutable bool ready_ = false;
  std::vector<GemmDesc> h_;
  mutable DBuf<GemmDesc> d_;
  mutable DBuf<int> prefix_;
  mutable std::vector<int> pre_;
  mutable const GemmDesc* dp_ = nullptr;
  mutable const int* pp_ = nullptr;
  void finalize_meta() const;
  mutable int totalN_ = 0, totalN32_ = 0, totalN128_ = 0, maxM_ = 0, maxN_ = 0, maxK_ = 0;
  mutable bool has_lower_ = false, has_mapk_ = false, has_bf_ = false;
  mutable bool glob_ = false;
};

// one-shot helper: single problem
void gemm1(cudaStream_t s, bool ta, bool tb, int M, int N, int K, double alpha, const double* A,
           int lda, const double* B, int ldb, double beta, double* C, int ldc);

}  // namespace rsf

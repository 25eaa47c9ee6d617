// Variable-size batched FP64 GEMM (see gemm.cuh).  Register-tiled DFMA:
// 256 threads, CTA tile BM x 64, BK = 16, each thread TM x 4 outputs with an
// interleaved (bank-conflict-free) column pattern; global->register prefetch
// of the next K-slab overlaps the FMA loop.
#include <ctime>
#include <cstdlib>

#include "gemm.cuh"

namespace rsf {

thread_local long long g_launches = 0;

namespace {
std::vector<std::pair<std::string, double>>& prof_table() {
  static std::vector<std::pair<std::string, double>> t;
  return t;
}
double wall() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}
}  // namespace

bool KStats::on = false;
namespace {
struct KRec { cudaEvent_t a, b; double flops, bytes; };
std::vector<KRec>& krecs() { static std::vector<KRec> v; return v; }
std::vector<cudaEvent_t>& kpool() { static std::vector<cudaEvent_t> v; return v; }
double k_launch = 0, k_sec = 0, k_flops = 0, k_bytes = 0;
cudaEvent_t get_ev() {
  auto& p = kpool();
  if (!p.empty()) { cudaEvent_t e = p.back(); p.pop_back(); return e; }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
void drain() {
  for (auto& r : krecs()) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    k_launch += 1; k_sec += ms * 1e-3; k_flops += r.flops; k_bytes += r.bytes;
    kpool().push_back(r.a);
    kpool().push_back(r.b);
  }
  krecs().clear();
}
}  // namespace
void KStats::record(cudaStream_t s, cudaEvent_t* e0, cudaEvent_t* e1) {
  if (e0) { *e0 = get_ev(); cudaEventRecord(*e0, s); }
  if (e1) { *e1 = get_ev(); cudaEventRecord(*e1, s); }
}
void KStats::push(cudaEvent_t e0, cudaEvent_t e1, double flops, double bytes) {
  krecs().push_back(KRec{e0, e1, flops, bytes});
  if (krecs().size() > 4096) drain();
}
void KStats::collect(double out[4]) {
  drain();
  out[0] = k_launch; out[1] = k_sec; out[2] = k_flops; out[3] = k_bytes;
}
void KStats::reset() { drain(); k_launch = k_sec = k_flops = k_bytes = 0; }

bool Prof::enabled() {
  static int e = -1;
  if (e < 0) { const char* v = getenv("RSF_PROFILE"); e = (v && v[0] == '1') ? 1 : 0; }
  return e == 1;
}
void Prof::add(const char* name, double sec) {
  for (auto& p : prof_table())
    if (p.first == name) { p.second += sec; return; }
  prof_table().emplace_back(name, sec);
}
std::string Prof::dump() {
  std::string r;
  for (auto& p : prof_table()) r += p.first + "=" + std::to_string(p.second) + ";";
  return r;
}
void Prof::reset() { prof_table().clear(); }
PhaseTimer::PhaseTimer(const char* n, cudaStream_t st) : name(n), s(st), on(Prof::enabled()) {
  if (on) { cudaStreamSynchronize(s); t0 = wall(); }
}
PhaseTimer::~PhaseTimer() {
  if (on) { cudaStreamSynchronize(s); Prof::add(name, wall() - t0); }
}

namespace {

constexpr int BN = 64;
constexpr int BK = 16;
constexpr int NT = 256;

__device__ __forceinline__ int find_prob(const int* __restrict__ prefix, int nprob, int x) {
  int lo = 0, hi = nprob - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (__ldg(prefix + mid) <= x) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <int BM, int TM, bool TA, bool TB>
__global__ void __launch_bounds__(NT) gemm_vb_kernel(const GemmDesc* __restrict__ descs,
                                                     const int* __restrict__ prefix, int nprob,
                                                     double* X0, double* X1, int ldx, int Mglob) {
  static_assert(BM / TM * (BN / 4) == NT, "thread layout");
  __shared__ __align__(16) double As[BK][BM];
  __shared__ __align__(16) double Bs[BK][BN];

  const int p = find_prob(prefix, nprob, blockIdx.x);
  const GemmDesc& dd = descs[p];
  const int M = dd.M < 0 ? Mglob : dd.M;
  const int N = dd.N, K = dd.K;
  const int m0 = blockIdx.y * BM;
  if (m0 >= M) return;
  const int n0 = (blockIdx.x - __ldg(prefix + p)) * BN;
  if (dd.lower && n0 >= m0 + BM) return;

  // per-call operands: offsets count columns of X0/X1 (ld = ldx)
  const double* A = dd.selA == 0 ? dd.A + dd.offA : (dd.selA == 1 ? X0 : X1) + dd.offA * (long long)ldx;
  const double* B = dd.selB == 0 ? dd.B + dd.offB : (dd.selB == 1 ? X0 : X1) + dd.offB * (long long)ldx;
  double* C = dd.selC == 0 ? dd.C + dd.offC : (dd.selC == 1 ? X0 : X1) + dd.offC * (long long)ldx;
  const long long lda = dd.selA ? ldx : dd.lda;
  const long long ldb = dd.selB ? ldx : dd.ldb;
  const long long ldc = dd.selC ? ldx : dd.ldc;
  const int* mapA = dd.mapA;
  const int* mapB = dd.mapB;
  const int* mapC = dd.mapC;
  const double alpha = dd.alpha, beta = dd.beta;

  const int tid = threadIdx.x;
  const int tx = tid & 15;   // 16 column groups
  const int ty = tid >> 4;   // BM/TM row groups

  constexpr int AE = BM * BK / NT;   // A elements per thread
  constexpr int BE = BK * BN / NT;   // B elements per thread (4)
  double ra[AE], rb[BE];

  auto load = [&](int k0) {
#pragma unroll
    for (int r = 0; r < AE; ++r) {
      int e = tid + r * NT;
      int i, l;
      if (!TA) { i = e % BM; l = e / BM; } else { l = e % BK; i = e / BK; }
      int gi = m0 + i, gl = k0 + l;
      double v = 0.0;
      if (gi < M && gl < K) {
        if (!TA) {
          long long c = mapA ? __ldg(mapA + gl) : gl;
          v = A[c * lda + gi];
        } else {
          long long c = mapA ? __ldg(mapA + gi) : gi;
          v = A[c * lda + gl];
        }
      }
      ra[r] = v;
    }
#pragma unroll
    for (int r = 0; r < BE; ++r) {
      int e = tid + r * NT;
      int l, j;
      if (!TB) { l = e % BK; j = e / BK; } else { j = e % BN; l = e / BN; }
      int gl = k0 + l, gj = n0 + j;
      double v = 0.0;
      if (gl < K && gj < N) {
        if (!TB) {
          long long c = mapB ? __ldg(mapB + gj) : gj;
          v = B[c * ldb + gl];
        } else {
          long long c = mapB ? __ldg(mapB + gl) : gl;
          v = B[c * ldb + gj];
        }
      }
      rb[r] = v;
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int r = 0; r < AE; ++r) {
      int e = tid + r * NT;
      int i, l;
      if (!TA) { i = e % BM; l = e / BM; } else { l = e % BK; i = e / BK; }
      As[l][i] = ra[r];
    }
#pragma unroll
    for (int r = 0; r < BE; ++r) {
      int e = tid + r * NT;
      int l, j;
      if (!TB) { l = e % BK; j = e / BK; } else { j = e % BN; l = e / BN; }
      Bs[l][j] = rb[r];
    }
  };

  // thread output coordinates (interleaved)
  int rows[TM];
#pragma unroll
  for (int u = 0; u < TM; ++u) {
    if (TM == 1) rows[u] = ty;
    else rows[u] = (u >> 1) * (2 * BM / TM) + ty * 2 + (u & 1);
  }
  const int c0 = tx * 2, c1 = 32 + tx * 2;

  double acc[TM][4];
#pragma unroll
  for (int u = 0; u < TM; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;

  if (K > 0) load(0);
  for (int k0 = 0; k0 < K; k0 += BK) {
    store();
    __syncthreads();
    if (k0 + BK < K) load(k0 + BK);
#pragma unroll
    for (int l = 0; l < BK; ++l) {
      double a[TM];
      if (TM == 1) {
        a[0] = As[l][rows[0]];
      } else {
#pragma unroll
        for (int u = 0; u < TM; u += 2) {
          double2 t = *reinterpret_cast<const double2*>(&As[l][rows[u]]);
          a[u] = t.x; a[u + 1] = t.y;
        }
      }
      double2 b0 = *reinterpret_cast<const double2*>(&Bs[l][c0]);
      double2 b1 = *reinterpret_cast<const double2*>(&Bs[l][c1]);
#pragma unroll
      for (int u = 0; u < TM; ++u) {
        acc[u][0] = fma(a[u], b0.x, acc[u][0]);
        acc[u][1] = fma(a[u], b0.y, acc[u][1]);
        acc[u][2] = fma(a[u], b1.x, acc[u][2]);
        acc[u][3] = fma(a[u], b1.y, acc[u][3]);
      }
    }
    __syncthreads();
  }

  const int cols[4] = {c0, c0 + 1, c1, c1 + 1};
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    int gj = n0 + cols[v];
    if (gj >= N) continue;
    long long cc = mapC ? __ldg(mapC + gj) : gj;
    double* Cc = C + cc * ldc;
#pragma unroll
    for (int u = 0; u < TM; ++u) {
      int gi = m0 + rows[u];
      if (gi >= M) continue;
      double r = alpha * acc[u][v];
      if (beta != 0.0) r = fma(beta, Cc[gi], r);
      Cc[gi] = r;
    }
  }
}

template <int BM, int TM>
void launch_variant(bool ta, bool tb, dim3 grid, cudaStream_t s, const GemmDesc* d, const int* pre,
                    int np, double* X0, double* X1, int ldx, int Mg) {
  if (!ta && !tb) gemm_vb_kernel<BM, TM, false, false><<<grid, NT, 0, s>>>(d, pre, np, X0, X1, ldx, Mg);
  else if (ta && !tb) gemm_vb_kernel<BM, TM, true, false><<<grid, NT, 0, s>>>(d, pre, np, X0, X1, ldx, Mg);
  else if (!ta && tb) gemm_vb_kernel<BM, TM, false, true><<<grid, NT, 0, s>>>(d, pre, np, X0, X1, ldx, Mg);
  else gemm_vb_kernel<BM, TM, true, true><<<grid, NT, 0, s>>>(d, pre, np, X0, X1, ldx, Mg);
}

}  // namespace

void GemmBatch::finalize(cudaStream_t s) const {
  std::vector<int> pre(h_.size() + 1, 0);
  maxM_ = 0;
  glob_ = false;
  for (size_t i = 0; i < h_.size(); ++i) {
    const GemmDesc& d = h_[i];
    int tn = (d.N > 0 && d.M != 0) ? ceil_div(d.N, BN) : 0;
    pre[i + 1] = pre[i] + tn;
    if (d.M < 0) glob_ = true; else maxM_ = std::max(maxM_, d.M);
  }
  totalN_ = pre.back();
  d_.alloc(h_.size(), s);
  d_.upload(h_);
  prefix_.alloc(pre.size(), s);
  prefix_.upload(pre);
  ready_ = true;
}

void GemmBatch::run(cudaStream_t s, double* X0, double* X1, int ldx, int Mglob) const {
  if (h_.empty()) return;
  if (!ready_) finalize(s);
  if (totalN_ == 0) return;
  int M = std::max(maxM_, glob_ ? Mglob : 0);
  if (M <= 0) return;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (KStats::on) KStats::record(s, &e0, nullptr);
  if (M <= 16) {
    dim3 grid(totalN_, ceil_div(M, 16));
    launch_variant<16, 1>(ta_, tb_, grid, s, d_.p, prefix_.p, (int)h_.size(), X0, X1, ldx, Mglob);
  } else {
    dim3 grid(totalN_, ceil_div(M, 64));
    launch_variant<64, 4>(ta_, tb_, grid, s, d_.p, prefix_.p, (int)h_.size(), X0, X1, ldx, Mglob);
  }
  if (KStats::on) {
    KStats::record(s, nullptr, &e1);
    // algorithmic flops 2MNK; compulsory bytes: A, B read once, C written (and read if beta != 0)
    double f = 0, b = 0;
    for (const auto& d : h_) {
      const double m = d.M < 0 ? Mglob : d.M;
      f += 2.0 * m * d.N * d.K;
      b += 8.0 * (m * d.K + (double)d.K * d.N + m * d.N * (d.beta != 0.0 ? 2.0 : 1.0));
    }
    KStats::push(e0, e1, f, b);
  }
  count_launch();
  RSF_LAUNCH_CHECK();
}

double GemmBatch::flops(int Mglob) const {
  double f = 0;
  for (auto& d : h_) f += 2.0 * (d.M < 0 ? Mglob : d.M) * (double)d.N * d.K;
  return f;
}

void gemm1(cudaStream_t s, bool ta, bool tb, int M, int N, int K, double alpha, const double* A,
           int lda, const double* B, int ldb, double beta, double* C, int ldc) {
  if (M <= 0 || N <= 0) return;
  GemmBatch g(ta, tb);
  GemmDesc d = gdesc(M, N, K);
  d.A = A; d.lda = lda; d.B = B; d.ldb = ldb; d.C = C; d.ldc = ldc;
  d.alpha = alpha; d.beta = beta;
  g.add(d);
  g.run(s);
}

}  // namespace rsf

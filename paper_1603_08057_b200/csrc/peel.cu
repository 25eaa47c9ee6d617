// Weak-admissibility matrix peeling of a black-box symmetric operator G
// (PAPER §3.2) on the GPU, and Alg. 1.
//
//   for l = 1..L (top-down):
//     W^(l)_k : Gaussian probes on the level-l boxes with quadrant k (R-R),
//               Philox4x32-10 counters (point, column, level, trace) -> Box-Muller
//     Y_k = G W_k - sum_{m<l} G^(m) W_k
//     per ordered sibling pair (i,j): U_ij = orth(Y_k(j)(I_i,:)) by Householder QR +
//       truncated CPQR at eps_peel (R-N); adaptive widths (R-M)
//     M_ij = (W_i^T U_ij)^+ (W_i^T Y_ij) (U_ji^T W_j)^+               (Eq. lowrankapprox)
//   extraction: H = (G - sum G^(m)) E, Tr = sum of leaf-block traces
//
// G X = 1/2 (F^-1 (F_i X) + F_i (F^-1 X)) or G = F^-1 (reading R-G).
// Everything runs on X' blocks (columns = probes, tree order) through the
// batched GEMM; the per-pair dense work uses the batched QR/CPQR/Cholesky.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <thread>
#include <functional>
#include <unordered_map>
#include <future>

#include "dense.cuh"
#include "peel.cuh"
#include "rrqr.cuh"
#include "rsf_kernels.cuh"

namespace rsf {

namespace {

constexpr int NT = 256;

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k.x += 0x9E3779B9u; k.y += 0xBB67AE85u; }
    const unsigned hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const unsigned hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

__device__ __forceinline__ double probe_normal(unsigned j, unsigned col, unsigned lev, unsigned tr,
                                               unsigned seed) {
  uint4 x = philox4x32_10(make_uint4(j, col, lev, tr), make_uint2(seed, 3u));
  const double u1 = ((double)(x.x >> 5) * 67108864.0 + (double)(x.y >> 6)) * (1.0 / 9007199254740992.0);
  const double u2 = ((double)(x.z >> 5) * 67108864.0 + (double)(x.w >> 6)) * (1.0 / 9007199254740992.0);
  return sqrt(-2.0 * log1p(-u1)) * cos(6.283185307179586 * u2);
}

__global__ void probes_kernel(double* X, int k, int t0, int t1, const int* __restrict__ perm,
                              const int* __restrict__ qmap, int g, int col0, int lev, int tr, unsigned seed,
                              long long ldx) {
  const long long tot = (long long)(t1 - t0) * k;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    const int t = t0 + (int)(e / k), j = (int)(e % k);
    double v = 0.0;
    if (!qmap || qmap[t] == g) v = probe_normal((unsigned)perm[t], (unsigned)(col0 + j), (unsigned)lev, (unsigned)tr, seed);
    X[(long long)(t - t0) * ldx + j] = v;
  }
}

// Hutchinson probes (R-W stream 4): X'(j, t) = +-1 from bit 0 of the first Philox
// word of counter (perm[t], col0 + j, 0, 0) under key (seed, 4)
__global__ void rademacher_kernel(double* X, int k, int n, const int* __restrict__ perm, int col0, unsigned seed) {
  const long long tot = (long long)n * k;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    const int t = (int)(e / k), j = (int)(e % k);
    const uint4 x = philox4x32_10(make_uint4((unsigned)perm[t], (unsigned)(col0 + j), 0u, 0u), make_uint2(seed, 4u));
    X[e] = (x.x & 1u) ? -1.0 : 1.0;
  }
}

// per-row dot products of two k x n X'-blocks: part[b * k + j] = sum_{t in block b} A'(j,t) B'(j,t)
__global__ void rowdot_kernel(const double* __restrict__ A, const double* __restrict__ B, int k, int n,
                              double* part) {
  const int per = (n + gridDim.x - 1) / gridDim.x;
  const int t0 = blockIdx.x * per, t1 = min(n, t0 + per);
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    double acc = 0.0;
    for (int t = t0; t < t1; ++t) acc += A[(long long)t * k + j] * B[(long long)t * k + j];
    part[(long long)blockIdx.x * k + j] = acc;
  }
}

// probe rows of a list of tree indices: X'(j, q) = normal(perm[rows[q]], col0 + j, level, trace)
__global__ void probes_rows_kernel(double* X, int k, const int* __restrict__ rows, long long nrows,
                                   const int* __restrict__ perm, int col0, int lev, int tr, unsigned seed) {
  const long long tot = nrows * k;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    const long long q = e / k;
    const int j = (int)(e - q * k);
    X[e] = probe_normal((unsigned)perm[rows[q]], (unsigned)(col0 + j), (unsigned)lev, (unsigned)tr, seed);
  }
}

// dst rows [r0, r0+k) of a (cap x n) X'-matrix <- src (k x n)
__global__ void rowblock_copy_kernel(double* dst, long long ldd, int r0, const double* src, int k, int n) {
  const long long tot = (long long)n * k;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    const long long t = e / k;
    const int j = (int)(e - t * k);
    dst[t * ldd + r0 + j] = src[e];
  }
}

// U (ni x k, ld ni) <- [I_k; 0]
struct EyeDesc { double* U; int ni, k; };
__global__ void eye_kernel(const EyeDesc* __restrict__ descs) {
  const EyeDesc d = descs[blockIdx.y];
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < (long long)d.ni * d.k; e += (long long)gridDim.x * NT) {
    const int r = (int)(e % d.ni), c = (int)(e / d.ni);
    d.U[e] = (r == c) ? 1.0 : 0.0;
  }
}

// E' (k x n): 1 where t - leafbegin[t] == e0 + j (and, with a class map, cls[t] == kappa)
__global__ void extract_probe_kernel(double* X, int k, int n, const int* __restrict__ lb, int e0,
                                     const int* __restrict__ cls = nullptr, int kappa = 0) {
  const long long tot = (long long)n * k;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    const int t = (int)(e / k), j = (int)(e % k);
    X[e] = (t - lb[t] == e0 + j && (!cls || cls[t] == kappa)) ? 1.0 : 0.0;
  }
}

// per-block partial sums of diag entries H'(t - lb[t] - e0, t) and of their magnitudes
__global__ void extract_diag_kernel(const double* H, int k, int n, const int* __restrict__ lb, int e0,
                                    double* part, double* parta, const int* __restrict__ cls = nullptr,
                                    int kappa = 0) {
  __shared__ double s1[NT], s2[NT];
  double a = 0.0, b = 0.0;
  for (int t = blockIdx.x * NT + threadIdx.x; t < n; t += gridDim.x * NT) {
    const int j = t - lb[t] - e0;
    if (j >= 0 && j < k && (!cls || cls[t] == kappa)) {
      const double v = H[(long long)t * k + j];
      a += v;
      b += fabs(v);
    }
  }
  s1[threadIdx.x] = a;
  s2[threadIdx.x] = b;
  __syncthreads();
  for (int o = NT / 2; o; o >>= 1) {
    if (threadIdx.x < o) { s1[threadIdx.x] += s1[threadIdx.x + o]; s2[threadIdx.x] += s2[threadIdx.x + o]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) { part[blockIdx.x] = s1[0]; parta[blockIdx.x] = s2[0]; }
}

__global__ void dot_kernel(const double* a, const double* b, long long n, double* part) {
  __shared__ double s[NT];
  double v = 0.0;
  for (long long i = blockIdx.x * (long long)NT + threadIdx.x; i < n; i += (long long)gridDim.x * NT) v += a[i] * b[i];
  s[threadIdx.x] = v;
  __syncthreads();
  for (int o = NT / 2; o; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}

__global__ void fill_kernel(double* y, double v, long long n) {
  for (long long i = blockIdx.x * (long long)NT + threadIdx.x; i < n; i += (long long)gridDim.x * NT) y[i] = v;
}

// out_a = sum_j sigma2 k(x'_a - x_j) u_j  (conditional mean, Remark conditional P:680-690): data
// coordinates and u staged in shared memory tiles, one new point per thread
__global__ void __launch_bounds__(NT) cross_matvec_kernel(const double* __restrict__ xs, const double* __restrict__ ys,
                                                          const double* __restrict__ u, int n,
                                                          const double* __restrict__ xyn, long long m, KParams kp,
                                                          double* out) {
  __shared__ double sx[NT], sy[NT], su[NT];
  for (long long a0 = (long long)blockIdx.x * NT; a0 < m; a0 += (long long)gridDim.x * NT) {
    const long long a = a0 + threadIdx.x;
    const double px = a < m ? xyn[2 * a] : 0.0, py = a < m ? xyn[2 * a + 1] : 0.0;
    double acc = 0.0;
    for (int j0 = 0; j0 < n; j0 += NT) {
      __syncthreads();
      const int j = j0 + threadIdx.x;
      sx[threadIdx.x] = j < n ? xs[j] : 0.0;
      sy[threadIdx.x] = j < n ? ys[j] : 0.0;
      su[threadIdx.x] = j < n ? u[j] : 0.0;
      __syncthreads();
      const int cnt = min(NT, n - j0);
      for (int q = 0; q < cnt; ++q) acc += entry_xy(kp, W_SIGMA, px - sx[q], py - sy[q], false) * su[q];
    }
    if (a < m) out[a] = acc;
  }
}

__global__ void axpby_kernel(double* y, const double* x, double a, double b, long long n) {
  for (long long i = blockIdx.x * (long long)NT + threadIdx.x; i < n; i += (long long)gridDim.x * NT)
    y[i] = a * x[i] + b * y[i];
}

int gxx(long long elems) {
  return (int)std::max<long long>(1, std::min<long long>((elems + NT - 1) / NT, 4096));
}

template <class D>
DBuf<D> up(const std::vector<D>& v, cudaStream_t s) {
  DBuf<D> b(std::max<size_t>(v.size(), 1), s);
  b.upload(v);
  return b;
}

// ----------------------------------------------------------------- G operator
// Z' rows [r0, r0+k) of a (cap x n) X'-matrix -> dst (k x n)
__global__ void rowblock_extract_kernel(double* dst, const double* src, long long lds, int r0, int k, int n) {
  const long long tot = (long long)n * k;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    const long long t = e / k;
    const int j = (int)(e - t * k);
    dst[e] = src[t * lds + r0 + j];
  }
}

// Y = 1/2 (Z'(rows [k, 2k)) + D)   (Z' is 2k x n, Y and D are k x n)
__global__ void half_sum_kernel(double* Y, const double* Z, const double* D, int k, int n) {
  const long long tot = (long long)n * k;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    const long long t = e / k;
    const int j = (int)(e - t * k);
    Y[e] = 0.5 * (Z[t * 2 * k + k + j] + D[e]);
  }
}

struct GOp {
  const Fact& F;
  const Fact* Fi;
  cudaStream_t s;
  DBuf<double> A, B, Z, tmp;
  int kcap = 0;
  double columns = 0;
  GOp(const Fact& f, const Fact* fi) : F(f), Fi(fi), s(op_stream(f)) {}
  void reserve(int k) {
    if (k <= kcap) return;
    kcap = k;
    const size_t n = F.n();
    A.alloc(n * k, s);
    if (Fi) { B.alloc(n * k, s); Z.alloc(2 * n * k, s); }
    tmp.alloc((size_t)std::max<long long>(F.tmp_cols, 1) * (Fi ? 2 : 1) * k, s);
  }
  // Y = G X (X preserved), X and Y are k x n
  void apply(const double* X, double* Y, int k) {
    RSF_PHASE("p.G_apply", s);
    reserve(k);
    const size_t bytes = (size_t)F.n() * k * sizeof(double);
    const int n = F.n();
    columns += k;
    if (!Fi) {
      RSF_CUDA(cudaMemcpyAsync(Y, X, bytes, cudaMemcpyDeviceToDevice, s));
      solve_internal(F, Y, k, tmp.p);
      return;
    }
    static const bool sym = getenv("RSF_GOP") && std::string(getenv("RSF_GOP")) == "sym";
    if (sym) {   // G' = L^-1 F_i L^-T (same trace as F^-1 F_i, R-Z variant): 1 solve + 1 apply
      RSF_CUDA(cudaMemcpyAsync(B.p, X, bytes, cudaMemcpyDeviceToDevice, s));
      solve_half_bwd(F, B.p, k, tmp.p);
      apply_only_internal(*Fi, B.p, Y, k);
      solve_half_fwd(F, Y, k, tmp.p);
      return;
    }
    // G X = 1/2 (F^-1 (F_i X) + F_i (F^-1 X)): both solves in one 2k-column solve
    RSF_CUDA(cudaMemcpyAsync(A.p, X, bytes, cudaMemcpyDeviceToDevice, s));
    apply_only_internal(*Fi, A.p, B.p, k);                      // B = F_i X
    rowblock_copy_kernel<<<gxx((long long)n * k), NT, 0, s>>>(Z.p, 2 * k, 0, X, k, n);
    rowblock_copy_kernel<<<gxx((long long)n * k), NT, 0, s>>>(Z.p, 2 * k, k, B.p, k, n);
    count_launch(2);
    solve_internal(F, Z.p, 2 * k, tmp.p);                       // Z = F^-1 [X, F_i X]
    rowblock_extract_kernel<<<gxx((long long)n * k), NT, 0, s>>>(A.p, Z.p, 2 * k, 0, k, n);
    count_launch();
    apply_only_internal(*Fi, A.p, B.p, k);                      // B = F_i F^-1 X
    half_sum_kernel<<<gxx((long long)n * k), NT, 0, s>>>(Y, Z.p, B.p, k, n);
    count_launch();
    RSF_LAUNCH_CHECK();
  }
};

__global__ void d2f_kernel(const double* __restrict__ a, float* __restrict__ b, long long n) {
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < n; e += (long long)gridDim.x * NT) b[e] = (float)a[e];
}

// ----------------------------------------------------------------- G^(m): shared row bases
// The peeled level-m operator G^(m) is stored with one
// orthonormal row basis per box:  G^(m)_ij ~= V_i B_ij V_j^T for every ordered
// sibling pair (i, j).  V_i spans the sketches of all three blocks of box row i
// (grown group by group, truncated at eps_peel relative to each block's own
// scale), the per-pair bases of Eq. lowrankapprox are
// U_ij = V_i Z_ij, and B_ij = Z_ij M_ij Z_ji^T with B_ji = B_ij^T.
// Storage is n * r_i per level instead of 3 n k_ij.
struct PeelLevel {
  std::vector<DBuf<double>> V;   // per box: V_i (n_i x r_i, ld n_i)
  DBuf<double> Brow;
  // FP32 storage of the same (opts.peel_f32): the subtraction GEMMs read them as an
  // FP32 op(B) and compute in FP64
  bool f32 = false;
  DBuf<float> store;                 // every V_i and Brow of the level in one allocation (no bin rounding,
  std::vector<size_t> vfo;           // one long-lived block per level in the pool): V_i at vfo[i],
  size_t browf_off = 0;              // Brow at browf_off
  const void* vptr(int b) const { return f32 ? (const void*)(store.p + vfo[b]) : (const void*)V[b].p; }
  const float* browf() const { return store.p + browf_off; }
  long long tcols = 0;   // tmp columns per probe column: sum r (T') + sum r (S')
  GemmBatch g1, g2, g3;
  std::vector<int> ib, ni, r, bidx;      // boxes with r > 0: range, basis size, level box index
  std::vector<long long> toff;           // T' column offsets
  // Y' -= G^(m) X'   (X', Y' are k x n; tmp has k * tcols doubles).  g1x (optional) replaces
  // the first step by a K-gathered version for right-hand sides known to vanish outside a
  // row subset (block-sparse probes)
  void subtract(cudaStream_t s, const double* X, double* Y, int k, double* tmp, const GemmBatch* g1x = nullptr,
                const GemmBatch* g3x = nullptr) const {
    if (g3.empty()) return;
    (g1x ? *g1x : g1).run(s, const_cast<double*>(X), tmp, k, k);   // T'_j = X'(:, I_j) V_j
    g2.run(s, nullptr, tmp, k, k);                  // S'_i = [T'_f]_{f in family(i)} Brow_i^T
    if (g3x && g3x->empty()) return;                // no row of Y' is needed
    (g3x ? *g3x : g3).run(s, Y, tmp, k, k);         // Y'(:, I_i) -= S'_i V_i^T
  }
  std::vector<long long> soff;           // S' column offsets
  DBuf<int> mapk;                        // strong admissibility: T' columns of IL(b), per box
};

// out (rows x q, ld rows) = transpose of rows piv[0:q] of src (c x rows, ld lds)
struct GatherTDesc { const double* src; long long lds; const int* piv; double* out; int rows, q; };
// 32 x 32 tiles through shared memory: the gathered rows piv[j0:j0+32] of one source column
// are read together (one 8*c-byte column, L1/L2 resident), the output columns are written
// coalesced (a direct element-per-thread transpose reads with stride lds).
constexpr int GT_TILE = 32, GT_ROWS = 8;
__global__ void __launch_bounds__(GT_TILE * GT_ROWS) gather_t_kernel(const GatherTDesc* __restrict__ descs) {
  __shared__ double tile[GT_TILE][GT_TILE + 1];
  const GatherTDesc d = descs[blockIdx.z];
  const int tilesT = (d.rows + GT_TILE - 1) / GT_TILE, tilesJ = (d.q + GT_TILE - 1) / GT_TILE;
  const int tx = threadIdx.x, ty0 = threadIdx.y;
  for (int ti = blockIdx.x; ti < tilesT * tilesJ; ti += gridDim.x) {
    const int t0 = (ti % tilesT) * GT_TILE, j0 = (ti / tilesT) * GT_TILE;
    const int jl = j0 + tx;
    const long long pj = jl < d.q ? __ldg(d.piv + jl) : 0;
    for (int ty = ty0; ty < GT_TILE; ty += GT_ROWS) {
      const int t = t0 + ty;
      if (t < d.rows && jl < d.q) tile[ty][tx] = d.src[(long long)t * d.lds + pj];
    }
    __syncthreads();
    for (int ty = ty0; ty < GT_TILE; ty += GT_ROWS) {
      const int j = j0 + ty, t = t0 + tx;
      if (t < d.rows && j < d.q) d.out[(long long)j * d.rows + t] = tile[tx][ty];
    }
    __syncthreads();
  }
}
void launch_gather_t(cudaStream_t s, const std::vector<GatherTDesc>& v) {
  if (v.empty()) return;
  long long mt = 1;
  for (auto& d : v) mt = std::max<long long>(mt, (long long)((d.rows + GT_TILE - 1) / GT_TILE) * ((d.q + GT_TILE - 1) / GT_TILE));
  auto dd = ring_up(v, s);
  for (size_t o = 0; o < v.size(); o += 65535) {
    const unsigned nz = (unsigned)std::min<size_t>(65535, v.size() - o);
    gather_t_kernel<<<dim3((unsigned)std::min<long long>(mt, 2048), 1, nz), dim3(GT_TILE, GT_ROWS), 0, s>>>(dd.p + o);
    count_launch();
  }
  RSF_LAUNCH_CHECK();
}

// out = max(out, max_j ||A(:, j)||)   (one CTA per problem)
struct ColMaxDesc { const double* A; long long lda; int rows, cols; double* out; };
__global__ void colmax_kernel(const ColMaxDesc* __restrict__ descs) {
  const ColMaxDesc d = descs[blockIdx.x];
  __shared__ double red[NT / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double mx = 0.0;
  for (int j = warp; j < d.cols; j += NT / 32) {
    const double* a = d.A + (long long)j * d.lda;
    double v = 0.0;
    for (int r = lane; r < d.rows; r += 32) v += a[r] * a[r];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    mx = fmax(mx, v);
  }
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int w = 0; w < NT / 32; ++w) v = fmax(v, red[w]);
    *d.out = fmax(*d.out, sqrt(v));
  }
}

void launch_colmax(cudaStream_t s, const std::vector<ColMaxDesc>& v) {
  if (v.empty()) return;
  auto d = ring_up(v, s);
  for (size_t o = 0; o < v.size(); o += 65535) {
    colmax_kernel<<<(unsigned)std::min<size_t>(65535, v.size() - o), NT, 0, s>>>(d.p + o);
    count_launch();
  }
  RSF_LAUNCH_CHECK();
}

// diagnostics: histogram of row norms of V_i (counts of rows with ||V(t,:)|| < 1e-12, 1e-10, 1e-8, 1e-6)
__global__ void rownorm_hist_kernel(const double* __restrict__ V, int rows, int cols, unsigned long long* cnt) {
  for (int t = blockIdx.x * NT + threadIdx.x; t < rows; t += gridDim.x * NT) {
    double s = 0.0;
    for (int j = 0; j < cols; ++j) { const double v = V[(long long)j * rows + t]; s += v * v; }
    const double nr = sqrt(s);
    if (nr < 1e-12) atomicAdd(cnt + 0, 1ull);
    if (nr < 1e-10) atomicAdd(cnt + 1, 1ull);
    if (nr < 1e-8) atomicAdd(cnt + 2, 1ull);
    if (nr < 1e-6) atomicAdd(cnt + 3, 1ull);
  }
}

template <class D, class K>
void launch_descs(cudaStream_t s, const std::vector<D>& v, long long maxelems, K kern) {
  if (v.empty() || maxelems <= 0) return;
  auto d = ring_up(v, s);
  for (size_t o = 0; o < v.size(); o += 65535) {
    const unsigned nz = (unsigned)std::min<size_t>(65535, v.size() - o);
    kern<<<dim3(gxx(maxelems), nz), NT, 0, s>>>(d.p + o);
    count_launch();
  }
  RSF_LAUNCH_CHECK();
}

// failure flags of batched factorizations, checked once per level instead of a host
// synchronisation per call
__global__ void info_or_kernel(const int* __restrict__ info, int n, int* flag) {
  for (int i = blockIdx.x * NT + threadIdx.x; i < n; i += gridDim.x * NT)
    if (info[i]) atomicOr(flag, 1);
}
void flag_infos(cudaStream_t s, const int* info, int n, int* dflag) {
  if (n <= 0) return;
  info_or_kernel<<<std::max(1, std::min(64, (n + NT - 1) / NT)), NT, 0, s>>>(info, n, dflag);
  count_launch();
}

// U <- orth(U) by two passes of U <- U chol(U^T U)^-T (CholeskyQR2), in place.
struct CQProb { double* U; int rows, k; };
void cholqr2_batched(cudaStream_t s, const std::vector<CQProb>& v, int lev, double* flops, int* dflag) {
  std::vector<CQProb> w;
  for (auto& p : v) if (p.k > 0 && p.rows > 0) w.push_back(p);
  if (w.empty()) return;
  long long st = 0, gt = 0;
  std::vector<long long> so(w.size()), go(w.size());
  for (size_t x = 0; x < w.size(); ++x) {
    so[x] = st; st += (long long)w[x].rows * w[x].k;
    go[x] = gt; gt += (long long)w[x].k * w[x].k;
  }
  DBuf<double> S(st, s), G(gt, s), Gi(gt, s), ls(w.size(), s);
  DBuf<int> inf(w.size(), s);
  for (int pass = 0; pass < 2; ++pass) {
    GemmBatch gg(true, false), gu(false, true);
    std::vector<PotrfProb> pp;
    for (size_t x = 0; x < w.size(); ++x) {
      const auto& p = w[x];
      double* src = pass == 0 ? p.U : S.p + so[x];
      double* dst = pass == 0 ? S.p + so[x] : p.U;
      GemmDesc d = gdesc(p.k, p.k, p.rows);        // Gram = U^T U
      d.A = src; d.lda = p.rows; d.B = src; d.ldb = p.rows; d.C = G.p + go[x]; d.ldc = p.k;
      gg.add(d);
      pp.push_back(PotrfProb{G.p + go[x], p.k, p.k, Gi.p + go[x], p.k});
      GemmDesc e = gdesc(p.rows, p.k, p.k);        // U <- U L^-T
      e.A = src; e.lda = p.rows; e.B = Gi.p + go[x]; e.ldb = p.k; e.C = dst; e.ldc = p.rows;
      e.btri = 2;
      gu.add(e);
      if (flops) *flops += 4.0 * p.rows * (double)p.k * p.k;
    }
    gg.run(s);
    potrf_batched(s, pp, ls.p, inf.p);
    flag_infos(s, inf.p, (int)w.size(), dflag);
    gu.run(s);
  }
}

struct PBox { int node, ib, ni, fam0, fam1, quad; };

}  // namespace

void gen_probes(cudaStream_t s, double* X, int k, int n, const int* perm, const int* qmap, int g,
                int col0, int level, int trace, unsigned long long seed) {
  probes_kernel<<<gxx((long long)n * k), NT, 0, s>>>(X, k, 0, n, perm, qmap, g, col0, level, trace,
                                                     (unsigned)(seed & 0xffffffffull), k);
  count_launch();
  RSF_LAUNCH_CHECK();
}

double ddot(cudaStream_t s, const double* a, const double* b, long long n) {
  const int G = 256;
  DBuf<double> part(G, s);
  dot_kernel<<<G, NT, 0, s>>>(a, b, n, part.p);
  count_launch();
  RSF_LAUNCH_CHECK();
  auto h = part.to_host(G);
  double r = 0.0;
  for (double v : h) r += v;
  return r;
}

double peel(const Fact& F, const Fact* Fi, const Opts& o, int trace_id, PeelDiag* diag, const Comm* comm) {
  // memory-saving mode: large blocks via cudaMalloc/cudaFree, from a trimmed pool (
  // measured faster than stream-ordered transients without arenas: 246.5 vs 268.5 s at config 4)
  BigSyncScope big_sync(o.peel_f32 != 0);
  const double t0 = now_s();
  cudaStream_t s = op_stream(F);
  Comm cm = comm ? *comm : F.ctx->comm;
  if (cm.world == 1) {   // one-process emulation of a rank group (tests; comm.cuh)
    const char* e = getenv("RSF_EMU_WORLD");
    cm.emu = e ? std::max(1, atoi(e)) : 1;
  }
  const int NP = cm.parts();
  const Tree& t = *F.tree;
  const int n = t.n, L = t.L;
  const unsigned long long seed = o.seed;
  const unsigned seed32 = (unsigned)(seed & 0xffffffffull);
  GOp G(F, Fi);
  std::vector<PeelLevel> peeled(L + 1);
  long long max_tcols = 0;
  PeelDiag pd;
  DBuf<int> dfail(1, s);   // set by any failed Cholesky of the level (CholeskyQR, core Gram matrices)
  dfail.zero();
  pd.cols.assign(L + 1, 0);
  pd.rank_max.assign(L + 1, 0);
  pd.rank_min.assign(L + 1, 0);
  pd.rank_med.assign(L + 1, 0);
  std::vector<int> lev_ranks;
  int prev_rank = -1;
  const int kb = std::max(16, o.probe_block);
  // bytes of transient per-batch buffers, and of W_i^T kept for a whole probe group (else the
  // probes are regenerated per batch).  RSF_PEEL_BUDGET_MB / RSF_PEEL_WCACHE_MB shrink them
  // (tests force the batch-split and regeneration paths at small sizes).
  auto env_mb = [](const char* k, double d) {
    const char* v = getenv(k);
    return (v && atof(v) >= 0) ? atof(v) * (1 << 20) : d;
  };
  // (memory-saving mode, opts.peel_f32: 4 GB / 2 GB -- DESIGN.md §7g)
  const double budget = env_mb("RSF_PEEL_BUDGET_MB", (o.peel_f32 ? 4.0 : 16.0) * (1ull << 30));
  const double wcache_budget = env_mb("RSF_PEEL_WCACHE_MB", (o.peel_f32 ? 2.0 : 8.0) * (1ull << 30));

  struct SparseSub { std::vector<GemmBatch> g1, g3; std::vector<char> has1, has3; };
  auto residual = [&](const double* W, double* Y, int k, int upto, const SparseSub* sp) {
    G.apply(W, Y, k);
    DBuf<double> tmp((size_t)std::max<long long>(max_tcols, 1) * k, s);
    RSF_PHASE("p.subtract", s);
    for (int m = 1; m < upto; ++m)
      peeled[m].subtract(s, W, Y, k, tmp.p, sp && sp->has1[m] ? &sp->g1[m] : nullptr,
                         sp && sp->has3[m] ? &sp->g3[m] : nullptr);
  };
  // T'_j = X'(:, I_j) V_j restricted to the rows where the level-l group-g probes are nonzero
  // ... and Y'(:, I_i) -= S'_i V_i^T only on the rows the level-l sketch uses (boxes of the
  // other three quadrants), as contiguous row ranges
  auto sparse_g1 = [&](const std::vector<int>& hq, int g, int upto, std::vector<DBuf<int>>& keep) {
    SparseSub sp;
    sp.g1.resize(upto);
    sp.g3.resize(upto);
    sp.has1.assign(upto, 0);
    sp.has3.assign(upto, 0);
    std::vector<GemmBatch>& out = sp.g1;
    for (int m = 1; m < upto; ++m) {
      const PeelLevel& P = peeled[m];
      if (P.g3.empty()) continue;
      std::vector<int> idx;
      std::vector<long long> off(P.ib.size() + 1, 0);
      for (size_t b = 0; b < P.ib.size(); ++b) {
        for (int t = 0; t < P.ni[b]; ++t)
          if (hq[P.ib[b] + t] == g) idx.push_back(t);
        off[b + 1] = idx.size();
      }
      keep.emplace_back(up(idx, s));
      const int* dk = keep.back().p;
      out[m].reset(false, false);
      for (size_t b = 0; b < P.ib.size(); ++b) {
        GemmDesc a = gdesc(-1, P.r[b], (int)(off[b + 1] - off[b]));
        a.selA = 1; a.offA = P.ib[b]; a.B = (const double*)P.vptr(P.bidx[b]); a.bf32 = P.f32; a.ldb = P.ni[b];
        a.selC = 2; a.offC = P.toff[b];
        a.mapK = dk + off[b];
        out[m].add(a);
      }
      out[m].finalize(s);
      sp.has1[m] = 1;
      sp.g3[m].reset(false, true);
      for (size_t b = 0; b < P.ib.size(); ++b) {
        int t = 0;
        while (t < P.ni[b]) {
          const int q = hq[P.ib[b] + t];
          if (q < 0 || q == g) { ++t; continue; }
          int e = t + 1;
          while (e < P.ni[b] && hq[P.ib[b] + e] >= 0 && hq[P.ib[b] + e] != g) ++e;
          GemmDesc d = gdesc(-1, e - t, P.r[b]);
          d.selA = 2; d.offA = P.soff[b]; d.B = (const double*)P.vptr(P.bidx[b]); d.offB = t; d.bf32 = P.f32;
          d.ldb = P.ni[b];
          d.selC = 1; d.offC = P.ib[b] + t; d.alpha = -1.0; d.beta = 1.0;
          sp.g3[m].add(d);
          t = e;
        }
      }
      if (!sp.g3[m].empty()) sp.g3[m].finalize(s);
      sp.has3[m] = 1;
    }
    return sp;
  };

  static const int verbose = getenv("RSF_VERBOSE") ? atoi(getenv("RSF_VERBOSE")) : 0;
  static const int max_lev = getenv("RSF_PEEL_LEVELS") ? atoi(getenv("RSF_PEEL_LEVELS")) : 1 << 30;
  // admissibility (next row f4): weak -- partners of a box are its siblings,
  // probe groups the 4 quadrants; strong -- partners are the interaction list
  // IL(b) = children of the parent's 3 x 3 neighbourhood not adjacent to b, probe groups the 36
  // classes (ix mod 6, iy mod 6) (each 6 x 6 window of a parent neighbourhood holds one box per
  // class), levels 2..L of a perfect quadtree
  const bool strong = o.strong != 0;
  if (strong)
    for (int l = 0; l <= L; ++l)
      RSF_REQUIRE((long long)t.levels[l].size() == (1ll << (2 * l)), ST_EINVAL,
                  "strong-admissibility peeling needs a perfect quadtree (every leaf at depth L)");
  for (int lev = strong ? 2 : 1; lev <= std::min(L, max_lev); ++lev) {
    const std::vector<int>& nodes = t.levels[lev];
    const int nb = (int)nodes.size();
    // boxes and families (siblings are consecutive in Morton order; Def. sibs)
    std::vector<PBox> bx(nb);
    int maxni = 0;
    for (int b = 0; b < nb; ++b) {
      const int nd = nodes[b];
      bx[b].node = nd; bx[b].ib = t.begin[nd]; bx[b].ni = t.end[nd] - t.begin[nd]; bx[b].quad = t.quad[nd];
      maxni = std::max(maxni, bx[b].ni);
    }
    int npairs = 0;
    for (int b = 0; b < nb;) {
      int e = b;
      while (e < nb && t.parent[nodes[e]] == t.parent[nodes[b]]) ++e;
      for (int x = b; x < e; ++x) { bx[x].fam0 = b; bx[x].fam1 = e; }
      npairs += (e - b) * (e - b - 1);
      b = e;
    }
    // part[b]: partner boxes (ascending); rowset[b]: the boxes whose cores form b's row of
    // Brow (weak: the whole family, b's own zero block included; strong: IL(b)); grp[b]: group
    const int NGRP = strong ? 36 : 4;
    std::vector<std::vector<int>> part(nb), rowset(nb);
    std::vector<int> grp(nb);
    if (!strong) {
      for (int b = 0; b < nb; ++b) {
        grp[b] = bx[b].quad;
        for (int x = bx[b].fam0; x < bx[b].fam1; ++x) {
          rowset[b].push_back(x);
          if (x != b) part[b].push_back(x);
        }
      }
    } else {
      std::unordered_map<long long, int> at;
      for (int b = 0; b < nb; ++b) at[(long long)t.ix[nodes[b]] * (1ll << 31) + t.iy[nodes[b]]] = b;
      npairs = 0;
      for (int b = 0; b < nb; ++b) {
        const int x = t.ix[nodes[b]], y = t.iy[nodes[b]];
        grp[b] = (x % 6) * 6 + (y % 6);
        const int px = x / 2, py = y / 2;
        for (int cx = 2 * px - 2; cx < 2 * px + 4; ++cx)
          for (int cy = 2 * py - 2; cy < 2 * py + 4; ++cy) {
            if (std::max(std::abs(cx - x), std::abs(cy - y)) <= 1) continue;
            auto it = at.find((long long)cx * (1ll << 31) + cy);
            if (it != at.end()) part[b].push_back(it->second);
          }
        std::sort(part[b].begin(), part[b].end());
        rowset[b] = part[b];
        npairs += (int)part[b].size();
      }
    }
    if (npairs == 0) continue;
    // pair slots: (b, position of the partner in part[b])
    std::vector<long long> pslot0(nb + 1, 0);
    for (int b = 0; b < nb; ++b) pslot0[b + 1] = pslot0[b] + (long long)part[b].size();
    auto pslot = [&](int b, int x) -> size_t {
      const auto& v = part[b];
      return (size_t)(pslot0[b] + (std::lower_bound(v.begin(), v.end(), x) - v.begin()));
    };
    // probe groups: W_g on the boxes of group g (quadrant R-R, or class), largest groups first
    std::vector<int> gcount(NGRP, 0);
    for (int b = 0; b < nb; ++b) if (!part[b].empty()) gcount[grp[b]]++;
    std::vector<int> gorder(NGRP);
    for (int g = 0; g < NGRP; ++g) gorder[g] = g;
    std::stable_sort(gorder.begin(), gorder.end(), [&](int a2, int b2) { return gcount[a2] > gcount[b2]; });
    std::vector<int> hq(n, -1);
    for (int b = 0; b < nb; ++b)
      for (int x = bx[b].ib; x < bx[b].ib + bx[b].ni; ++x) hq[x] = grp[b];
    DBuf<int> qmap = up(hq, s);
    const int cmax = ((maxni + o.oversample) + 7) / 8 * 8;
    // initial width (R-M): level 1 from the factor's level-1 skeleton sizes, deeper levels
    // from the previous level's ranks
    int hint = o.peel_start;
    if (prev_rank < 0 && F.levels.size() > 1)
      for (int kk : F.levels[1].k) hint = std::max(hint, kk);
    // (0.6: the eps_peel-rank a sketch reveals grows with its width, so a wide first guess is
    // accepted at a higher rank and inflates every later level; measured at config 3: 0.6 with one
    // restart 25.1 s per evaluation, 0.75 without restarts 27.8 s)
    int c = (prev_rank < 0) ? (strong ? o.peel_start : (int)std::ceil(0.6 * hint)) : prev_rank + o.oversample;
    int restarts = 0;
    c = std::min(std::max(c, o.oversample + 8), cmax);
    c = (c + 7) / 8 * 8;

    // per-level state (reset when the width grows)
    std::vector<int> rb(nb, 0);                   // basis size r_i
    std::vector<DBuf<double>> Vb(nb), Ab(nb);     // V_i (n_i x r_i, ld n_i), A_i = W_i^T V_i (c x r_i, ld c)
    std::vector<int> vcap(nb, 0);                 // allocated columns of V_i / A_i (grown exactly)
    std::vector<int> vmax(nb, 0);                 // most columns V_i can take: min(n_i, c per sibling group)
    // per ordered pair (index: pslot(b, partner))
    struct PairData { int k = 0, rz = 0, arena = -1; double *Z = nullptr, *X = nullptr, *Lm = nullptr, *Gi = nullptr; };
    std::vector<PairData> pdat((size_t)std::max<long long>(pslot0[nb], 1));
    // The per-pair data live in arenas, one per (pair-core batch, group of the act boxes); an arena is
    // released as soon as every pair it holds has its core (a pair {i, j} is complete once the groups of
    // i and of j have both been sketched), so at most ~7/12 of a level's pair data are resident at once
    // (was: all of it until the level end -- 23 GB at level 5 of config 4)
    std::vector<DBuf<double>> arenas;
    std::vector<int> arena_uses;
    double pair_bytes = 0, pair_peak = 0;   // per-pair data of the level: resident now / peak (diagnostics)
    // finished cores: B_ij blocks (rz_i x rz_j, ld rz_i) until Brow's layout (final r's) is known
    struct CBlock { int i, j; const double* p; int ri, rj; };
    std::vector<CBlock> cblocks;
    std::vector<DBuf<double>> cbufs;
    std::vector<char> gdone(NGRP, 0);
    // cores of complete pairs {i < j}: M_ij = Lm_ij (X_ji^T)^+ = Lm_ij X_ji (X_ji^T X_ji)^-1,
    // B_ij = Z_ij M_ij Z_ji^T, B_ji = B_ij^T -> blocks in cbufs; the pairs' arenas are
    // released when their last pair is done
    auto compute_cores = [&](const std::vector<std::pair<int, int>>& cand) {
      RSF_PHASE("p.cores", s);
      long long mt = 0, bt = 0;
      std::vector<std::array<long long, 4>> mo;
      std::vector<std::pair<int, int>> pl;
      for (const auto& ij : cand) {
        const int i = ij.first, j = ij.second;
        const PairData& a = pdat[pslot(i, j)];
        const PairData& b2 = pdat[pslot(j, i)];
        if (a.k == 0 || b2.k == 0) continue;
        std::array<long long, 4> m{};
        m[0] = mt; mt += (long long)a.k * b2.k;                 // T1, then M
        m[1] = mt; mt += (long long)a.k * b2.k;                 // T2
        m[2] = mt; mt += (long long)std::max(a.rz, b2.rz) * std::max(a.k, b2.k) * 2;  // T3 / T4
        m[3] = bt; bt += 2ll * a.rz * b2.rz;                    // B_ij, B_ji
        mo.push_back(m);
        pl.emplace_back(i, j);
      }
      if (!pl.empty()) {
        DBuf<double> Mw(std::max<long long>(mt, 1), s);
        cbufs.emplace_back(DBuf<double>((size_t)std::max<long long>(bt, 1), s));
        double* Bb = cbufs.back().p;
        GemmBatch m1(false, false), m2(false, true), m3(false, false), m4(false, false), m5(false, true),
            m6(false, true), m7(false, true);
        for (size_t q = 0; q < pl.size(); ++q) {
          const int i = pl[q].first, j = pl[q].second;
          const PairData& a = pdat[pslot(i, j)];
          const PairData& b2 = pdat[pslot(j, i)];
          const int k1 = a.k, k2 = b2.k;
          double* T1p = Mw.p + mo[q][0];
          double* T2p = Mw.p + mo[q][1];
          double* T3p = Mw.p + mo[q][2];
          double* T4p = T3p + (long long)std::max(a.rz, b2.rz) * std::max(k1, k2);
          double* Bij = Bb + mo[q][3];
          double* Bji = Bij + (long long)a.rz * b2.rz;
          GemmDesc d1 = gdesc(k1, k2, c);     // T1 = Lm_ij X_ji
          d1.A = a.Lm; d1.lda = k1; d1.B = b2.X; d1.ldb = c; d1.C = T1p; d1.ldc = k1;
          m1.add(d1);
          GemmDesc d2 = gdesc(k1, k2, k2);    // T2 = T1 Gi_ji^T
          d2.A = T1p; d2.lda = k1; d2.B = b2.Gi; d2.ldb = k2; d2.C = T2p; d2.ldc = k1;
          m2.add(d2);
          GemmDesc d3 = gdesc(k1, k2, k2);    // M = T2 Gi_ji   (into T1)
          d3.A = T2p; d3.lda = k1; d3.B = b2.Gi; d3.ldb = k2; d3.C = T1p; d3.ldc = k1;
          m3.add(d3);
          GemmDesc d4 = gdesc(a.rz, k2, k1);  // T3 = Z_ij M
          d4.A = a.Z; d4.lda = a.rz; d4.B = T1p; d4.ldb = k1; d4.C = T3p; d4.ldc = a.rz;
          m4.add(d4);
          GemmDesc d5 = gdesc(a.rz, b2.rz, k2);   // B_ij = T3 Z_ji^T
          d5.A = T3p; d5.lda = a.rz; d5.B = b2.Z; d5.ldb = b2.rz; d5.C = Bij; d5.ldc = a.rz;
          m5.add(d5);
          GemmDesc d6 = gdesc(b2.rz, k1, k2);     // T4 = Z_ji M^T
          d6.A = b2.Z; d6.lda = b2.rz; d6.B = T1p; d6.ldb = k1; d6.C = T4p; d6.ldc = b2.rz;
          m6.add(d6);
          GemmDesc d7 = gdesc(b2.rz, a.rz, k1);   // B_ji = T4 Z_ij^T
          d7.A = T4p; d7.lda = b2.rz; d7.B = a.Z; d7.ldb = a.rz; d7.C = Bji; d7.ldc = b2.rz;
          m7.add(d7);
          pd.flops += 2.0 * k1 * (double)k2 * c + 2.0 * a.rz * (double)b2.rz * (k1 + k2);
          cblocks.push_back(CBlock{i, j, Bij, a.rz, b2.rz});
          cblocks.push_back(CBlock{j, i, Bji, b2.rz, a.rz});
        }
        m1.run(s); m2.run(s); m3.run(s); m4.run(s); m5.run(s); m6.run(s); m7.run(s);
      }
      // release the pair data of the candidates (stream-ordered: after the GEMMs above)
      for (const auto& ij : cand)
        for (int side = 0; side < 2; ++side) {
          PairData& q = side ? pdat[pslot(ij.second, ij.first)] : pdat[pslot(ij.first, ij.second)];
          if (q.arena >= 0 && --arena_uses[q.arena] == 0) {
            pair_bytes -= 8.0 * arenas[q.arena].n;
            arenas[q.arena].release();
          }
          q.arena = -1;
        }
    };
    int mr = 0;
    while (true) {
      std::fill(rb.begin(), rb.end(), 0);
      for (auto& v : Vb) v.release();
      for (auto& v : Ab) v.release();
      // fixed capacity per box: every probe group adds at most c directions (no regrowth)
      // V_i and A_i grow to exactly the columns they take (reallocated as the chunks add
      // directions) instead of being reserved at their upper bound min(n_i, 3c): at config 4
      // the bound reserved ~50 GB per level at levels 1-3 against 17-35 GB of final bases
      // (the upper bound is still reserved up front when it is small -- <= 16 GB for the level:
      // fewer, fixed-size allocations; config 3 reserves 6 GB at level 1)
      std::fill(vcap.begin(), vcap.end(), 0);
      double vres = 0;
      for (int b = 0; b < nb; ++b) {
        const int ng = (int)part[b].size();
        vmax[b] = ng <= 0 ? 0 : std::min(bx[b].ni, ng * c);
        vres += 8.0 * bx[b].ni * (double)vmax[b];
      }
      static const double vres_max = getenv("RSF_VRESERVE_GB") ? atof(getenv("RSF_VRESERVE_GB")) * (1ull << 30)
                                                               : 16.0 * (1ull << 30);
      if (vres <= vres_max)
        for (int b = 0; b < nb; ++b) {
          if (vmax[b] == 0) continue;
          vcap[b] = vmax[b];
          Vb[b].alloc((size_t)bx[b].ni * vcap[b], s);
          Ab[b].alloc((size_t)c * vcap[b], s);
        }
      arenas.clear();
      arena_uses.clear();
      cblocks.clear();
      cbufs.clear();
      std::fill(gdone.begin(), gdone.end(), 0);
      pair_bytes = 0;
      pair_peak = 0;
      for (auto& q : pdat) q = PairData{};
      bool fail = false;
      mr = 0;
      lev_ranks.clear();
      for (int g : gorder) {
        if (gcount[g] == 0) continue;
        // boxes i with a partner j in group g (at most one: one sibling per quadrant, one box per
        // class in a parent neighbourhood)
        std::vector<int> act_all, partner_all;
        for (int b = 0; b < nb; ++b) {
          if (grp[b] == g) continue;
          for (int x : part[b])
            if (grp[x] == g) { act_all.push_back(b); partner_all.push_back(x); break; }
        }
        if (act_all.empty()) continue;
        // memory-saving mode: when the group's per-box sketch products (P_ij: c x c, C_ij: c x (r_i + c)
        // per act box -- 53 GB at level 6 of config 4) exceed a third of the free memory, the act boxes
        // are taken in subsets, each re-running the G applies of the group (same probes, same
        // residual; only the boxes whose sketches are kept differ)
        int nsub = 1;
        if (o.peel_f32) {
          double need = 0;
          for (int b : act_all) need += 8.0 * c * ((double)c + std::min<double>(bx[b].ni, rb[b] + c));
          size_t fr = 0, tot = 0;
          cudaMemGetInfo(&fr, &tot);
          if (cm.use_nccl()) {   // the same subsets on every rank of the group (their collectives pair up)
            std::vector<double> all((size_t)cm.world);
            double mine = (double)fr;
            cm.allgather_host(s, &mine, 1, all.data());
            fr = (size_t)*std::min_element(all.begin(), all.end());
          }
          const double avail = std::max(4.0 * (1ull << 30), 0.33 * (double)fr);
          nsub = std::max(1, (int)std::ceil(need / avail));
          if (verbose && nsub > 1)
            fprintf(stderr, "    level %d group %d: %zu act boxes in %d subsets (%.1f GB of sketch products, %.1f GB free)\n",
                    lev, g, act_all.size(), nsub, 1e-9 * need, 1e-9 * fr);
        }
        for (int sub = 0; sub < nsub && !fail; ++sub) {
        const size_t a0 = act_all.size() * sub / nsub, a1 = act_all.size() * (sub + 1) / nsub;
        std::vector<int> act(act_all.begin() + a0, act_all.begin() + a1), partner(partner_all.begin() + a0, partner_all.begin() + a1);
        if (act.empty()) continue;
        const size_t NA = act.size();
        // per act box, for the whole group: P_ij = W_i^T Y_ij (c x c), C_ij' = Y_ij^T [V_i ...]
        // (c x (r_i + c) upper bound, ld c), the block scale ref_ij = max_j ||W_i^T Y_ij(:, j)||
        std::vector<long long> po(NA), cco(NA), cccap(NA);
        long long pt = 0, cct = 0;
        for (size_t x = 0; x < NA; ++x) {
          const int i = act[x];
          po[x] = pt; pt += (long long)c * c;
          cccap[x] = std::min<long long>(bx[i].ni, (long long)rb[i] + c);
          cco[x] = cct; cct += (long long)c * cccap[x];
        }
        DBuf<double> P(pt, s), CC(std::max<long long>(cct, 1), s), ref(NA, s);
        if (verbose > 1) {
          size_t fr = 0, tot = 0;
          cudaMemGetInfo(&fr, &tot);
          fprintf(stderr, "    level %d group %d: act %zu width %d  P %.2f GB CC %.2f GB  free %.2f GB\n", lev, g, NA, c,
                  8e-9 * pt, 8e-9 * cct, 1e-9 * fr);
        }
        ref.zero();
        CC.zero();
        // W_i^T of every act box for the whole group when it fits (else regenerated per batch)
        std::vector<long long> wco(NA);
        long long wct = 0;
        for (size_t x = 0; x < NA; ++x) { wco[x] = wct; wct += (long long)c * bx[act[x]].ni; }
        DBuf<double> Wc;
        if (8.0 * wct <= wcache_budget) {
          Wc.alloc(wct, s);
          std::vector<int> rows;   // tree indices of the act boxes, in Wc order
          rows.reserve(wct / c);
          for (size_t x = 0; x < NA; ++x) {
            const PBox& b = bx[act[x]];
            for (int q = 0; q < b.ni; ++q) rows.push_back(b.ib + q);
          }
          DBuf<int> drows = up(rows, s);
          probes_rows_kernel<<<gxx((long long)rows.size() * c), NT, 0, s>>>(Wc.p, c, drows.p, (long long)rows.size(),
                                                                          t.d_perm.p, 0, lev, trace_id, seed32);
          count_launch();
          RSF_LAUNCH_CHECK();
        }
        // sketch Y'_g = ((G - sum_{m<l} G^(m)) W_g)^T in chunks of kb probe columns;
        // every chunk extends the bases V_i of the boxes that see it
        std::vector<DBuf<int>> g1keep;
        const SparseSub g1sp = sparse_g1(hq, g, lev, g1keep);
        // equal chunks of <= kb columns (multiple of 8) instead of kb-wide chunks plus a thin tail
        // (sharded: every rank owns a 1/NP slice of each chunk, so chunks are NP times wider)
        // (capped so that the chunk and its gather buffer stay within 16 GB)
        const int kbp = std::max(kb, std::min(kb * NP, (int)std::min<long long>(1 << 20, (16ll << 30) / (16ll * n))));
        const int nch = (c + kbp - 1) / kbp;
        const int kc = std::min(kbp, ((c + nch - 1) / nch + 7) / 8 * 8);
        const long long slot = (long long)cm.kmax(kc) * n;
        DBuf<double> W(NP > 1 ? (size_t)slot : (size_t)n * kc, s), Y((size_t)n * kc, s);
        DBuf<double> gath(NP > 1 ? (size_t)slot * NP : 0, s);
        for (int c0 = 0; c0 < c; c0 += kc) {
          const int k = std::min(kc, c - c0);
          if (NP == 1) {
            gen_probes(s, W.p, k, n, t.d_perm.p, qmap.p, g, c0, lev, trace_id, seed);
            residual(W.p, Y.p, k, lev, &g1sp);
          } else {
            // this rank's (or every emulated rank's) column slice, then one exchange per chunk
            RSF_PHASE("p.exchange", s);
            for (int r = cm.p0(); r < cm.p1(); ++r) {
              long long lo, hi;
              Comm::slice(k, NP, r, &lo, &hi);
              if (hi == lo) continue;
              gen_probes(s, W.p, (int)(hi - lo), n, t.d_perm.p, qmap.p, g, c0 + (int)lo, lev, trace_id, seed);
              residual(W.p, gath.p + r * slot, (int)(hi - lo), lev, &g1sp);
            }
            cm.exchange(s, gath.p, slot);
            cm.merge(s, gath.p, slot, k, n, Y.p);
          }
          RSF_PHASE("p.basis", s);
          size_t x0 = 0;
          while (x0 < NA) {
            size_t x1 = x0;
            double bytes = 0;
            while (x1 < NA) {
              const PBox& b = bx[act[x1]];
              const double bb = 8.0 * ((double)b.ni * (c + 3.0 * k) + 3.0 * (double)c * k + 2.0 * (double)k * (rb[act[x1]] + k));
              if (x1 > x0 && bytes + bb > budget) break;
              bytes += bb;
              ++x1;
            }
            const size_t B = x1 - x0;
            std::vector<long long> wo(B), c1o(B), pro(B);
            long long wt = 0, c1t = 0, prt = 0;
            for (size_t x = 0; x < B; ++x) {
              const int i = act[x0 + x];
              wo[x] = wt; wt += (long long)c * bx[i].ni;
              c1o[x] = c1t; c1t += (long long)k * rb[i];
              pro[x] = prt; prt += (long long)c * k;
            }
            DBuf<double> Wi(Wc.p ? 1 : wt, s), C1(std::max<long long>(c1t, 1), s), Pr(prt, s);
            DBuf<int> pivr((size_t)k * B, s);
            GemmBatch gp(false, true), gc(false, false), gr(false, true), gpr(false, true);
            std::vector<ColMaxDesc> cm;
            std::vector<CopyProb> pcp;
            std::vector<double*> Wp(B);
            for (size_t x = 0; x < B; ++x) {
              const size_t xa = x0 + x;
              const int i = act[xa];
              const PBox& b = bx[i];
              if (Wc.p) {
                Wp[x] = Wc.p + wco[xa];
              } else {
                // W_i^T (c x n_i): the same Philox entries as box i's rows of its own group's probes
                Wp[x] = Wi.p + wo[x];
                probes_kernel<<<gxx((long long)b.ni * c), NT, 0, s>>>(Wp[x], c, b.ib, b.ib + b.ni, t.d_perm.p,
                                                                    nullptr, 0, 0, lev, trace_id, seed32, c);
                count_launch();
              }
              double* Yi = Y.p + (long long)b.ib * k;
              GemmDesc d = gdesc(c, k, b.ni);              // P_ij(:, chunk) = W_i^T Y_ij(:, chunk)
              d.A = Wp[x]; d.lda = c; d.B = Yi; d.ldb = k; d.C = P.p + po[xa] + (long long)c * c0; d.ldc = c;
              gp.add(d);
              cm.push_back(ColMaxDesc{P.p + po[xa] + (long long)c * c0, c, c, k, ref.p + xa});
              pd.flops += 2.0 * c * (double)k * b.ni;
              if (rb[i] > 0) {                             // Res = (I - V_i V_i^T) Y_ij(:, chunk)
                GemmDesc e = gdesc(k, rb[i], b.ni);
                e.A = Yi; e.lda = k; e.B = Vb[i].p; e.ldb = b.ni; e.C = C1.p + c1o[x]; e.ldc = k;
                gc.add(e);
                GemmDesc f = gdesc(k, b.ni, rb[i]);
                f.A = C1.p + c1o[x]; f.lda = k; f.B = Vb[i].p; f.ldb = b.ni; f.C = Yi; f.ldc = k;
                f.alpha = -1.0; f.beta = 1.0;
                gr.add(f);
                pd.flops += 4.0 * k * (double)rb[i] * b.ni;
                GemmDesc h = gdesc(c, k, rb[i]);           // W_i^T Res = W_i^T Y - A_i C1^T
                h.A = Ab[i].p; h.lda = c; h.B = C1.p + c1o[x]; h.ldb = k; h.C = Pr.p + pro[x]; h.ldc = c;
                h.alpha = -1.0; h.beta = 1.0;
                gpr.add(h);
              }
              pcp.push_back(CopyProb{P.p + po[xa] + (long long)c * c0, c, Pr.p + pro[x], c, c, k, 1.0});
            }
            RSF_LAUNCH_CHECK();
            { RSF_PHASE("b.sketchP", s); gp.run(s); launch_colmax(s, cm); copy_batched(s, pcp); }
            { RSF_PHASE("b.project", s); gc.run(s); gr.run(s); gpr.run(s); }
            PhaseSeq pseq(s);
            pseq.next("b.rrqr");
            std::vector<RRQRProb> rp;
            for (size_t x = 0; x < B; ++x) {
              RRQRProb r{Pr.p + pro[x], c, c, k, pivr.p + (long long)x * k, nullptr, nullptr, 0};
              r.ref_in = ref.p + x0 + x;                   // threshold eps_peel * ||Y_ij|| (the block's scale)
              rp.push_back(r);
            }
            std::vector<int> qq = rrqr_batched(s, rp, o.eps_peel,
                                               seed ^ (0x9E3779B97F4A7C15ull * (unsigned long long)(lev + 64 * (trace_id + 3) + 4096 * c0))).k;
            pseq.next("b.orth");
            // new orthonormal directions Q_i = orth(Res(:, pivr[0:q])), re-orthogonalized against V_i
            long long qt = 0, rt = 0;
            std::vector<long long> qo(B), ro(B);
            for (size_t x = 0; x < B; ++x) {
              const int i = act[x0 + x];
              qq[x] = std::min<int>(qq[x], std::min<int>((int)(cccap[x0 + x] - rb[i]), vmax[i] - rb[i]));
              qo[x] = qt; qt += (long long)bx[i].ni * qq[x];
              ro[x] = rt; rt += (long long)qq[x] * qq[x];
              if (rb[i] + qq[x] > vcap[i]) {   // grow V_i (n_i x r, ld n_i) and A_i (c x r, ld c)
                const int nc = rb[i] + qq[x];
                DBuf<double> nv((size_t)bx[i].ni * nc, s), na((size_t)c * nc, s);
                if (rb[i] > 0) {
                  RSF_CUDA(cudaMemcpyAsync(nv.p, Vb[i].p, (size_t)bx[i].ni * rb[i] * sizeof(double),
                                           cudaMemcpyDeviceToDevice, s));
                  RSF_CUDA(cudaMemcpyAsync(na.p, Ab[i].p, (size_t)c * rb[i] * sizeof(double),
                                           cudaMemcpyDeviceToDevice, s));
                }
                Vb[i] = std::move(nv);
                Ab[i] = std::move(na);
                vcap[i] = nc;
              }
            }
            DBuf<double> Q0(std::max<long long>(qt, 1), s), Ri(std::max<long long>(rt, 1), s);
            // the new directions are formed in place in the free columns of V_i
            std::vector<double*> Qp(B, nullptr);
            for (size_t x = 0; x < B; ++x) {
              const int i = act[x0 + x];
              if (qq[x] > 0) Qp[x] = Vb[i].p + (long long)bx[i].ni * rb[i];
            }
            std::vector<GatherTDesc> gd;
            std::vector<EyeDesc> ed;
            std::vector<TrsmProb> tp;
            long long mx = 0;
            for (size_t x = 0; x < B; ++x) {
              const int i = act[x0 + x];
              if (qq[x] == 0) continue;
              gd.push_back(GatherTDesc{Y.p + (long long)bx[i].ib * k, k, pivr.p + (long long)x * k, Q0.p + qo[x], bx[i].ni, qq[x]});
              ed.push_back(EyeDesc{Ri.p + ro[x], qq[x], qq[x]});
              tp.push_back(TrsmProb{Pr.p + pro[x], c, Ri.p + ro[x], qq[x], qq[x], qq[x]});
              mx = std::max(mx, (long long)bx[i].ni * qq[x]);
            }
            launch_gather_t(s, gd);
            launch_descs(s, ed, mx, eye_kernel);
            trsm_upper_batched(s, tp);                    // R11^-1 of the residual sketch
            GemmBatch g0(false, false);
            std::vector<CQProb> cq;
            for (size_t x = 0; x < B; ++x) {
              const int i = act[x0 + x];
              if (qq[x] == 0) continue;
              GemmDesc d = gdesc(bx[i].ni, qq[x], qq[x]);   // Q0 R11^-1 (well conditioned)
              d.A = Q0.p + qo[x]; d.lda = bx[i].ni; d.B = Ri.p + ro[x]; d.ldb = qq[x]; d.C = Qp[x]; d.ldc = bx[i].ni;
              g0.add(d);
              cq.push_back(CQProb{Qp[x], bx[i].ni, qq[x]});
            }
            g0.run(s);
            Q0.release();
            {
              GemmBatch gh(true, false), gq(false, false);
              long long ht = 0;
              std::vector<long long> hoff(B);
              for (size_t x = 0; x < B; ++x) { hoff[x] = ht; ht += (long long)rb[act[x0 + x]] * qq[x]; }
              DBuf<double> H(std::max<long long>(ht, 1), s);
              for (size_t x = 0; x < B; ++x) {
                const int i = act[x0 + x];
                if (qq[x] == 0 || rb[i] == 0) continue;
                GemmDesc d = gdesc(rb[i], qq[x], bx[i].ni);  // H = V^T Q
                d.A = Vb[i].p; d.lda = bx[i].ni; d.B = Qp[x]; d.ldb = bx[i].ni; d.C = H.p + hoff[x]; d.ldc = rb[i];
                gh.add(d);
                GemmDesc e = gdesc(bx[i].ni, qq[x], rb[i]);  // Q -= V H
                e.A = Vb[i].p; e.lda = bx[i].ni; e.B = H.p + hoff[x]; e.ldb = rb[i]; e.C = Qp[x]; e.ldc = bx[i].ni;
                e.alpha = -1.0; e.beta = 1.0;
                gq.add(e);
              }
              if (!gh.empty()) { gh.run(s); gq.run(s); }
              cholqr2_batched(s, cq, lev, &pd.flops, dfail.p);   // right factors keep Q orthogonal to V_i
            }
            // C_ij'(chunk, :) = Y_ij(:, chunk)^T [V_i, Q_i] = [C1, Res^T Q_i]; A_i <- [A_i, W_i^T Q_i]
            // (V_i <- [V_i, Q_i] happened in place)
            pseq.next("b.grow");
            GemmBatch gcq(false, false), gan(false, false);
            std::vector<CopyProb> cc1;
            for (size_t x = 0; x < B; ++x) {
              const size_t xa = x0 + x;
              const int i = act[xa];
              if (rb[i] > 0) cc1.push_back(CopyProb{C1.p + c1o[x], k, CC.p + cco[xa] + c0, c, k, rb[i], 1.0});
              if (qq[x] == 0) continue;
              GemmDesc d = gdesc(k, qq[x], bx[i].ni);
              d.A = Y.p + (long long)bx[i].ib * k; d.lda = k; d.B = Qp[x]; d.ldb = bx[i].ni;
              d.C = CC.p + cco[xa] + c0 + (long long)c * rb[i]; d.ldc = c;
              gcq.add(d);
              GemmDesc e = gdesc(c, qq[x], bx[i].ni);
              e.A = Wp[x]; e.lda = c; e.B = Qp[x]; e.ldb = bx[i].ni;
              e.C = Ab[i].p + (long long)c * rb[i]; e.ldc = c;
              gan.add(e);
              pd.flops += 4.0 * c * (double)qq[x] * bx[i].ni;
            }
            copy_batched(s, cc1);
            gcq.run(s);
            gan.run(s);
            for (size_t x = 0; x < B; ++x) rb[act[x0 + x]] += qq[x];
            x0 = x1;
          }
        }
        W.release();
        Y.release();
        gath.release();
        // eps_peel-rank of every sibling block from its Gaussian sketch P_ij (R-N); adaptivity (R-M)
        DBuf<int> piv((size_t)c * NA, s);
        std::vector<int> kk(NA, 0);
        // R11 of every box's pivoted QR (k x k, ld k), kept for the pair cores; the c x c copies the
        // RRQR works on exist one budget-sized batch of boxes at a time (one batch -- the whole
        // group -- unless the copies exceed the budget: at level 6 of config 4 they were 22 GB)
        std::vector<DBuf<double>> r11buf;
        std::vector<const double*> r11p(NA, nullptr);
        std::vector<int> r11ld(NA, 1);
        {
          RSF_PHASE("p.sketch_rank", s);
          size_t y0 = 0;
          while (y0 < NA) {
            size_t y1 = y0;
            while (y1 < NA && (y1 == y0 || 8.0 * (po[y1] + (long long)c * c - po[y0]) <= budget)) ++y1;
            const long long pb = (long long)(y1 - y0) * c * c;
            DBuf<double> Pc(pb, s);
            RSF_CUDA(cudaMemcpyAsync(Pc.p, P.p + po[y0], pb * sizeof(double), cudaMemcpyDeviceToDevice, s));
            std::vector<RRQRProb> rp;
            for (size_t x = y0; x < y1; ++x)
              rp.push_back(RRQRProb{Pc.p + (po[x] - po[y0]), c, c, c, piv.p + (long long)x * c, nullptr, nullptr, 0});
            std::vector<int> kb = rrqr_batched(s, rp, o.eps_peel, seed ^ (0xD1B54A32D192ED03ull * (unsigned long long)(lev + 64 * (trace_id + 1)))).k;
            long long rt = 0;
            for (size_t x = y0; x < y1; ++x) { kk[x] = kb[x - y0]; rt += (long long)kk[x] * kk[x]; }
            r11buf.emplace_back(DBuf<double>((size_t)std::max<long long>(rt, 1), s));
            std::vector<CopyProb> cr;
            long long ro = 0;
            for (size_t x = y0; x < y1; ++x) {
              r11p[x] = r11buf.back().p + ro;
              r11ld[x] = std::max(1, kk[x]);
              if (kk[x] > 0) cr.push_back(CopyProb{Pc.p + (po[x] - po[y0]), c, r11buf.back().p + ro, kk[x], kk[x], kk[x], 1.0});
              ro += (long long)kk[x] * kk[x];
            }
            copy_batched(s, cr);
            y0 = y1;
          }
        }
        for (size_t x = 0; x < NA; ++x) mr = std::max(mr, kk[x]);
        if (mr > c - o.oversample && c < cmax) { fail = true; break; }
        lev_ranks.insert(lev_ranks.end(), kk.begin(), kk.end());
        // per-pair basis Z_ij = orth(C_ij(:, piv[0:k])) in the coordinates of V_i
        // (U_ij = V_i Z_ij = orth(Y_ij), R-N) and the left core factor
        //   X_ij = W_i^T U_ij,  Lm_ij = X_ij^+ (W_i^T Y_ij)       (Eq. lowrankapprox)
        RSF_PHASE("p.pair_core", s);
        size_t x0 = 0;
        while (x0 < NA) {
          size_t x1 = x0;
          double bytes = 0;
          while (x1 < NA) {
            const double bb = 8.0 * (3.0 * rb[act[x1]] * (double)c + 6.0 * (double)c * c);
            if (x1 > x0 && bytes + bb > budget) break;
            bytes += bb;
            ++x1;
          }
          const size_t B = x1 - x0;
          long long zt = 0;
          std::vector<long long> zo(B), xo(B), lo(B), go(B);
          for (size_t x = 0; x < B; ++x) {
            const size_t xa = x0 + x;
            const int i = act[xa];
            kk[xa] = std::min(kk[xa], rb[i]);
            const long long k = kk[xa];
            zo[x] = zt; zt += (long long)rb[i] * k;
            xo[x] = zt; zt += (long long)c * k;
            lo[x] = zt; zt += k * c;
            go[x] = zt; zt += k * k;
          }
          // persistent blocks [Z | X | Lm | Gi] of every act box in the arena of its own group
          std::vector<double*> ga(B, nullptr);
          std::vector<int> gai(B, -1);
          {
            std::vector<long long> gsz(NGRP, 0), gb(B, 0);
            for (size_t x = 0; x < B; ++x) {
              const int q = grp[act[x0 + x]];
              const long long k = kk[x0 + x];
              gb[x] = gsz[q];
              gsz[q] += (long long)rb[act[x0 + x]] * k + 2ll * c * k + k * k;
            }
            std::vector<int> gidx(NGRP, -1);
            for (int q = 0; q < NGRP; ++q)
              if (gsz[q] > 0) {
                gidx[q] = (int)arenas.size();
                arenas.emplace_back(DBuf<double>((size_t)gsz[q], s));
                arena_uses.push_back(0);
                pair_bytes += 8.0 * gsz[q];
              }
            pair_peak = std::max(pair_peak, pair_bytes);
            for (size_t x = 0; x < B; ++x) {
              const int q = grp[act[x0 + x]];
              if (gidx[q] < 0) continue;
              gai[x] = gidx[q];
              ga[x] = arenas[gidx[q]].p + gb[x];
            }
          }
          auto AP = [&](size_t x, long long off) { return ga[x] + (off - zo[x]); };
          DBuf<double> Z0(std::max<long long>(zt, 1), s), Ri2(std::max<long long>(zt, 1), s), T1(std::max<long long>(zt, 1), s);
          std::vector<GatherTDesc> gz;
          std::vector<EyeDesc> ez;
          std::vector<TrsmProb> tz;
          long long mz = 0;
          for (size_t x = 0; x < B; ++x) {
            const size_t xa = x0 + x;
            const int i = act[xa];
            const int k = kk[xa];
            if (k == 0) continue;
            gz.push_back(GatherTDesc{CC.p + cco[xa], c, piv.p + (long long)xa * c, Z0.p + zo[x], rb[i], k});
            ez.push_back(EyeDesc{Ri2.p + go[x], k, k});
            tz.push_back(TrsmProb{r11p[xa], r11ld[xa], Ri2.p + go[x], k, k, k});
            mz = std::max(mz, (long long)rb[i] * k);
          }
          PhaseSeq cseq(s);
          cseq.next("c.z");
          launch_gather_t(s, gz);
          launch_descs(s, ez, mz, eye_kernel);
          trsm_upper_batched(s, tz);
          GemmBatch gz1(false, false);
          std::vector<CQProb> cz;
          for (size_t x = 0; x < B; ++x) {
            const size_t xa = x0 + x;
            const int i = act[xa];
            const int k = kk[xa];
            if (k == 0) continue;
            GemmDesc d = gdesc(rb[i], k, k);
            d.A = Z0.p + zo[x]; d.lda = rb[i]; d.B = Ri2.p + go[x]; d.ldb = k; d.C = AP(x, zo[x]); d.ldc = rb[i];
            gz1.add(d);
            cz.push_back(CQProb{AP(x, zo[x]), rb[i], k});
          }
          gz1.run(s);
          cholqr2_batched(s, cz, lev, &pd.flops, dfail.p);
          GemmBatch gx(false, false), gg(true, false), gt1(true, false), gt2(false, false), gt3(true, false);
          std::vector<PotrfProb> pp;
          for (size_t x = 0; x < B; ++x) {
            const size_t xa = x0 + x;
            const int i = act[xa];
            const int k = kk[xa];
            if (k == 0) continue;
            GemmDesc a = gdesc(c, k, rb[i]);               // X = A_i Z
            a.A = Ab[i].p; a.lda = c; a.B = AP(x, zo[x]); a.ldb = rb[i]; a.C = AP(x, xo[x]); a.ldc = c;
            gx.add(a);
            GemmDesc d = gdesc(k, k, c);                   // X^T X
            d.A = AP(x, xo[x]); d.lda = c; d.B = AP(x, xo[x]); d.ldb = c; d.C = T1.p + go[x]; d.ldc = k;
            gg.add(d);
            pp.push_back(PotrfProb{T1.p + go[x], k, k, AP(x, go[x]), k});
            GemmDesc e = gdesc(k, c, c);                   // X^T P
            e.A = AP(x, xo[x]); e.lda = c; e.B = P.p + po[xa]; e.ldb = c; e.C = Z0.p + lo[x]; e.ldc = k;
            gt1.add(e);
            GemmDesc f = gdesc(k, c, k);                   // L^-1 (X^T P)
            f.A = AP(x, go[x]); f.lda = k; f.B = Z0.p + lo[x]; f.ldb = k; f.C = Ri2.p + lo[x]; f.ldc = k;
            gt2.add(f);
            GemmDesc h = gdesc(k, c, k);                   // Lm = L^-T L^-1 X^T P
            h.A = AP(x, go[x]); h.lda = k; h.B = Ri2.p + lo[x]; h.ldb = k; h.C = AP(x, lo[x]); h.ldc = k;
            gt3.add(h);
            pd.flops += 2.0 * c * (double)k * rb[i] + 4.0 * k * (double)c * c;
          }
          cseq.next("c.xlm");
          gx.run(s);
          gg.run(s);
          {
            DBuf<double> ls(std::max<size_t>(pp.size(), 1), s);
            DBuf<int> inf(std::max<size_t>(pp.size(), 1), s);
            potrf_batched(s, pp, ls.p, inf.p);
            flag_infos(s, inf.p, (int)pp.size(), dfail.p);
          }
          gt1.run(s); gt2.run(s); gt3.run(s);
          for (size_t x = 0; x < B; ++x) {
            const size_t xa = x0 + x;
            const int i = act[xa], j = partner[xa];
            PairData& q = pdat[pslot(i, j)];
            q.k = kk[xa]; q.rz = rb[i];
            if (gai[x] < 0) continue;   // k = 0: no block
            q.Z = AP(x, zo[x]); q.X = AP(x, xo[x]); q.Lm = AP(x, lo[x]); q.Gi = AP(x, go[x]);
            q.arena = gai[x];
            ++arena_uses[gai[x]];
          }
          x0 = x1;
        }
        // cores of the pairs completed by this group: (i, j in g) whose other side (j, i) came with
        // the group of i, sketched earlier
        std::vector<std::pair<int, int>> done;
        for (size_t x = 0; x < NA; ++x)
          if (gdone[grp[act[x]]]) done.emplace_back(std::min(act[x], partner[x]), std::max(act[x], partner[x]));
        compute_cores(done);
        }   // subsets
        if (fail) break;
        gdone[g] = 1;
      }
      if (!fail) break;
      ++restarts;
      int nc = (mr >= c - 1) ? (int)std::ceil(1.4 * c) : std::max(c + 8, (int)std::ceil(1.1 * mr) + o.oversample);
      c = std::max(std::min((nc + 7) / 8 * 8, cmax), c + 8);
    }
    pd.cols[lev] = c;
    pd.rank_max[lev] = mr;
    if (!lev_ranks.empty()) {
      std::sort(lev_ranks.begin(), lev_ranks.end());
      pd.rank_min[lev] = lev_ranks.front();
      pd.rank_med[lev] = lev_ranks[lev_ranks.size() / 2];
    }
    prev_rank = mr;
    for (auto& v : Ab) v.release();

    // ---- cores: M_ij = Lm_ij (X_ji^T)^+ = Lm_ij X_ji (X_ji^T X_ji)^-1, B_ij = Z_ij M_ij Z_ji^T,
    //      B_ji = B_ij^T; Brow_i = [B_ij]_{j in family(i)} (r_i x R_fam, zero self block)
    PeelLevel& PL = peeled[lev];
    std::vector<long long> fo(nb), bo(nb);     // column offset of box b inside its family row; Brow offsets
    long long brt = 0;
    // column offset of box x inside b's row of cores: sum of r_y over y in rowset[b], y < x
    auto fo_of = [&](int b, int x) -> long long {
      long long off = 0;
      for (int y : rowset[b]) { if (y >= x) break; off += rb[y]; }
      return off;
    };
    for (int b = 0; b < nb; ++b) {
      long long off = 0, tot = 0;
      for (int x : rowset[b]) { if (x < b) off += rb[x]; tot += rb[x]; }
      fo[b] = off;
      bo[b] = brt; brt += (long long)rb[b] * tot;
    }
    PL.Brow.alloc(std::max<long long>(brt, 1), s);
    PL.Brow.zero();
    {   // the finished B_ij blocks into their places in Brow (zero rows/columns past rz)
      std::vector<CopyProb> cp;
      for (const CBlock& q : cblocks)
        cp.push_back(CopyProb{q.p, q.ri, PL.Brow.p + bo[q.i] + (long long)rb[q.i] * fo_of(q.i, q.j), rb[q.i],
                              q.ri, q.rj, 1.0});
      copy_batched(s, cp);
      cblocks.clear();
      cbufs.clear();
    }
    arenas.clear();
    arena_uses.clear();
    for (auto& q : pdat) q = PairData{};
    if (dfail.to_host(1)[0])
      throw Error(ST_ENUMERIC, "peeling: Cholesky of a sketch basis or core Gram matrix failed at level " +
                                   std::to_string(lev));

    // ---- subtraction batches of G^(lev)
    PL.V.clear();
    PL.V.resize(nb);
    {   // exactly sized buffers move over; reserved ones are copied to their size box by box
      std::vector<CopyProb> cpv;
      for (int b = 0; b < nb; ++b) {
        if (rb[b] == 0) continue;
        if (vcap[b] == rb[b]) { PL.V[b] = std::move(Vb[b]); continue; }
        PL.V[b].alloc((size_t)bx[b].ni * rb[b], s);
        cpv.push_back(CopyProb{Vb[b].p, bx[b].ni, PL.V[b].p, bx[b].ni, bx[b].ni, rb[b], 1.0});
      }
      copy_batched(s, cpv);
      for (auto& v : Vb) v.release();
    }
    double vbytes = 0;
    for (auto& v : PL.V) vbytes += 8.0 * v.n;
    double browbytes = 8.0 * PL.Brow.n;
    if (o.peel_f32) {   // FP32 storage of G^(lev), box by box
      PL.f32 = true;
      PL.vfo.assign(nb, 0);
      size_t tot = 0;
      for (int b = 0; b < nb; ++b) { PL.vfo[b] = tot; tot += (PL.V[b].n + 3) & ~(size_t)3; }   // 16-byte aligned
      PL.browf_off = tot;
      tot += PL.Brow.n;
      PL.store.alloc(std::max<size_t>(tot, 1), s);
      for (int b = 0; b < nb; ++b) {
        if (!PL.V[b].p) continue;
        d2f_kernel<<<gxx((long long)PL.V[b].n), NT, 0, s>>>(PL.V[b].p, PL.store.p + PL.vfo[b], (long long)PL.V[b].n);
        count_launch();
        PL.V[b].release();
      }
      d2f_kernel<<<gxx((long long)PL.Brow.n), NT, 0, s>>>(PL.Brow.p, PL.store.p + PL.browf_off, (long long)PL.Brow.n);
      count_launch();
      RSF_LAUNCH_CHECK();
      PL.Brow.release();
      vbytes *= 0.5;
      browbytes *= 0.5;
    }
    pd.stored_bytes += vbytes + browbytes;
    PL.g1.reset(false, false);
    PL.g2.reset(false, true);
    PL.g3.reset(false, true);
    long long tc = 0;
    std::vector<long long> toff(nb), soff(nb);
    for (int b = 0; b < nb; ++b) { toff[b] = tc; tc += rb[b]; }
    for (int b = 0; b < nb; ++b) { soff[b] = tc; tc += rb[b]; }
    // strong: the T' columns of IL(b) are not contiguous -> a K-gather list per box
    std::vector<long long> moff(nb, 0);
    if (strong) {
      std::vector<int> hm;
      for (int b = 0; b < nb; ++b) {
        moff[b] = (long long)hm.size();
        for (int x : rowset[b])
          for (int q = 0; q < rb[x]; ++q) hm.push_back((int)(toff[x] + q));
      }
      PL.mapk = up(hm, s);
    }
    for (int b = 0; b < nb; ++b) {
      if (rb[b] == 0) continue;
      long long tot = 0;
      for (int x : rowset[b]) tot += rb[x];
      GemmDesc a = gdesc(-1, rb[b], bx[b].ni);            // T'_b = X'(:, I_b) V_b
      a.selA = 1; a.offA = bx[b].ib; a.B = (const double*)PL.vptr(b); a.bf32 = PL.f32; a.ldb = bx[b].ni;
      a.selC = 2; a.offC = toff[b];
      PL.g1.add(a);
      PL.ib.push_back(bx[b].ib); PL.ni.push_back(bx[b].ni); PL.r.push_back(rb[b]); PL.bidx.push_back(b);
      PL.toff.push_back(toff[b]); PL.soff.push_back(soff[b]);
      GemmDesc d = gdesc(-1, rb[b], (int)tot);            // S'_b = T'_row Brow_b^T
      d.selA = 2; d.offA = strong ? 0 : toff[bx[b].fam0]; d.ldb = rb[b];
      if (PL.f32) { d.B = (const double*)PL.browf(); d.offB = bo[b]; d.bf32 = 1; } else d.B = PL.Brow.p + bo[b];
      d.selC = 2; d.offC = soff[b];
      if (strong) d.mapA = PL.mapk.p + moff[b];
      if (tot == 0) continue;                              // (strong: no partner has a basis)
      PL.g2.add(d);
      GemmDesc e = gdesc(-1, bx[b].ni, rb[b]);            // Y'(:, I_b) -= S'_b V_b^T
      e.selA = 2; e.offA = soff[b]; e.B = (const double*)PL.vptr(b); e.bf32 = PL.f32; e.ldb = bx[b].ni;
      e.selC = 1; e.offC = bx[b].ib;
      e.alpha = -1.0; e.beta = 1.0;
      PL.g3.add(e);
    }
    PL.tcols = tc;
    max_tcols = std::max(max_tcols, tc);
    for (GemmBatch* g : {&PL.g1, &PL.g2, &PL.g3})
      if (!g->empty()) g->finalize(s);
    // memory-saving mode: the per-box blocks of this level (<= 64 MB, power-of-two bins) go back to
    // the stream-ordered pool instead of waiting in the bin cache for sizes the next level never asks
    if (o.peel_f32) { dev_cache_trim_bins(s); pool_trim(); }
    if (verbose) {
      RSF_CUDA(cudaStreamSynchronize(s));
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      long long rsum = 0;
      int rmax = 0;
      for (int b = 0; b < nb; ++b) { rsum += rb[b]; rmax = std::max(rmax, rb[b]); }
      fprintf(stderr, "[peel tr%d] level %d boxes %d pairs %d cols %d rank_max %d restarts %d basis sum %lld max %d "
                      "V %.2f GB Brow %.2f GB dev_used %.2f GB t %.2f s\n",
              trace_id, lev, nb, npairs, c, mr, restarts, rsum, rmax, 1e-9 * vbytes, 1e-9 * browbytes,
              1e-9 * (tot - fr), now_s() - t0);
      {
        cudaMemPool_t pool;
        int dev = 0;
        cudaGetDevice(&dev);
        unsigned long long res = 0, used = 0;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
          cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res);
          cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
        }
        fprintf(stderr, "    memory: pool reserved %.2f GB used %.2f GB, bin caches %.2f GB, pair data of the level (peak) %.2f GB\n",
                1e-9 * res, 1e-9 * used, 1e-9 * dev_cache_bytes(), 1e-9 * pair_peak);
      }
      if (verbose > 1 && !PL.f32) {
        DBuf<unsigned long long> cnt(4, s);
        RSF_CUDA(cudaMemsetAsync(cnt.p, 0, 4 * sizeof(unsigned long long), s));
        long long rows = 0;
        for (int b = 0; b < nb; ++b)
          if (rb[b] > 0) {
            rownorm_hist_kernel<<<gxx(bx[b].ni), NT, 0, s>>>(PL.V[b].p, bx[b].ni, rb[b], cnt.p);
            rows += bx[b].ni;
          }
        auto h = cnt.to_host(4);
        fprintf(stderr, "    V rows %lld: row norm < 1e-12: %llu, < 1e-10: %llu, < 1e-8: %llu, < 1e-6: %llu\n", rows,
                h[0], h[1], h[2], h[3]);
      }
    }
  }

  // ---- extraction
  std::vector<int> lb(n, 0);
  int nL = 0;
  for (int nd = 0; nd < (int)t.lev.size(); ++nd) {
    if (!t.is_leaf(nd)) continue;
    for (int x = t.begin[nd]; x < t.end[nd]; ++x) lb[x] = t.begin[nd];
    nL = std::max(nL, t.end[nd] - t.begin[nd]);
  }
  DBuf<int> dlb = up(lb, s);
  RSF_PHASE("p.extract", s);
  double tr = 0.0, tra = 0.0;
  const int GB = 256;
  // (sharded: the nL extraction columns are split over the parts; partial leaf traces are
  // summed over the ranks in rank order)
  // (strong: the leaf near field remains in the residual, so the identity probes go to the 9
  // leaf classes (ix mod 3, iy mod 3) in turn -- one box per class in every 3 x 3 neighbourhood)
  double trp[2] = {0.0, 0.0};
  DBuf<int> dcls;
  if (strong) {
    std::vector<int> hc(n, 0);
    for (int nd : t.levels[L])
      for (int x = t.begin[nd]; x < t.end[nd]; ++x) hc[x] = (t.ix[nd] % 3) * 3 + (t.iy[nd] % 3);
    dcls = up(hc, s);
  }
  for (int kap = 0; kap < (strong ? 9 : 1); ++kap)
    for (int r = cm.p0(); r < cm.p1(); ++r) {
      long long lo, hi;
      Comm::slice(nL, NP, r, &lo, &hi);
      for (int e0 = (int)lo; e0 < (int)hi; e0 += kb) {
        const int k = std::min<int>(kb, (int)hi - e0);
        DBuf<double> E((size_t)n * k, s), H((size_t)n * k, s), part(GB, s), parta(GB, s);
        extract_probe_kernel<<<gxx((long long)n * k), NT, 0, s>>>(E.p, k, n, dlb.p, e0, dcls.p, kap);
        count_launch();
        RSF_LAUNCH_CHECK();
        residual(E.p, H.p, k, L + 1, nullptr);
        extract_diag_kernel<<<GB, NT, 0, s>>>(H.p, k, n, dlb.p, e0, part.p, parta.p, dcls.p, kap);
        count_launch();
        RSF_LAUNCH_CHECK();
        auto hp = part.to_host(GB), ha = parta.to_host(GB);
        for (int i = 0; i < GB; ++i) { trp[0] += hp[i]; trp[1] += ha[i]; }
      }
    }
  cm.allsum(s, trp, 2);
  tr = trp[0];
  tra = trp[1];
  pd.nL = nL;
  pd.cancellation = tr != 0.0 ? tra / std::fabs(tr) : INFINITY;
  pd.applies = G.columns;
  RSF_CUDA(cudaStreamSynchronize(s));
  pd.seconds = now_s() - t0;
  if (diag) *diag = pd;
  return tr;
}

// Hutchinson estimate of Tr(F^-1 F_i) (Fi != null) or Tr(F^-1): (1/q) sum_p u_p^T F^-1 F_i u_p
// with Rademacher u_p; u^T F^-1 F_i u = (F^-1 u)^T (F_i u), one solve + one apply
// per probe.  Deterministic (fixed-order reductions).
void hutch(const Fact& F, const Fact* Fi, long long q, unsigned long long seed, double* mean, double* se) {
  RSF_REQUIRE(q >= 1, ST_EINVAL, "hutch: nprobe < 1");
  cudaStream_t s = op_stream(F);
  const Tree& t = *F.tree;
  const int n = t.n, kb = 512, GB = 256;
  DBuf<double> U((size_t)n * kb, s), A((size_t)n * kb, s), B, C, tmp((size_t)std::max<long long>(F.tmp_cols, 1) * kb, s);
  if (Fi) { B.alloc((size_t)n * kb, s); C.alloc((size_t)n * kb, s); }
  DBuf<double> part((size_t)GB * kb, s);
  std::vector<double> vals;
  vals.reserve(q);
  for (long long p0 = 0; p0 < q; p0 += kb) {
    const int k = (int)std::min<long long>(kb, q - p0);
    const long long nn = (long long)n * k;
    rademacher_kernel<<<gxx(nn), NT, 0, s>>>(U.p, k, n, t.d_perm.p, (int)p0, (unsigned)(seed & 0xffffffffull));
    count_launch();
    RSF_CUDA(cudaMemcpyAsync(A.p, U.p, nn * sizeof(double), cudaMemcpyDeviceToDevice, s));
    solve_internal(F, A.p, k, tmp.p);                                   // A = F^-1 U
    const double* other = U.p;
    if (Fi) {
      RSF_CUDA(cudaMemcpyAsync(B.p, U.p, nn * sizeof(double), cudaMemcpyDeviceToDevice, s));
      apply_only_internal(*Fi, B.p, C.p, k);                            // C = F_i U
      other = C.p;
    }
    rowdot_kernel<<<GB, 256, 0, s>>>(A.p, other, k, n, part.p);
    count_launch();
    RSF_LAUNCH_CHECK();
    const std::vector<double> h = part.to_host((size_t)GB * k);
    for (int j = 0; j < k; ++j) {
      double v = 0.0;
      for (int b = 0; b < GB; ++b) v += h[(size_t)b * k + j];
      vals.push_back(v);
    }
  }
  double m = 0.0;
  for (double v : vals) m += v;
  m /= (double)vals.size();
  double var = 0.0;
  for (double v : vals) var += (v - m) * (v - m);
  *mean = m;
  *se = vals.size() > 1 ? std::sqrt(var / (double)(vals.size() - 1) / (double)vals.size()) : INFINITY;
}

// conditional mean E[z' | z] = Sigma_12 Sigma_22^-1 z at m new points (Remark conditional,
// P:680-690): u = F^-1 z through the factor, then the cross-covariance product on the fly
void cond_mean(const Fact& F, const double* z, const double* xyn, long long m, double* out) {
  RSF_REQUIRE(F.which == W_SIGMA, ST_EINVAL, "conditional mean needs a Sigma factor");
  cudaStream_t s = op_stream(F);
  const Tree& t = *F.tree;
  const int n = t.n;
  DBuf<double> u(n, s), tmp((size_t)std::max<long long>(F.tmp_cols, 1), s);
  to_internal(s, t, z, n, 1, u.p);
  solve_internal(F, u.p, 1, tmp.p);
  if (m > 0) {
    const int grid = (int)std::min<long long>((m + NT - 1) / NT, 148 * 8);
    cross_matvec_kernel<<<grid, NT, 0, s>>>(t.xs.p, t.ys.p, u.p, n, xyn, m, F.kp, out);
    count_launch();
    RSF_LAUNCH_CHECK();
  }
}

void fill_peel_diag(const PeelDiag& d, rsf_peel_diag* out) {
  std::memset(out, 0, sizeof(*out));
  out->levels = (int)d.cols.size() - 1;
  for (size_t l = 0; l < d.cols.size() && l < 32; ++l) {
    out->cols[l] = d.cols[l];
    out->rank_max[l] = d.rank_max[l];
    if (l < d.rank_min.size()) { out->rank_min[l] = d.rank_min[l]; out->rank_med[l] = d.rank_med[l]; }
  }
  out->nL = d.nL;
  out->cancellation = d.cancellation;
  out->applies = d.applies;
  out->seconds = d.seconds;
  out->stored_bytes = d.stored_bytes;
}

// ----------------------------------------------------------------- Alg. 1
EvalResult mle_eval(Ctx& ctx, const double* xy, const double* z, int n, const KParams& kp, int p,
                    const int* theta, double eps, int leaf, const Opts& o, bool profile) {
  // memory-saving mode: large blocks via cudaMalloc/cudaFree, from a trimmed pool (
  // measured faster than stream-ordered transients without arenas: 246.5 vs 268.5 s at config 4)
  BigSyncScope big_sync(o.peel_f32 != 0);
  EvalResult R;
  const long long l0 = g_launches;
  const double T0 = now_s();
  cudaStream_t s = ctx.stream;
  KTrace::set_stream(s);
  auto is_dev = [](const void* ptr) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) { cudaGetLastError(); return false; }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
  };
  DBuf<double> xyd, zd;
  const double* dxy = xy;
  const double* dz = z;
  if (!is_dev(xy)) { xyd.alloc(2 * (size_t)n, s); xyd.upload(xy, 2 * (size_t)n); dxy = xyd.p; }
  if (!is_dev(z)) { zd.alloc(n, s); zd.upload(z, n); dz = zd.p; }
  double t = now_s();
  auto tree = build_tree(ctx, dxy, n, leaf, o.max_depth);
  R.t_tree = now_s() - t;
  for (int i = 0; i < p; ++i)
    RSF_REQUIRE(!(profile && theta[i] == W_SIGMA2), ST_EINVAL,
                "profile likelihood: sigma2 is profiled out, not a theta component");

  // Jobs (Alg. 1): the traces Tr(F^-1 F_i) are independent given F and u: one job
  // per general component (compression of Sigma_i, which needs only the tree; then
  // q_i = u^T F_i u and the peeling, which need F and u) plus one job for Tr(F^-1) when sigma^2
  // or the nugget is in theta (reading R-G).  With more than one job they run concurrently,
  // each on its own stream from its own host thread, the compressions alongside the Sigma
  // factor: the latency-bound phases of one job (rank-revealing QR, panels, small batches)
  // overlap the GEMMs of another.  Results do not depend on it.
  std::shared_ptr<Fact> F;
  DBuf<double> u;
  double trinv = NAN, utu = NAN, t_trinv = 0;
  PeelDiag pd_trinv;
  std::vector<double> qv(p, NAN), trv(p, NAN), tcomp(p, 0.0), tsol(p, 0.0), tpl(p, 0.0), ffl(p, 0.0);
  std::promise<void> f_promise;
  std::shared_future<void> f_ready = f_promise.get_future().share();
  cudaEvent_t f_event = nullptr;   // recorded on the main stream once F and u are complete
  std::function<void()> wait_f = [&]() {
    f_ready.get();
    if (f_event && ctx_stream(ctx) != s) RSF_CUDA(cudaStreamWaitEvent(ctx_stream(ctx), f_event, 0));
  };
  // sharded evaluation: the jobs are dealt to G = min(jobs, ranks) rank groups
  // (job j to group j mod G, rank r in group r mod G); a job's communicator holds its group's
  // ranks, which split its probe columns.  Communicators are split from the group's communicator
  // on the calling thread, in job order (the same on every rank).
  auto job_comm = [&](int j) -> const Comm* { return ctx.comm.use_nccl() ? &ctx.job_comms[j] : &ctx.comm; };
  std::vector<std::function<void()>> jobs;
  std::vector<int> job_theta;   // theta index of a general job, -1 for the Tr(F^-1) job
  bool need_trinv = false;
  for (int i = 0; i < p; ++i) {
    const int w = theta[i];
    if (w == W_SIGMA2 || w == W_NUGGET) { need_trinv = true; continue; }
    const int jid = (int)jobs.size();
    job_theta.push_back(i);
    jobs.push_back([&, i, w, jid]() {
      double t1 = now_s();
      auto Fi = factor(ctx, tree, kp, w, eps, o);
      tcomp[i] = now_s() - t1;
      ffl[i] = Fi->diag.flops_id + Fi->diag.flops_elim;
      wait_f();
      cudaStream_t s2 = ctx_stream(ctx);
      t1 = now_s();
      DBuf<double> x(n, s2), y(n, s2);
      RSF_CUDA(cudaMemcpyAsync(x.p, u.p, n * sizeof(double), cudaMemcpyDeviceToDevice, s2));
      apply_only_internal(*Fi, x.p, y.p, 1);
      qv[i] = ddot(s2, u.p, y.p, n);
      tsol[i] = now_s() - t1;
      t1 = now_s();
      trv[i] = peel(*F, Fi.get(), o, i, &R.pd[i], job_comm(jid));
      tpl[i] = now_s() - t1;
    });
  }
  if (need_trinv) {
    const int jid = (int)jobs.size();
    job_theta.push_back(-1);
    jobs.push_back([&, jid]() {
      wait_f();
      const double t1 = now_s();
      trinv = peel(*F, nullptr, o, 100, &pd_trinv, job_comm(jid));
      utu = ddot(ctx_stream(ctx), u.p, u.p, n);
      t_trinv = now_s() - t1;
    });
  }

  const int njobs = (int)jobs.size();
  const int NG = Comm::job_groups(njobs, ctx.comm.world);
  // ranks per group by the jobs' estimated work: a general theta_i job compresses
  // Sigma_i and peels G = (F^-1 F_i + F_i F^-1)/2 (2 solves + 2 applies per probe column), the
  // Tr(F^-1) job peels F^-1 (1 solve per column) -- measured 185 s vs 55 s at config 4
  std::vector<double> gw(NG, 0.0);
  for (int j = 0; j < njobs; ++j) gw[j % NG] += job_theta[j] >= 0 ? 3.0 : 1.0;
  const int my_group = Comm::group_of_rank(gw, ctx.comm.world, ctx.comm.rank);
  auto mine = [&](int j) { return ctx.comm.world == 1 || j % NG == my_group; };
  if (ctx.comm.use_nccl() && ctx.job_comms_njobs != njobs) {
    for (auto& jc : ctx.job_comms)
      if (jc.owned) nccl_destroy(jc.nccl);
    ctx.job_comms.assign(njobs, Comm{});
    for (int j = 0; j < njobs; ++j) {
      void* c = nccl_split_color(ctx.comm.nccl, mine(j) ? j % NG : -1, ctx.comm.rank);
      if (!c) continue;
      Comm jc;
      jc.nccl = c;
      jc.owned = true;
      jc.force = ctx.comm.force;
      nccl_query(c, &jc.rank, &jc.world);
      ctx.job_comms[j] = jc;
    }
    ctx.job_comms_njobs = njobs;
  }
  {   // this rank runs the jobs of its group only
    std::vector<std::function<void()>> run;
    for (int j = 0; j < njobs; ++j)
      if (mine(j)) run.push_back(jobs[j]);
    jobs.swap(run);
  }

  // F ~ Sigma (solve-only), u = F^-1 z (k = 1), q0 = z^T u; profile terms (Eq. prof)
  double Qp = 0.0;
  auto main_part = [&]() {
    double t1 = now_s();
    F = factor(ctx, tree, kp, W_SIGMA, eps, o, /*solve_only=*/true);
    R.t_factor = now_s() - t1;
    R.fdiag = F->diag;
    R.L = tree->L;
    R.n0 = F->n0;
    R.flops_factor += F->diag.flops_id + F->diag.flops_elim + F->diag.flops_top;
    R.logdet = F->logdet;
    t1 = now_s();
    DBuf<double> zt(n, s), tmp((size_t)std::max<long long>(F->tmp_cols, 1), s);
    u.alloc(n, s);
    to_internal(s, *tree, dz, n, 1, zt.p);
    RSF_CUDA(cudaMemcpyAsync(u.p, zt.p, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    solve_internal(*F, u.p, 1, tmp.p);
    R.quad = ddot(s, zt.p, u.p, n);
    R.ell = -0.5 * R.quad - 0.5 * R.logdet - 0.5 * n * std::log(2.0 * M_PI);
    if (profile) {
      // profile likelihood (Eq. prof): z ~ N(mu 1, s2 Sigma) with mu, s2 profiled out,
      //   Q = z^T (Sigma + 1 1^T)^-1 z = z^T u - (1^T u)^2 / (1 + 1^T w),  w = F^-1 1 (Sherman-Morrison)
      //   l~ = -1/2 log|Sigma| - n/2 log Q + n/2 (log n - 1 - log 2 pi)          (reading R-Prof)
      //   v = (Sigma + 1 1^T)^-1 z = u - w (1^T u) / (1 + 1^T w)   (held in u from here on)
      DBuf<double> one(n, s), wv(n, s);
      fill_kernel<<<gxx(n), NT, 0, s>>>(one.p, 1.0, n);
      count_launch();
      RSF_CUDA(cudaMemcpyAsync(wv.p, one.p, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
      solve_internal(*F, wv.p, 1, tmp.p);
      const double a = ddot(s, one.p, wv.p, n), b = ddot(s, one.p, u.p, n);
      Qp = R.quad - b * b / (1.0 + a);
      R.ell = -0.5 * R.logdet - 0.5 * n * std::log(Qp) + 0.5 * n * (std::log((double)n) - 1.0 - std::log(2.0 * M_PI));
      axpby_kernel<<<gxx(n), NT, 0, s>>>(u.p, wv.p, -b / (1.0 + a), 1.0, n);   // u <- u - w b/(1+a)
      count_launch();
      RSF_LAUNCH_CHECK();
      R.quad = Qp;
    }
    R.t_solve = now_s() - t1;
  };

  static const bool par_on = !(getenv("RSF_PAR_TRACES") && getenv("RSF_PAR_TRACES")[0] == '0');
  R.jobs = njobs;
  R.groups = NG;
  double tj0 = 0.0;
  // memory plan: a shape that ran out of memory with its jobs side by side runs them serially
  bool planned_serial = false;
  for (auto& sh : ctx.serial_shapes) planned_serial = planned_serial || (sh.first == n && sh.second == njobs);
  // (the profiler and the launch trace synchronise one stream at a time, and the per-site GEMM
  // log would time launches that share the GPU with another job's: serial then)
  // (opts.peel_f32 is the memory-saving mode: the trace jobs also run one after the other, so one
  // peeled representation is resident at a time -- DESIGN.md §7g)
  if (!par_on || jobs.size() < 2 || Prof::enabled() || KTrace::on() || GemmLog::on() || planned_serial || o.peel_f32) {
    main_part();
    f_promise.set_value();
    tj0 = now_s();
    for (auto& j : jobs) j();
  } else {
    R.concurrent = 1;
    tj0 = now_s();
    while (ctx.aux.size() < jobs.size()) {
      cudaStream_t a2;
      RSF_CUDA(cudaStreamCreateWithFlags(&a2, cudaStreamNonBlocking));
      ctx.aux.push_back(a2);
    }
    cudaEvent_t t_event;
    RSF_CUDA(cudaEventCreateWithFlags(&t_event, cudaEventDisableTiming));
    RSF_CUDA(cudaEventCreateWithFlags(&f_event, cudaEventDisableTiming));
    RSF_CUDA(cudaEventRecord(t_event, s));   // the tree is complete on the main stream
    int dev = 0;
    RSF_CUDA(cudaGetDevice(&dev));
    std::vector<std::exception_ptr> err(jobs.size());
    std::vector<long long> nl(jobs.size(), 0);
    std::vector<std::thread> th;
    for (size_t j = 0; j < jobs.size(); ++j)
      th.emplace_back([&, j]() {
        const long long l0j = g_launches;
        try {
          RSF_CUDA(cudaSetDevice(dev));
          StreamScope scope(ctx.aux[j]);
          RSF_CUDA(cudaStreamWaitEvent(ctx.aux[j], t_event, 0));
          // test hook: the last job reports out-of-memory (exercises the serial fallback)
          static const bool test_oom = getenv("RSF_TEST_PAR_OOM") && getenv("RSF_TEST_PAR_OOM")[0] == '1';
          if (test_oom && j + 1 == jobs.size()) throw Error(ST_ENOMEM, "RSF_TEST_PAR_OOM");
          jobs[j]();
          RSF_CUDA(cudaStreamSynchronize(ctx.aux[j]));
        } catch (...) {
          err[j] = std::current_exception();
        }
        nl[j] = g_launches - l0j;
      });
    std::exception_ptr main_err;
    try {
      main_part();
      RSF_CUDA(cudaEventRecord(f_event, s));
      f_promise.set_value();
    } catch (...) {
      main_err = std::current_exception();
      f_promise.set_exception(main_err);   // releases the jobs waiting for F
    }
    for (auto& x : th) x.join();
    cudaEventDestroy(t_event);
    cudaEventDestroy(f_event);
    f_event = nullptr;
    for (long long v : nl) g_launches += v;
    // Out of memory with the jobs side by side: release what the jobs' streams cached and
    // run everything again in the serial order (peak memory of one job at a time)
    auto is_oom = [](const std::exception_ptr& e) {
      if (!e) return false;
      try { std::rethrow_exception(e); } catch (const Error& x) { return x.code == ST_ENOMEM; } catch (...) {}
      return false;
    };
    bool oom = is_oom(main_err);
    for (auto& e : err) oom = oom || is_oom(e);
    // (on a rank group a one-rank rerun would leave its peers' collectives unmatched: report)
    if (oom && ctx.comm.world == 1) {
      for (size_t j = 0; j < jobs.size(); ++j) {
        cudaStreamSynchronize(ctx.aux[j]);
        dev_cache_trim(ctx.aux[j]);
      }
      cudaGetLastError();
      F.reset();
      u.release();
      wait_f = []() {};
      R.flops_factor = 0;
      R.serial_fallback = 1;
      ctx.serial_shapes.emplace_back((long long)n, njobs);
      main_part();
      for (auto& j : jobs) j();
    } else {
      if (main_err) std::rethrow_exception(main_err);
      for (auto& e : err)
        if (e) std::rethrow_exception(e);
    }
  }
  RSF_CUDA(cudaStreamSynchronize(s));
  R.t_jobs_wall = now_s() - tj0;
  // (RSF_EMU_EXCHANGE=1 routes a single-GPU evaluation through the same record exchange: tests)
  const bool emu_exchange = getenv("RSF_EMU_EXCHANGE") && getenv("RSF_EMU_EXCHANGE")[0] == '1';
  if ((ctx.comm.use_nccl() || emu_exchange) && njobs > 0) {
    // every job's results from the lowest rank of the group that ran it (all members hold the
    // same values): one all-gather of fixed-size records over the whole group
    constexpr int RS = 13 + 4 * 32;
    std::vector<double> rec((size_t)njobs * RS, 0.0), all((size_t)ctx.comm.world * njobs * RS);
    for (int j = 0; j < njobs; ++j) {
      if (!mine(j)) continue;
      double* r = rec.data() + (size_t)j * RS;
      const int i = job_theta[j];
      const PeelDiag& pd = i >= 0 ? R.pd[i] : pd_trinv;
      r[0] = 1.0;
      r[1] = i >= 0 ? qv[i] : utu;
      r[2] = i >= 0 ? trv[i] : trinv;
      r[3] = i >= 0 ? tcomp[i] : 0.0;
      r[4] = i >= 0 ? tsol[i] : 0.0;
      r[5] = i >= 0 ? tpl[i] : t_trinv;
      r[6] = i >= 0 ? ffl[i] : 0.0;
      r[7] = pd.nL; r[8] = pd.cancellation; r[9] = pd.applies; r[10] = pd.seconds; r[11] = pd.flops;
      r[12] = pd.stored_bytes;
      for (size_t l = 0; l < pd.cols.size() && l < 32; ++l) {
        r[13 + l] = pd.cols[l]; r[45 + l] = pd.rank_max[l];
        r[77 + l] = l < pd.rank_min.size() ? pd.rank_min[l] : 0; r[109 + l] = l < pd.rank_med.size() ? pd.rank_med[l] : 0;
      }
    }
    ctx.comm.allgather_host(s, rec.data(), njobs * RS, all.data());
    for (int j = 0; j < njobs; ++j) {
      const double* r = nullptr;
      for (int rk = 0; rk < ctx.comm.world && !r; ++rk)
        if (all[((size_t)rk * njobs + j) * RS] == 1.0) r = all.data() + ((size_t)rk * njobs + j) * RS;
      RSF_REQUIRE(r != nullptr, ST_ENCCL, "sharded evaluation: a trace job ran on no rank");
      const int i = job_theta[j];
      PeelDiag& pd = i >= 0 ? R.pd[i] : pd_trinv;
      if (i >= 0) { qv[i] = r[1]; trv[i] = r[2]; tcomp[i] = r[3]; tsol[i] = r[4]; tpl[i] = r[5]; ffl[i] = r[6]; }
      else { utu = r[1]; trinv = r[2]; t_trinv = r[5]; }
      pd.nL = (int)r[7]; pd.cancellation = r[8]; pd.applies = r[9]; pd.seconds = r[10]; pd.flops = r[11];
      const int nl = std::min(32, tree->L + 1);
      pd.stored_bytes = r[12];
      pd.cols.assign(nl, 0);
      pd.rank_max.assign(nl, 0);
      pd.rank_min.assign(nl, 0);
      pd.rank_med.assign(nl, 0);
      for (int l = 0; l < nl; ++l) {
        pd.cols[l] = (int)r[13 + l]; pd.rank_max[l] = (int)r[45 + l];
        pd.rank_min[l] = (int)r[77 + l]; pd.rank_med[l] = (int)r[109 + l];
      }
    }
  }
  R.t_peel += t_trinv;
  for (int i = 0; i < p; ++i) {
    const int w = theta[i];
    double q, tr;
    if (w == W_SIGMA2 || w == W_NUGGET) {
      R.pd[i] = pd_trinv;
      if (w == W_NUGGET) { q = utu; tr = trinv; }
      else { q = (R.quad - kp.nugget * utu) / kp.sigma2; tr = (n - kp.nugget * trinv) / kp.sigma2; }
    } else {
      q = qv[i];
      tr = trv[i];
      R.t_compress += tcomp[i];
      R.t_solve += tsol[i];
      R.t_peel += tpl[i];
      R.flops_factor += ffl[i];
    }
    R.q[i] = q;
    R.trace[i] = tr;
    R.grad[i] = profile ? 0.5 * n * q / Qp - 0.5 * tr : 0.5 * q - 0.5 * tr;
  }
  RSF_CUDA(cudaStreamSynchronize(s));
  R.t_total = now_s() - T0;
  R.launches = g_launches - l0;
  return R;
}

void fill_eval_diag(const EvalResult& r, rsf_eval_diag* out) {
  std::memset(out, 0, sizeof(*out));
  out->logdet = r.logdet;
  out->quad = r.quad;
  for (int i = 0; i < 4; ++i) { out->q[i] = r.q[i]; out->trace[i] = r.trace[i]; fill_peel_diag(r.pd[i], &out->peel[i]); }
  out->t_tree = r.t_tree;
  out->t_factor = r.t_factor;
  out->t_compress = r.t_compress;
  out->t_solve = r.t_solve;
  out->t_peel = r.t_peel;
  out->t_total = r.t_total;
  out->flops_factor = r.flops_factor;
  out->kernel_launches = (double)r.launches;
  out->t_jobs_wall = r.t_jobs_wall;
  out->jobs = r.jobs;
  out->concurrent = r.concurrent;
  out->serial_fallback = r.serial_fallback;
  out->groups = r.groups;
  out->fact.levels = r.L;
  out->fact.top_size = r.n0;
  const auto& d = r.fdiag;
  for (size_t i = 0; i < d.level_boxes.size() && i < 32; ++i) {
    int lev = r.L - (int)i;
    if (lev < 0 || lev >= 32) continue;
    out->fact.level_boxes[lev] = d.level_boxes[i];
    out->fact.level_active[lev] = d.level_I[i];
    out->fact.level_skel[lev] = d.level_S[i];
    out->fact.level_maxI[lev] = d.level_maxI[i];
  }
  out->fact.flops_id = d.flops_id;
  out->fact.flops_elim = d.flops_elim;
  out->fact.flops_top = d.flops_top;
  out->fact.factor_bytes = d.bytes_factor;
  out->fact.seconds = r.t_factor;
}

}  // namespace rsf

// Batched dense FP64 factorizations (see dense.cuh).
#include <algorithm>
#include <mutex>

#include <cooperative_groups.h>

#include "dense.cuh"

namespace rsf {

namespace cg = cooperative_groups;

namespace {

constexpr int NT = 256;
constexpr size_t SMEM_BUDGET = 200 * 1024;
constexpr size_t SMEM_MAX = 227 * 1024;   // sm_100 opt-in dynamic shared memory per CTA

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum; sh must hold >= 32 doubles; all threads get the result
__device__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = (threadIdx.x < (blockDim.x >> 5)) ? sh[threadIdx.x] : 0.0;
  if (w == 0) r = warp_sum(r);
  if (threadIdx.x == 0) sh[0] = r;
  __syncthreads();
  return sh[0];
}

// LAPACK dlarfg-style reflector: given alpha = x0 and sigma = ||x(1:)||^2,
// H = I - tau v v^T with v0 = 1 maps x to beta e1.
__device__ __forceinline__ void householder(double alpha, double sigma, double& tau, double& beta,
                                            double& scale) {
  if (sigma == 0.0) {
    tau = 0.0; beta = alpha; scale = 0.0;
    return;
  }
  double mu = sqrt(alpha * alpha + sigma);
  beta = (alpha >= 0.0) ? -mu : mu;
  tau = (beta - alpha) / beta;
  scale = 1.0 / (alpha - beta);
}

// ------------------------------------------------------------------ QR panel
struct PanelDesc {
  double* A;       // points at A(j0, j0)
  long long lda;
  int rows, ncol;  // rows = m - j0, ncol = panel width
  double* V;       // explicit unit-lower V, rows x ncol, ld = rows
  double* T;       // ncol x ncol, ld = QR_NB
  double* tau;     // ncol (may be null)
  int smem;        // panel staged in shared memory
};

template <int NTH>
__global__ void __launch_bounds__(NTH) qr_panel_kernel(const PanelDesc* __restrict__ descs) {
  extern __shared__ double sm[];
  const PanelDesc d = descs[blockIdx.x];
  double* red = sm;                 // 32
  double* scal = sm + 32;           // 8
  double* taus = sm + 40;           // QR_NB
  double* G = taus + QR_NB;         // QR_NB * QR_NB
  double* Ts = G + QR_NB * QR_NB;   // QR_NB * QR_NB
  double* pan = Ts + QR_NB * QR_NB;
  const int rows = d.rows, ncol = d.ncol;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* P;
  long long ldp;
  if (d.smem) {
    P = pan;
    ldp = rows;
    for (long long e = tid; e < (long long)rows * ncol; e += NTH) {
      int r = (int)(e % rows), c = (int)(e / rows);
      P[e] = d.A[c * d.lda + r];
    }
    __syncthreads();
  } else {
    P = d.A;
    ldp = d.lda;
  }
  for (int jj = 0; jj < ncol; ++jj) {
    const int len = rows - jj;
    double* x = P + jj * ldp + jj;
    double s = 0.0;
    for (int r = 1 + tid; r < len; r += NTH) s += x[r] * x[r];
    s = block_sum(s, red);
    if (tid == 0) {
      double tau, beta, scale;
      householder(len > 0 ? x[0] : 0.0, s, tau, beta, scale);
      scal[0] = tau; scal[1] = beta; scal[2] = scale;
      taus[jj] = tau;
    }
    __syncthreads();
    const double tau = scal[0], scale = scal[2];
    if (tau != 0.0)
      for (int r = 1 + tid; r < len; r += NTH) x[r] *= scale;
    __syncthreads();
    if (tid == 0 && len > 0) x[0] = scal[1];
    // apply H to the remaining panel columns
    if (tau != 0.0) {
      for (int col = jj + 1 + warp; col < ncol; col += NTH / 32) {
        double* y = P + col * ldp + jj;
        double dot = 0.0;
        for (int r = 1 + lane; r < len; r += 32) dot += x[r] * y[r];
        dot = warp_sum(dot);
        dot += y[0];
        const double w = tau * dot;
        for (int r = 1 + lane; r < len; r += 32) y[r] -= w * x[r];
        __syncwarp();
        if (lane == 0) y[0] -= w;
      }
    }
    __syncthreads();
  }
  if (d.smem) {
    for (long long e = tid; e < (long long)rows * ncol; e += NTH) {
      int r = (int)(e % rows), c = (int)(e / rows);
      d.A[c * d.lda + r] = P[e];
    }
  }
  // explicit V
  for (long long e = tid; e < (long long)rows * ncol; e += NTH) {
    int r = (int)(e % rows), c = (int)(e / rows);
    d.V[e] = (r < c) ? 0.0 : (r == c ? 1.0 : P[c * ldp + r]);
  }
  // G(l, i) = v_l . v_i for l < i
  const int npair = ncol * (ncol - 1) / 2;
  for (int pidx = warp; pidx < npair; pidx += NTH / 32) {
    // decode pair (l, i), l < i
    int i = 1, acc = 0;
    while (acc + i <= pidx) { acc += i; ++i; }
    int l = pidx - acc;
    const double* vl = P + l * ldp;
    const double* vi = P + i * ldp;
    double dot = 0.0;
    for (int r = i + 1 + lane; r < rows; r += 32) dot += vl[r] * vi[r];
    dot = warp_sum(dot);
    if (lane == 0) G[l * QR_NB + i] = dot + vl[i];
  }
  __syncthreads();
  // T (forward, columnwise): T(i,i) = tau_i; T(0:i,i) = -tau_i T(0:i,0:i) G(0:i,i)
  if (warp == 0) {
    for (int i = 0; i < ncol; ++i) {
      double v = 0.0;
      if (lane < i) {
        for (int l2 = lane; l2 < i; ++l2) v += Ts[lane + l2 * QR_NB] * G[l2 * QR_NB + i];
      }
      __syncwarp();
      if (lane < i) Ts[lane + i * QR_NB] = -taus[i] * v;
      for (int r = i + 1 + lane; r < QR_NB; r += 32) Ts[r + i * QR_NB] = 0.0;
      if (lane == 0) Ts[i + i * QR_NB] = taus[i];
      __syncwarp();
    }
  }
  __syncthreads();
  for (int e = tid; e < QR_NB * QR_NB; e += NTH) {
    int r = e % QR_NB, c = e / QR_NB;
    d.T[e] = (r < ncol && c < ncol) ? Ts[e] : 0.0;
  }
  if (d.tau)
    for (int e = tid; e < ncol; e += NTH) d.tau[e] = taus[e];
}

// explicit V for an already-factored panel (ormqr)
struct VDesc { const double* A; long long lda; int rows, ncol; double* V; };
__global__ void build_v_kernel(const VDesc* __restrict__ descs) {
  const VDesc d = descs[blockIdx.y];
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < (long long)d.rows * d.ncol;
       e += (long long)gridDim.x * NT) {
    int r = (int)(e % d.rows), c = (int)(e / d.rows);
    d.V[e] = (r < c) ? 0.0 : (r == c ? 1.0 : d.A[c * d.lda + r]);
  }
}

// ------------------------------------------------------------------ CPQR + T
struct CPQRDesc {
  const double* R; long long ldr; int q, c;
  double* W; long long ldw; int smem;
  double* T; int* piv; int* kout;
  double* Rout; double* tau;
  double eps; int want_T;
};

__global__ void __launch_bounds__(NT) cpqr_kernel(const CPQRDesc* __restrict__ descs) {
  extern __shared__ double sm[];
  const CPQRDesc d = descs[blockIdx.x];
  const int q = d.q, c = d.c;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* red = sm;          // 64
  double* scal = sm + 64;    // 8
  double* nrm = sm + 72;     // c
  int* ipiv = reinterpret_cast<int*>(nrm + c);   // c ints
  int* redi = ipiv + c;                           // 32 ints
  size_t off = 72 + c + ((size_t)c + 32 + 1) / 2 + 1;
  double* W = d.smem ? (sm + off) : d.W;
  const long long ldw = d.smem ? q : d.ldw;
  double* taus = d.tau;

  for (long long e = tid; e < (long long)q * c; e += NT) {
    int i = (int)(e % q), j = (int)(e / q);
    W[j * ldw + i] = (i <= j) ? d.R[j * d.ldr + i] : 0.0;
  }
  for (int j = tid; j < c; j += NT) ipiv[j] = j;
  __syncthreads();
  for (int j = warp; j < c; j += NT / 32) {
    double s = 0.0;
    for (int i = lane; i < q; i += 32) { double v = W[j * ldw + i]; s += v * v; }
    s = warp_sum(s);
    if (lane == 0) nrm[j] = s;
  }
  __syncthreads();
  const int kmax = min(q, c);
  double ref = 0.0;
  int k = 0;
  for (int i = 0; i < kmax; ++i) {
    // argmax over nrm[i..c), lowest position on ties
    double bv = -1.0;
    int bi = c;
    for (int j = i + tid; j < c; j += NT) {
      double v = nrm[j];
      if (v > bv) { bv = v; bi = j; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    __syncthreads();
    if (lane == 0) { red[warp] = bv; redi[warp] = bi; }
    __syncthreads();
    if (tid == 0) {
      double v = red[0]; int b = redi[0];
      for (int w = 1; w < NT / 32; ++w)
        if (red[w] > v || (red[w] == v && redi[w] < b)) { v = red[w]; b = redi[w]; }
      scal[0] = v;
      redi[0] = b;
    }
    __syncthreads();
    const double nr = sqrt(fmax(scal[0], 0.0));
    const int p = redi[0];
    if (i == 0) ref = nr;
    if (!(ref > 0.0) || !(nr > d.eps * ref)) break;
    if (p != i) {
      for (int r = tid; r < q; r += NT) {
        double t = W[i * ldw + r]; W[i * ldw + r] = W[p * ldw + r]; W[p * ldw + r] = t;
      }
      if (tid == 0) {
        double t = nrm[i]; nrm[i] = nrm[p]; nrm[p] = t;
        int ti = ipiv[i]; ipiv[i] = ipiv[p]; ipiv[p] = ti;
      }
      __syncthreads();
    }
    double* x = W + i * ldw + i;
    const int len = q - i;
    double s = 0.0;
    for (int r = 1 + tid; r < len; r += NT) s += x[r] * x[r];
    s = block_sum(s, red);
    if (tid == 0) {
      double tau, beta, scale;
      householder(x[0], s, tau, beta, scale);
      scal[2] = tau; scal[3] = beta; scal[4] = scale;
      if (taus) taus[i] = tau;
    }
    __syncthreads();
    const double tau = scal[2], scale = scal[4];
    if (tau != 0.0)
      for (int r = 1 + tid; r < len; r += NT) x[r] *= scale;
    __syncthreads();
    if (tid == 0) x[0] = scal[3];
    for (int j = i + 1 + warp; j < c; j += NT / 32) {
      double* y = W + j * ldw + i;
      double dot = 0.0;
      if (tau != 0.0) {
        for (int r = 1 + lane; r < len; r += 32) dot += x[r] * y[r];
        dot = warp_sum(dot);
        dot += y[0];
      }
      const double w = tau * dot;
      double ss = 0.0;
      for (int r = 1 + lane; r < len; r += 32) {
        double v = y[r] - w * x[r];
        y[r] = v;
        ss += v * v;
      }
      ss = warp_sum(ss);
      __syncwarp();
      if (lane == 0) { y[0] -= w; nrm[j] = ss; }
    }
    __syncthreads();
    k = i + 1;
  }
  __syncthreads();
  if (tid == 0) d.kout[0] = k;
  for (int j = tid; j < c; j += NT) d.piv[j] = ipiv[j];
  if (d.want_T) {
    // T = R11^-1 R12, back substitution per column (warp per column)
    for (int j = k + warp; j < c; j += NT / 32) {
      double* y = W + j * ldw;
      for (int i = k - 1; i >= 0; --i) {
        __syncwarp();
        const double xi = y[i] / W[i * ldw + i];
        __syncwarp();
        if (lane == 0) y[i] = xi;
        for (int r = lane; r < i; r += 32) y[r] -= W[i * ldw + r] * xi;
      }
      __syncwarp();
      for (int r = lane; r < k; r += 32) d.T[(long long)(j - k) * c + r] = y[r];
    }
  }
  if (d.Rout) {
    __syncthreads();
    for (long long e = tid; e < (long long)q * c; e += NT) {
      int i = (int)(e % q), j = (int)(e / q);
      d.Rout[j * (long long)q + i] = W[j * ldw + i];
    }
  }
}

// ------------------------------------------------------------------ Cholesky
struct DiagDesc {
  double* A; long long lda;   // points at A(j0, j0)
  int nb;                     // block size actually used (<= CH_NB)
  double* Dinv;               // CH_NB x CH_NB scratch (ld CH_NB)
  double* Linv; long long ldi;  // optional: Linv(j0, j0)
  double* logsum; int* info; int col0;
};

__global__ void __launch_bounds__(NT) potrf_diag_kernel(const DiagDesc* __restrict__ descs) {
  extern __shared__ double dsm[];
  double* S = dsm;
  double* X = dsm + CH_NB * CH_NB;
  __shared__ int fail;
  __shared__ double red[32];
  const DiagDesc d = descs[blockIdx.x];
  if (*d.info) return;
  const int nb = d.nb, tid = threadIdx.x;
  for (int e = tid; e < nb * nb; e += NT) {
    int i = e % nb, j = e / nb;
    S[e] = (i >= j) ? d.A[j * d.lda + i] : 0.0;
  }
  if (tid == 0) fail = 0;
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    double djj = S[j * nb + j];
    if (!(djj > 0.0)) {
      if (tid == 0) fail = j + 1;
      break;
    }
    djj = sqrt(djj);
    __syncthreads();
    for (int i = j + 1 + tid; i < nb; i += NT) S[j * nb + i] /= djj;
    if (tid == 0) S[j * nb + j] = djj;
    __syncthreads();
    const int m = nb - j - 1;
    for (int e = tid; e < m * m; e += NT) {
      int i = j + 1 + e % m, l = j + 1 + e / m;
      if (i >= l) S[l * nb + i] -= S[j * nb + i] * S[j * nb + l];
    }
    __syncthreads();
  }
  __syncthreads();
  if (fail) {
    if (tid == 0) *d.info = d.col0 + fail;
    return;
  }
  // inverse of the lower-triangular block, one column per thread
  if (tid < nb) {
    const int c = tid;
    for (int i = 0; i < c; ++i) X[c * nb + i] = 0.0;
    X[c * nb + c] = 1.0 / S[c * nb + c];
    for (int i = c + 1; i < nb; ++i) {
      double s = 0.0;
      for (int l = c; l < i; ++l) s += S[l * nb + i] * X[c * nb + l];
      X[c * nb + i] = -s / S[i * nb + i];
    }
  }
  double ls = 0.0;
  for (int j = tid; j < nb; j += NT) ls += log(S[j * nb + j]);
  ls = block_sum(ls, red);
  if (tid == 0) *d.logsum += ls;
  __syncthreads();
  for (int e = tid; e < nb * nb; e += NT) {
    int i = e % nb, j = e / nb;
    d.A[j * d.lda + i] = (i >= j) ? S[e] : 0.0;
    d.Dinv[j * CH_NB + i] = X[e];
    if (d.Linv) d.Linv[j * d.ldi + i] = X[e];
  }
}

struct ZDesc { double* A; long long lda; int n; };
struct RDesc { double* A; long long lda; int m, n; };
__global__ void zero_rect_kernel(const RDesc* __restrict__ descs) {
  const RDesc d = descs[blockIdx.y];
  const long long tot = (long long)d.m * d.n;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT)
    d.A[(e / d.m) * d.lda + (e % d.m)] = 0.0;
}
__global__ void zero_upper_kernel(const ZDesc* __restrict__ descs) {
  const ZDesc d = descs[blockIdx.y];
  const long long tot = (long long)d.n * d.n;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    int i = (int)(e % d.n), j = (int)(e / d.n);
    if (i < j) d.A[j * d.lda + i] = 0.0;
  }
}

__global__ void zero_all_kernel(const ZDesc* __restrict__ descs) {
  const ZDesc d = descs[blockIdx.y];
  const long long tot = (long long)d.n * d.n;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    int i = (int)(e % d.n), j = (int)(e / d.n);
    d.A[j * d.lda + i] = 0.0;
  }
}

__global__ void copy_kernel(const CopyProb* __restrict__ descs) {
  const CopyProb d = descs[blockIdx.y];
  const long long tot = (long long)d.rows * d.cols;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    int i = (int)(e % d.rows), j = (int)(e / d.rows);
    d.dst[j * d.ldd + i] = d.alpha * d.src[j * d.lds + i];
  }
}

template <class D>
RPtr<D> upload_descs(const std::vector<D>& v, cudaStream_t s) {
  return ring_up(v, s);
}

int grid_x_for(long long maxelems) {
  long long g = (maxelems + NT - 1) / NT;
  return (int)std::max<long long>(1, std::min<long long>(g, 256));
}

// launch a per-problem elementwise kernel with grid.y = problems (chunked to 65535)
template <class D, class K>
void launch_y(cudaStream_t s, const std::vector<D>& v, long long maxelems, K kern) {
  if (v.empty()) return;
  auto d = upload_descs(v, s);
  const int gx = grid_x_for(maxelems);
  for (size_t o = 0; o < v.size(); o += 65535) {
    int ny = (int)std::min<size_t>(65535, v.size() - o);
    kern<<<dim3(gx, ny), NT, 0, s>>>(d.p + o);
    count_launch();
    RSF_LAUNCH_CHECK();
  }
}

// Cluster panel factorization for tall panels: the rows are distributed over the CL CTAs
// of a thread-block cluster and held in shared memory.  Every Householder step needs the
// column norm below the diagonal and the dot products with the remaining columns; each CTA
// computes its partial sums over its rows and writes them to every CTA's exchange buffer
// (DSMEM, double-buffered by step parity), one cluster barrier per column.  The sums over
// ranks are taken in rank order, so the result is deterministic.
constexpr int PC_NT = 512, PC_NW = PC_NT / 32;
constexpr int PC_MAXROWS = 480;            // rows per CTA: QR_NB * 480 * 8 B = 120 KB
constexpr int PC_NPAIR = QR_NB * (QR_NB - 1) / 2;
constexpr int PC_XW = 2 * QR_NB + 2;       // exchange width per rank

template <int CL>
__global__ void __launch_bounds__(PC_NT) qr_panel_cl_kernel(const PanelDesc* __restrict__ descs) {
  extern __shared__ double pcm[];
  __shared__ double xch[2][CL][PC_XW];
  __shared__ double scal[4];
  __shared__ double wv[QR_NB];
  __shared__ double taus[QR_NB];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const PanelDesc d = descs[blockIdx.x / CL];
  const int rows = d.rows, ncol = d.ncol;
  const int chunk = max((rows + CL - 1) / CL, QR_NB);   // rows < QR_NB (R, pivots) live in rank 0
  const int r0 = rank * chunk, nr = max(0, min(rows, r0 + chunk) - r0);
  double* P = pcm;                          // local rows: P[c * chunk + lr]
  double* gbuf = pcm + QR_NB * chunk;       // rank 0: partial Gram [CL][PC_NPAIR]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < ncol * nr; e += PC_NT) {
    const int c = e / nr, lr = e % nr;
    P[c * chunk + lr] = d.A[(long long)c * d.lda + r0 + lr];
  }
  __syncthreads();
  for (int j = 0; j < ncol; ++j) {
    const int buf = j & 1;
    // partial sums over the local rows below the diagonal: sigma (column j) and x . y_c (c > j)
    for (int c = j + warp; c < ncol; c += PC_NW) {
      double acc = 0.0;
      const double* x = P + j * chunk;
      const double* y = P + c * chunk;
      for (int lr = lane; lr < nr; lr += 32)
        if (r0 + lr > j) acc += x[lr] * y[lr];
#pragma unroll
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) wv[c - j] = acc;      // wv[0] = sigma, wv[c - j] = dot_c
    }
    __syncthreads();
    // publish (rank 0 adds alpha = x_j and y_c[j], its own rows)
    if (tid < CL) {
      double* dst = &cluster.map_shared_rank(&xch[0][0][0], tid)[(buf * CL + rank) * PC_XW];
      for (int q = 0; q < ncol - j; ++q) dst[q] = wv[q];
      if (rank == 0) {
        dst[QR_NB] = P[j * chunk + j];
        for (int c = j + 1; c < ncol; ++c) dst[QR_NB + 1 + (c - j - 1)] = P[c * chunk + j];
      }
    }
    cluster.sync();
    if (tid == 0) {
      double sigma = 0.0;
      for (int r = 0; r < CL; ++r) sigma += xch[buf][r][0];
      const double alpha = xch[buf][0][QR_NB];
      double tau = 0.0, beta = alpha, scale = 0.0;
      if (sigma != 0.0) {
        const double mu = sqrt(alpha * alpha + sigma);
        beta = (alpha >= 0.0) ? -mu : mu;
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      scal[0] = tau; scal[1] = beta; scal[2] = scale;
      taus[j] = tau;
      for (int c = j + 1; c < ncol; ++c) {
        double dot = 0.0;
        for (int r = 0; r < CL; ++r) dot += xch[buf][r][c - j];
        wv[c - j] = tau * (xch[buf][0][QR_NB + 1 + (c - j - 1)] + scale * dot);
      }
    }
    __syncthreads();
    const double scale = scal[2];
    // v = x(j+1:)/scale-normalised; y_c -= w_c v
    for (int lr = tid; lr < nr; lr += PC_NT) {
      const int g = r0 + lr;
      if (g <= j) continue;
      const double v = P[j * chunk + lr] * scale;
      P[j * chunk + lr] = v;
      for (int c = j + 1; c < ncol; ++c) P[c * chunk + lr] -= wv[c - j] * v;
    }
    if (rank == 0 && tid == 0) {
      for (int c = j + 1; c < ncol; ++c) P[c * chunk + j] -= wv[c - j];
      P[j * chunk + j] = scal[1];
    }
    __syncthreads();
  }
  // write back R (rank 0's top rows) and the reflectors, explicit unit-lower V
  for (int e = tid; e < ncol * nr; e += PC_NT) {
    const int c = e / nr, lr = e % nr, g = r0 + lr;
    const double v = P[c * chunk + lr];
    d.A[(long long)c * d.lda + g] = v;
    d.V[(long long)c * rows + g] = (g < c) ? 0.0 : (g == c ? 1.0 : v);
  }
  // partial Gram G(l, i) = sum_{rows > i} v_l v_i (l < i) -> rank 0
  for (int pidx = warp; pidx < ncol * (ncol - 1) / 2; pidx += PC_NW) {
    int i = 1, acc0 = 0;
    while (acc0 + i <= pidx) { acc0 += i; ++i; }
    const int l = pidx - acc0;
    double acc = 0.0;
    for (int lr = lane; lr < nr; lr += 32)
      if (r0 + lr > i) acc += P[l * chunk + lr] * P[i * chunk + lr];
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) cluster.map_shared_rank(gbuf, 0)[rank * PC_NPAIR + pidx] = acc;
  }
  cluster.sync();
  if (rank != 0) return;
  // rank 0: G(l, i) = v_l(i) + sum over ranks; T (forward, columnwise) as qr_panel_kernel
  double* G = gbuf + CL * PC_NPAIR;       // QR_NB x QR_NB
  double* Ts = G + QR_NB * QR_NB;
  for (int pidx = tid; pidx < ncol * (ncol - 1) / 2; pidx += PC_NT) {
    int i = 1, acc0 = 0;
    while (acc0 + i <= pidx) { acc0 += i; ++i; }
    const int l = pidx - acc0;
    double v = P[l * chunk + i];   // v_l(i) (row i < QR_NB lives in rank 0)
    for (int r = 0; r < CL; ++r) v += gbuf[r * PC_NPAIR + pidx];
    G[l * QR_NB + i] = v;
  }
  __syncthreads();
  if (warp == 0) {
    for (int i = 0; i < ncol; ++i) {
      double v = 0.0;
      if (lane < i)
        for (int l2 = lane; l2 < i; ++l2) v += Ts[lane + l2 * QR_NB] * G[l2 * QR_NB + i];
      __syncwarp();
      if (lane < i) Ts[lane + i * QR_NB] = -taus[i] * v;
      for (int r = i + 1 + lane; r < QR_NB; r += 32) Ts[r + i * QR_NB] = 0.0;
      if (lane == 0) Ts[i + i * QR_NB] = taus[i];
      __syncwarp();
    }
  }
  __syncthreads();
  for (int e = tid; e < QR_NB * QR_NB; e += PC_NT) {
    const int r = e % QR_NB, c = e / QR_NB;
    d.T[e] = (r < ncol && c < ncol) ? Ts[e] : 0.0;
  }
  if (d.tau)
    for (int e = tid; e < ncol; e += PC_NT) d.tau[e] = taus[e];
}

template <int CL>
void launch_panel_cl(cudaStream_t s, const PanelDesc* d, int np, int chunk) {
  static std::once_flag attr_once;
  const size_t smem = ((size_t)QR_NB * chunk + (size_t)CL * PC_NPAIR + 2 * QR_NB * QR_NB) * sizeof(double);
  std::call_once(attr_once, [&] {
    cudaFuncAttributes fa;
    RSF_CUDA(cudaFuncGetAttributes(&fa, qr_panel_cl_kernel<CL>));
    RSF_CUDA(cudaFuncSetAttribute(qr_panel_cl_kernel<CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(SMEM_MAX - fa.sharedSizeBytes)));
    if (CL > 8) RSF_CUDA(cudaFuncSetAttribute(qr_panel_cl_kernel<CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  });
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(np * CL));
  cfg.blockDim = dim3(PC_NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  RSF_CUDA(cudaLaunchKernelEx(&cfg, qr_panel_cl_kernel<CL>, d));
  count_launch();
}

// Register-resident panel factorization (round 2): every thread of the cluster holds ONE row
// of the panel (QR_NB doubles in registers), rows distributed over the CL CTAs (<= 512 each).
// A Householder step needs the column norm below the diagonal and the dot products with the
// later columns: each thread forms its 32 products, a warp "transpose reduction" (31 shuffles,
// lane c ends with the warp's sum for column c) and a 16-way sum in shared memory give the
// CTA's partials, which go to every CTA of the cluster through DSMEM (double-buffered by step
// parity) -- one cluster barrier and two CTA barriers per column, no serial per-thread loops.
// Sums over warps and ranks are taken in a fixed order (deterministic).  The WY factor T comes
// from the Gram matrix of the reflectors, reduced the same way.
constexpr int PR_NT = 512, PR_NW = PR_NT / 32;

// Warp "transpose reduction" of 32 per-lane values f(c), c = 0..31: on return lane c holds the
// sum over the warp's lanes of f(c).  31 shuffles; the first stage forms the values on the fly
// (only 16 live at a time).
template <class F>
__device__ __forceinline__ double transpose_reduce32(F f, int lane) {
  double v[16];
  {
    const bool up = (lane & 16) != 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const double lo = f(i), hi = f(i + 16);
      v[i] = (up ? hi : lo) + __shfl_xor_sync(0xffffffffu, up ? lo : hi, 16);
    }
  }
#pragma unroll
  for (int h = 8; h >= 1; h >>= 1) {
    const bool up = (lane & h) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const double lo = v[i], hi = v[i + h];
      v[i] = (up ? hi : lo) + __shfl_xor_sync(0xffffffffu, up ? lo : hi, h);
    }
  }
  return v[0];
}

template <int CL>
__global__ void __launch_bounds__(PR_NT, 1) qr_panel_reg_kernel(const PanelDesc* __restrict__ descs) {
  static_assert(QR_NB == 32, "one warp lane per panel column");
  __shared__ double red[PR_NW][QR_NB];
  __shared__ double xch[2][CL][QR_NB];      // per-rank partial sums (slot j: sigma)
  __shared__ double xrow[2][QR_NB];         // row j of the panel (rank 0)
  __shared__ double wv[QR_NB], taus[QR_NB], scal[4];
  __shared__ double G[QR_NB * QR_NB], Ts[QR_NB * QR_NB];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const PanelDesc d = descs[blockIdx.x / CL];
  const int rows = d.rows, ncol = d.ncol;
  const int chunk = max((rows + CL - 1) / CL, QR_NB);
  const int r0 = rank * chunk, nr = max(0, min(rows, r0 + chunk) - r0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = r0 + tid;                   // this thread's global panel row
  const bool mine = tid < nr;
  double a[QR_NB];
#pragma unroll
  for (int c = 0; c < QR_NB; ++c) a[c] = (mine && c < ncol) ? d.A[(long long)c * d.lda + g] : 0.0;
  // (the step index j stays a loop variable -- a fully unrolled loop of 32 steps measured ~25k
  // instructions of code, thrashing the instruction cache; a[j] is read with a 32-way select)
  auto pick = [&](int j) {
    double v = 0.0;
#pragma unroll
    for (int c = 0; c < QR_NB; ++c) v = (c == j) ? a[c] : v;
    return v;
  };
  // One transpose reduction per step gives, for the rows below the diagonal, x . a_c for EVERY
  // column c: c > j the dot products of the update, c == j the norm sigma, and c < j (a_c already
  // holds the reflector v_c) the Gram entries v_c . v_j of the WY factor T once scaled -- no
  // separate Gram pass after the panel.
#pragma unroll 1
  for (int j = 0; j < ncol; ++j) {
    const int buf = j & 1;
    const double aj = pick(j);
    const double x = (mine && g > j) ? aj : 0.0;
    const double ps = transpose_reduce32([&](int c) { return x * a[c]; }, lane);
    red[warp][lane] = ps;
    if (rank == 0 && tid == j) {
#pragma unroll
      for (int c = 0; c < QR_NB; ++c) xrow[buf][c] = a[c];
    }
    __syncthreads();
    if (tid < QR_NB) {
      double sacc = 0.0;
      for (int w = 0; w < PR_NW; ++w) sacc += red[w][tid];
      const double rv = xrow[buf][tid];
#pragma unroll 1
      for (int q = 0; q < CL; ++q) {
        cluster.map_shared_rank(&xch[0][0][0], q)[(buf * CL + rank) * QR_NB + tid] = sacc;
        if (rank == 0 && q > 0) cluster.map_shared_rank(&xrow[0][0], q)[buf * QR_NB + tid] = rv;
      }
    }
    cluster.sync();
    if (tid < QR_NB) {
      double sigma = 0.0, dot = 0.0;
      for (int r = 0; r < CL; ++r) { sigma += xch[buf][r][j]; dot += xch[buf][r][tid]; }
      const double alpha = xrow[buf][j];
      double tau = 0.0, beta = alpha, scale = 0.0;
      if (sigma != 0.0) {
        const double mu = sqrt(alpha * alpha + sigma);
        beta = (alpha >= 0.0) ? -mu : mu;
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      wv[tid] = (tid > j) ? tau * (xrow[buf][tid] + scale * dot) : 0.0;
      if (tid < j) G[tid * QR_NB + j] = xrow[buf][tid] + scale * dot;   // v_tid(j) + v_tid . v_j below row j
      if (tid == 0) { scal[0] = tau; scal[1] = beta; scal[2] = scale; taus[j] = tau; }
    }
    __syncthreads();
    if (mine && g > j) {
      const double v = aj * scal[2];
#pragma unroll
      for (int c = 0; c < QR_NB; ++c) a[c] = (c == j) ? v : fma(-wv[c], v, a[c]);   // wv = 0 for c <= j
    } else if (mine && g == j) {
      const double beta = scal[1];
#pragma unroll
      for (int c = 0; c < QR_NB; ++c) a[c] = (c == j) ? beta : a[c] - wv[c];
    }
  }
  // write back R (rows < ncol of rank 0) and the reflectors; explicit unit-lower V
  if (mine) {
#pragma unroll
    for (int c = 0; c < QR_NB; ++c) {
      if (c >= ncol) break;
      d.A[(long long)c * d.lda + g] = a[c];
      d.V[(long long)c * rows + g] = (g < c) ? 0.0 : (g == c ? 1.0 : a[c]);
    }
  }
  if (rank != 0) return;
  __syncthreads();
  if (warp == 0) {
    for (int i = 0; i < ncol; ++i) {
      double v = 0.0;
      if (lane < i)
        for (int l2 = lane; l2 < i; ++l2) v += Ts[lane + l2 * QR_NB] * G[l2 * QR_NB + i];
      __syncwarp();
      if (lane < i) Ts[lane + i * QR_NB] = -taus[i] * v;
      for (int r = i + 1 + lane; r < QR_NB; r += 32) Ts[r + i * QR_NB] = 0.0;
      if (lane == 0) Ts[i + i * QR_NB] = taus[i];
      __syncwarp();
    }
  }
  __syncthreads();
  for (int e = tid; e < QR_NB * QR_NB; e += PR_NT) {
    const int r = e % QR_NB, c = e / QR_NB;
    d.T[e] = (r < ncol && c < ncol) ? Ts[e] : 0.0;
  }
  if (d.tau)
    for (int e = tid; e < ncol; e += PR_NT) d.tau[e] = taus[e];
}

template <int CL>
void launch_panel_reg(cudaStream_t s, const PanelDesc* d, int np) {
  static std::once_flag attr_once;
  const size_t smem = 0;
  std::call_once(attr_once, [&] {
    if (CL > 8) RSF_CUDA(cudaFuncSetAttribute(qr_panel_reg_kernel<CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  });
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(np * CL));
  cfg.blockDim = dim3(PR_NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  RSF_CUDA(cudaLaunchKernelEx(&cfg, qr_panel_reg_kernel<CL>, d));
  count_launch();
}

// panels in global memory (too tall for shared memory) are latency bound: give them
// 1024 threads (one warp per remaining panel column, 4x the loads in flight)
void launch_panels(cudaStream_t s, const std::vector<PanelDesc>& pd, const PanelDesc* d, size_t smem_need) {
  static std::once_flag attr_once;
  std::call_once(attr_once, [&] {
    RSF_CUDA(cudaFuncSetAttribute(qr_panel_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_MAX));
    RSF_CUDA(cudaFuncSetAttribute(qr_panel_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_MAX));
  });
  bool tall = false;
  int maxrows = 0;
  for (auto& p : pd) { tall |= (p.smem == 0); maxrows = std::max(maxrows, p.rows); }
  static const bool reg_on = !(getenv("RSF_PANEL_REG") && getenv("RSF_PANEL_REG")[0] == '0');
  if (reg_on && maxrows <= 16 * PR_NT && pd.size() <= 65535) {
    int CL = 1;
    while ((maxrows + CL - 1) / CL > PR_NT) CL *= 2;
    switch (CL) {
      case 1: launch_panel_reg<1>(s, d, (int)pd.size()); break;
      case 2: launch_panel_reg<2>(s, d, (int)pd.size()); break;
      case 4: launch_panel_reg<4>(s, d, (int)pd.size()); break;
      case 8: launch_panel_reg<8>(s, d, (int)pd.size()); break;
      default: launch_panel_reg<16>(s, d, (int)pd.size()); break;
    }
    RSF_LAUNCH_CHECK();
    return;
  }
  static const bool cl_on = !(getenv("RSF_PANEL_CLUSTER") && getenv("RSF_PANEL_CLUSTER")[0] == '0');
  if (tall && cl_on && maxrows <= 16 * PC_MAXROWS && pd.size() <= 65535) {
    int CL = 2;
    while ((maxrows + CL - 1) / CL > PC_MAXROWS) CL *= 2;
    const int chunk = std::max((maxrows + CL - 1) / CL, QR_NB);
    switch (CL) {
      case 2: launch_panel_cl<2>(s, d, (int)pd.size(), chunk); break;
      case 4: launch_panel_cl<4>(s, d, (int)pd.size(), chunk); break;
      case 8: launch_panel_cl<8>(s, d, (int)pd.size(), chunk); break;
      default: launch_panel_cl<16>(s, d, (int)pd.size(), chunk); break;
    }
    RSF_LAUNCH_CHECK();
    return;
  }
  for (size_t o = 0; o < pd.size(); o += 65535) {
    const unsigned nb = (unsigned)std::min<size_t>(65535, pd.size() - o);
    if (tall) qr_panel_kernel<1024><<<nb, 1024, smem_need, s>>>(d + o);
    else qr_panel_kernel<NT><<<nb, NT, smem_need, s>>>(d + o);
    count_launch();
    RSF_LAUNCH_CHECK();
  }
}

}  // namespace

void copy_batched(cudaStream_t s, const std::vector<CopyProb>& probs) {
  long long mx = 0;
  for (auto& p : probs) mx = std::max(mx, (long long)p.rows * p.cols);
  if (mx == 0) return;
  launch_y(s, probs, mx, copy_kernel);
}

// ------------------------------------------------------------------ geqrf
void geqrf_batched(cudaStream_t s, const std::vector<QRProb>& probs, bool keep_q) {
  if (probs.empty()) return;
  static std::once_flag attr_once;
  std::call_once(attr_once, [&] {
  });
  const int P = (int)probs.size();
  // workspace: V (m x QR_NB), T (QR_NB^2), W and W2 (QR_NB x c)
  std::vector<long long> voff(P), woff(P), toff(P);
  long long vtot = 0, wtot = 0;
  int maxk = 0;
  for (int i = 0; i < P; ++i) {
    voff[i] = vtot; vtot += (long long)probs[i].m * QR_NB;
    woff[i] = wtot; wtot += (long long)QR_NB * probs[i].c;
    toff[i] = (long long)i * QR_NB * QR_NB;
    maxk = std::max(maxk, std::min(probs[i].m, probs[i].c));
  }
  DBuf<double> V(vtot, s), W(wtot, s), W2(wtot, s), Tscr(keep_q ? 0 : (size_t)P * QR_NB * QR_NB, s);
  const size_t base_smem = (40 + QR_NB + 2 * QR_NB * QR_NB) * sizeof(double);
  for (int j0 = 0; j0 < maxk; j0 += QR_NB) {
    std::vector<PanelDesc> pd;
    GemmBatch g1(true, false), g2(false, false), g3(false, true);
    size_t smem_need = base_smem;
    for (int i = 0; i < P; ++i) {
      const QRProb& q = probs[i];
      const int kk = std::min(q.m, q.c);
      if (j0 >= kk) continue;
      const int nbp = std::min(QR_NB, kk - j0);
      const int rows = q.m - j0;
      PanelDesc d;
      d.A = q.A + j0 * q.lda + j0;
      d.lda = q.lda;
      d.rows = rows;
      d.ncol = nbp;
      d.V = V.p + voff[i];
      d.T = keep_q ? q.Tws + (long long)(j0 / QR_NB) * QR_NB * QR_NB : Tscr.p + toff[i];
      d.tau = keep_q && q.tau ? q.tau + j0 : nullptr;
      const size_t pbytes = (size_t)rows * nbp * sizeof(double);
      d.smem = (base_smem + pbytes <= SMEM_MAX) ? 1 : 0;
      if (d.smem) smem_need = std::max(smem_need, base_smem + pbytes);
      pd.push_back(d);
      const int j1 = j0 + nbp;
      const int c2 = q.c - j1;
      if (c2 > 0) {
        // compact-WY update with the skinny dimension as N (the 128-row tiles stay full):
        GemmDesc a = gdesc(c2, nbp, rows);          // W^T = A2^T V
        a.A = q.A + (long long)j1 * q.lda + j0; a.lda = (int)q.lda;
        a.B = d.V; a.ldb = rows;
        a.C = W.p + woff[i]; a.ldc = c2;
        g1.add(a);
        GemmDesc b = gdesc(c2, nbp, nbp);           // W2^T = W^T T
        b.A = W.p + woff[i]; b.lda = c2;
        b.B = d.T; b.ldb = QR_NB;
        b.C = W2.p + woff[i]; b.ldc = c2;
        g2.add(b);
        GemmDesc c = gdesc(rows, c2, nbp);          // A2 -= V W2
        c.A = d.V; c.lda = rows;
        c.B = W2.p + woff[i]; c.ldb = c2;
        c.C = q.A + (long long)j1 * q.lda + j0; c.ldc = (int)q.lda;
        c.alpha = -1.0; c.beta = 1.0;
        g3.add(c);
      }
    }
    if (pd.empty()) continue;
    auto dd = upload_descs(pd, s);
    launch_panels(s, pd, dd.p, smem_need);
    RSF_LAUNCH_CHECK();
    g1.run(s);
    g2.run(s);
    g3.run(s);
  }
}

void panel_step_batched(cudaStream_t s, const std::vector<PanelStep>& v) {
  if (v.empty()) return;
  static std::once_flag attr_once;
  std::call_once(attr_once, [&] {
  });
  const size_t base_smem = (40 + QR_NB + 2 * QR_NB * QR_NB) * sizeof(double);
  size_t smem_need = base_smem;
  std::vector<PanelDesc> pd;
  GemmBatch g1(true, false), g2(false, false), g3(false, true);
  for (const PanelStep& q : v) {
    PanelDesc d;
    d.A = q.A; d.lda = q.lda; d.rows = q.rows; d.ncol = q.ncol;
    d.V = q.V; d.T = q.T; d.tau = nullptr;
    const size_t pbytes = (size_t)q.rows * q.ncol * sizeof(double);
    d.smem = (base_smem + pbytes <= SMEM_MAX) ? 1 : 0;
    if (d.smem) smem_need = std::max(smem_need, base_smem + pbytes);
    pd.push_back(d);
    if (q.c2 > 0) {
      double* A2 = q.A + (long long)q.ncol * q.lda;
      GemmDesc a = gdesc(q.c2, q.ncol, q.rows);     // W^T = A2^T V
      a.A = A2; a.lda = (int)q.lda; a.B = q.V; a.ldb = q.rows; a.C = q.W; a.ldc = q.c2;
      g1.add(a);
      GemmDesc b = gdesc(q.c2, q.ncol, q.ncol);     // W2^T = W^T T
      b.A = q.W; b.lda = q.c2; b.B = q.T; b.ldb = QR_NB; b.C = q.W2; b.ldc = q.c2;
      g2.add(b);
      GemmDesc c = gdesc(q.rows, q.c2, q.ncol);     // A2 -= V W2
      c.A = q.V; c.lda = q.rows; c.B = q.W2; c.ldb = q.c2; c.C = A2; c.ldc = (int)q.lda;
      c.alpha = -1.0; c.beta = 1.0;
      g3.add(c);
    }
  }
  auto dd = upload_descs(pd, s);
  launch_panels(s, pd, dd.p, smem_need);
  g1.run(s);
  g2.run(s);
  g3.run(s);
}

void ormqr_batched(cudaStream_t s, const std::vector<QApplyProb>& probs, bool trans) {
  if (probs.empty()) return;
  const int P = (int)probs.size();
  std::vector<long long> voff(P), woff(P);
  long long vtot = 0, wtot = 0;
  int maxk = 0;
  for (int i = 0; i < P; ++i) {
    voff[i] = vtot; vtot += (long long)probs[i].m * QR_NB;
    woff[i] = wtot; wtot += (long long)QR_NB * probs[i].nc;
    maxk = std::max(maxk, std::min(probs[i].m, probs[i].c));
  }
  DBuf<double> V(vtot, s), W(wtot, s), W2(wtot, s);
  const int npan = (maxk + QR_NB - 1) / QR_NB;
  for (int pi = 0; pi < npan; ++pi) {
    const int pp = trans ? pi : (npan - 1 - pi);
    const int j0 = pp * QR_NB;
    std::vector<VDesc> vd;
    GemmBatch g1(true, false), g2(!trans ? false : true, false), g3(false, false);
    long long mx = 0;
    for (int i = 0; i < P; ++i) {
      const QApplyProb& q = probs[i];
      const int kk = std::min(q.m, q.c);
      if (j0 >= kk || q.nc <= 0) continue;
      const int nbp = std::min(QR_NB, kk - j0);
      const int rows = q.m - j0;
      VDesc v{q.A + j0 * q.lda + j0, q.lda, rows, nbp, V.p + voff[i]};
      vd.push_back(v);
      mx = std::max(mx, (long long)rows * nbp);
      const double* Tp = q.Tws + (long long)pp * QR_NB * QR_NB;
      GemmDesc a = gdesc(nbp, q.nc, rows);          // W = V^T C
      a.A = V.p + voff[i]; a.lda = rows;
      a.B = q.C + j0; a.ldb = (int)q.ldc;
      a.C = W.p + woff[i]; a.ldc = QR_NB;
      g1.add(a);
      GemmDesc b = gdesc(nbp, q.nc, nbp);           // W2 = T^T W (Q^T) or T W (Q)
      b.A = Tp; b.lda = QR_NB;
      b.B = W.p + woff[i]; b.ldb = QR_NB;
      b.C = W2.p + woff[i]; b.ldc = QR_NB;
      g2.add(b);
      GemmDesc c = gdesc(rows, q.nc, nbp);          // C -= V W2
      c.A = V.p + voff[i]; c.lda = rows;
      c.B = W2.p + woff[i]; c.ldb = QR_NB;
      c.C = q.C + j0; c.ldc = (int)q.ldc;
      c.alpha = -1.0; c.beta = 1.0;
      g3.add(c);
    }
    if (vd.empty()) continue;
    launch_y(s, vd, mx, build_v_kernel);
    g1.run(s);
    g2.run(s);
    g3.run(s);
  }
}

// ------------------------------------------------------------------ cpqr
void cpqr_id_batched(cudaStream_t s, const std::vector<CPQRProb>& probs, double eps, int* d_k,
                     bool want_T) {
  if (probs.empty()) return;
  static std::once_flag attr_once;
  std::call_once(attr_once, [&] {
    RSF_CUDA(cudaFuncSetAttribute(cpqr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(SMEM_BUDGET + 24 * 1024)));
  });
  std::vector<CPQRDesc> dv;
  size_t smem_need = 0;
  for (size_t i = 0; i < probs.size(); ++i) {
    const CPQRProb& p = probs[i];
    CPQRDesc d;
    d.R = p.R; d.ldr = p.ldr; d.q = p.q; d.c = p.c;
    size_t hdr = (72 + p.c + ((size_t)p.c + 32 + 1) / 2 + 1) * sizeof(double);
    size_t wbytes = (size_t)p.q * p.c * sizeof(double);
    if (hdr + wbytes <= SMEM_BUDGET) {
      d.smem = 1; d.W = nullptr; d.ldw = p.q;
      smem_need = std::max(smem_need, hdr + wbytes);
    } else {
      RSF_REQUIRE(p.W != nullptr, ST_ECUDA, "cpqr: workspace required");
      RSF_REQUIRE(hdr <= SMEM_BUDGET + 16 * 1024, ST_EINVAL, "cpqr: block too wide");
      d.smem = 0; d.W = p.W; d.ldw = p.q;
      smem_need = std::max(smem_need, hdr);
    }
    d.T = p.T; d.piv = p.piv; d.kout = d_k + i;
    d.Rout = p.Rout; d.tau = p.tau;
    d.eps = eps; d.want_T = want_T ? 1 : 0;
    dv.push_back(d);
  }
  auto dd = upload_descs(dv, s);
  for (size_t o = 0; o < dv.size(); o += 65535) {
    unsigned nb = (unsigned)std::min<size_t>(65535, dv.size() - o);
    cpqr_kernel<<<nb, NT, smem_need, s>>>(dd.p + o);
    count_launch();
    RSF_LAUNCH_CHECK();
  }
}

// ------------------------------------------------------------------ potrf (+ inverse)
void potrf_batched(cudaStream_t s, const std::vector<PotrfProb>& probs, double* d_logsum, int* d_info) {
  if (probs.empty()) return;
  static std::once_flag attr_once;
  std::call_once(attr_once, [&] {
    RSF_CUDA(cudaFuncSetAttribute(potrf_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(2 * CH_NB * CH_NB * sizeof(double))));
  });
  const int P = (int)probs.size();
  RSF_CUDA(cudaMemsetAsync(d_logsum, 0, P * sizeof(double), s));
  RSF_CUDA(cudaMemsetAsync(d_info, 0, P * sizeof(int), s));
  int maxn = 0;
  std::vector<long long> woff(P);
  long long wtot = 0;
  for (int i = 0; i < P; ++i) {
    maxn = std::max(maxn, probs[i].n);
    woff[i] = wtot;
    wtot += (long long)CH_NB * probs[i].n;
  }
  if (maxn == 0) return;
  DBuf<double> Dinv((size_t)P * CH_NB * CH_NB, s), Wb(wtot, s);
  {  // Linv starts at zero (upper triangle and not-yet-written blocks)
    std::vector<ZDesc> z;
    long long mx = 0;
    for (auto& p : probs)
      if (p.Linv && p.n) { z.push_back(ZDesc{p.Linv, p.ldi, p.n}); mx = std::max(mx, (long long)p.n * p.n); }
    launch_y(s, z, mx, zero_all_kernel);
  }
  for (int j0 = 0; j0 < maxn; j0 += CH_NB) {
    std::vector<DiagDesc> dd;
    std::vector<CopyProb> cp;
    GemmBatch gp(false, true), gt(false, true);
    for (int i = 0; i < P; ++i) {
      const PotrfProb& p = probs[i];
      if (p.n <= j0) continue;
      const int nb = std::min(CH_NB, p.n - j0);
      DiagDesc d;
      d.A = p.A + j0 * p.lda + j0; d.lda = p.lda; d.nb = nb;
      d.Dinv = Dinv.p + (long long)i * CH_NB * CH_NB;
      d.Linv = p.Linv ? p.Linv + j0 * p.ldi + j0 : nullptr; d.ldi = p.ldi;
      d.logsum = d_logsum + i; d.info = d_info + i; d.col0 = j0;
      dd.push_back(d);
      const int j1 = j0 + nb, r = p.n - j1;
      if (r > 0) {
        GemmDesc a = gdesc(r, nb, nb);            // W = A21 Dinv^T
        a.A = p.A + j0 * p.lda + j1; a.lda = (int)p.lda;
        a.B = d.Dinv; a.ldb = CH_NB;
        a.C = Wb.p + woff[i]; a.ldc = r;
        gp.add(a);
        cp.push_back(CopyProb{Wb.p + woff[i], r, p.A + j0 * p.lda + j1, p.lda, r, nb, 1.0});
        GemmDesc t = gdesc(r, r, nb);             // A22 -= L21 L21^T (lower tiles)
        t.A = p.A + j0 * p.lda + j1; t.lda = (int)p.lda;
        t.B = p.A + j0 * p.lda + j1; t.ldb = (int)p.lda;
        t.C = p.A + j1 * p.lda + j1; t.ldc = (int)p.lda;
        t.alpha = -1.0; t.beta = 1.0; t.lower = 1;
        gt.add(t);
      }
    }
    if (dd.empty()) continue;
    auto ddev = upload_descs(dd, s);
    for (size_t o = 0; o < dd.size(); o += 65535) {
      unsigned nb = (unsigned)std::min<size_t>(65535, dd.size() - o);
      potrf_diag_kernel<<<nb, NT, 2 * CH_NB * CH_NB * sizeof(double), s>>>(ddev.p + o);
      count_launch();
      RSF_LAUNCH_CHECK();
    }
    gp.run(s);
    copy_batched(s, cp);
    gt.run(s);
  }
  // zero the strict upper triangle (the SYRK tiles straddle the diagonal)
  std::vector<ZDesc> zd;
  long long mx = 0;
  for (auto& p : probs)
    if (p.n > 0) { zd.push_back(ZDesc{p.A, p.lda, p.n}); mx = std::max(mx, (long long)p.n * p.n); }
  launch_y(s, zd, mx, zero_upper_kernel);
  // explicit inverse: block rows  X(r0:, 0:r0) = -Dinv_rr * (L(r0:, 0:r0) X(0:r0, 0:r0))
  bool want_inv = false;
  for (auto& p : probs) want_inv |= (p.Linv != nullptr);
  if (!want_inv) return;
  static const bool rec_inv = !(getenv("RSF_TRINV_REC") && getenv("RSF_TRINV_REC")[0] == '0');
  if (rec_inv) {
    // Linv holds the inverses of the CH_NB x CH_NB diagonal blocks (potrf_diag_kernel).  Merge
    // neighbouring inverted diagonal blocks of size sb into blocks of size 2 sb, all problems and
    // all pairs of a size in one batch (2 GEMMs + 1 zeroing launch per doubling instead of 2 GEMMs
    // per 64-row block row):
    //   [L11 0; L21 L22]^-1 = [X11 0; -X22 L21 X11  X22]
    // T^T = (L21 X11)^T = X11^T L21^T is parked in the (zero) strict upper triangle at rows of
    // block 1, columns of block 2, then X21 = -X22 (T^T)^T, then the parked block is zeroed
    // again (the next doubling reads X11 / X22 as full blocks with zero upper triangles).
    for (int sb = CH_NB; sb < maxn; sb *= 2) {
      GemmBatch g1(true, true), g2(false, true);
      std::vector<RDesc> zr;
      long long mz = 0;
      for (int i = 0; i < P; ++i) {
        const PotrfProb& p = probs[i];
        if (!p.Linv) continue;
        for (int a = 0; a + sb < p.n; a += 2 * sb) {
          const int b = a + sb, s2 = std::min(sb, p.n - b);
          double* Tt = p.Linv + (long long)b * p.ldi + a;        // sb x s2 (upper triangle)
          GemmDesc d1 = gdesc(sb, s2, sb);                        // T^T = X11^T L21^T
          d1.A = p.Linv + (long long)a * p.ldi + a; d1.lda = (int)p.ldi;
          d1.B = p.A + (long long)a * p.lda + b; d1.ldb = (int)p.lda;
          d1.C = Tt; d1.ldc = (int)p.ldi;
          g1.add(d1);
          GemmDesc d2 = gdesc(s2, sb, s2);                        // X21 = -X22 T
          d2.A = p.Linv + (long long)b * p.ldi + b; d2.lda = (int)p.ldi;
          d2.B = Tt; d2.ldb = (int)p.ldi;
          d2.C = p.Linv + (long long)a * p.ldi + b; d2.ldc = (int)p.ldi;
          d2.alpha = -1.0;
          g2.add(d2);
          zr.push_back(RDesc{Tt, p.ldi, sb, s2});
          mz = std::max(mz, (long long)sb * s2);
        }
      }
      g1.run(s);
      g2.run(s);
      launch_y(s, zr, mz, zero_rect_kernel);
    }
    return;
  }
  DBuf<double> tmp(wtot, s);
  for (int r0 = CH_NB; r0 < maxn; r0 += CH_NB) {
    GemmBatch g1(false, false), g2(false, false);
    for (int i = 0; i < P; ++i) {
      const PotrfProb& p = probs[i];
      if (!p.Linv || p.n <= r0) continue;
      const int rb = std::min(CH_NB, p.n - r0);
      GemmDesc a = gdesc(rb, r0, r0);
      a.A = p.A + r0; a.lda = (int)p.lda;
      a.B = p.Linv; a.ldb = (int)p.ldi;
      a.C = tmp.p + woff[i]; a.ldc = rb;
      g1.add(a);
      GemmDesc b = gdesc(rb, r0, rb);
      b.A = p.Linv + r0 * p.ldi + r0; b.lda = (int)p.ldi;
      b.B = tmp.p + woff[i]; b.ldb = rb;
      b.C = p.Linv + r0; b.ldc = (int)p.ldi;
      b.alpha = -1.0;
      g2.add(b);
    }
    g1.run(s);
    g2.run(s);
  }
}

}  // namespace rsf

// Fused small-box level sweeps (see sweep.cuh).
#include "sweep.cuh"
#include <mutex>

namespace rsf {

namespace {

constexpr int NT = 256;

// out[j][rho] = alpha * sum_kk in[kk][rho] * M(kk, j) + beta * out[j][rho]   for j < N, rho < KC
// (slab layout [column][rho], ld KC).  M(kk, j) = Mat[kk + j * ldm] (TR = false) or
// Mat[j + kk * ldm] (TR = true); Mat is read through the read-only cache (every CTA of a
// box reads the same matrix).
template <int KC, bool TR>
__device__ __forceinline__ void slab_mm(double* __restrict__ out, const double* __restrict__ in, int K, int N,
                                        const double* __restrict__ Mat, int ldm, double alpha, double beta) {
  constexpr int G = NT / KC;   // column groups
  const int rho = threadIdx.x % KC, cg = threadIdx.x / KC;
  for (int j0 = cg; j0 < N; j0 += 4 * G) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int jj[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) jj[u] = min(j0 + u * G, N - 1);
    for (int kk = 0; kk < K; ++kk) {
      const double x = in[kk * KC + rho];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double m = TR ? __ldg(Mat + jj[u] + (long long)kk * ldm) : __ldg(Mat + kk + (long long)jj[u] * ldm);
        acc[u] = fma(x, m, acc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + u * G;
      if (j < N) {
        double* o = out + j * KC + rho;
        *o = (beta == 0.0) ? alpha * acc[u] : fma(beta, *o, alpha * acc[u]);
      }
    }
  }
}

// KC = 32, register-blocked: thread (rp, cg) with rp = tid % 16, cg = tid / 16 owns the outputs
// (j, rho) for rho in {rp, rp + 16} and j = cg + 16 u, u < 4: per K step 2 shared loads + 4
// (warp-pairwise uniform) matrix loads feed 8 FMAs (slab_mm: 1 + 4 loads for 4 FMAs)
template <bool TR>
__device__ __forceinline__ void slab_mm32(double* __restrict__ out, const double* __restrict__ in, int K, int N,
                                          const double* __restrict__ Mat, int ldm, double alpha, double beta) {
  constexpr int KC = 32;
  const int rp = threadIdx.x & 15, cg = threadIdx.x >> 4;   // 16 x 16
  for (int j0 = cg; j0 < N; j0 += 64) {
    double a0[4] = {0.0, 0.0, 0.0, 0.0}, a1[4] = {0.0, 0.0, 0.0, 0.0};
    int jj[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) jj[u] = min(j0 + 16 * u, N - 1);
    for (int kk = 0; kk < K; ++kk) {
      const double x0 = in[kk * KC + rp], x1 = in[kk * KC + rp + 16];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double m = TR ? __ldg(Mat + jj[u] + (long long)kk * ldm) : __ldg(Mat + kk + (long long)jj[u] * ldm);
        a0[u] = fma(x0, m, a0[u]);
        a1[u] = fma(x1, m, a1[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + 16 * u;
      if (j < N) {
        double* o0 = out + j * KC + rp;
        double* o1 = o0 + 16;
        *o0 = (beta == 0.0) ? alpha * a0[u] : fma(beta, *o0, alpha * a0[u]);
        *o1 = (beta == 0.0) ? alpha * a1[u] : fma(beta, *o1, alpha * a1[u]);
      }
    }
  }
}

template <int KC, bool TR>
__device__ __forceinline__ void slab_mm_any(double* __restrict__ out, const double* __restrict__ in, int K, int N,
                                            const double* __restrict__ Mat, int ldm, double alpha, double beta) {
  if constexpr (KC == 32) slab_mm32<TR>(out, in, K, N, Mat, ldm, alpha, beta);
  else slab_mm<KC, TR>(out, in, K, N, Mat, ldm, alpha, beta);
}

template <int KC>
__device__ __forceinline__ void load_cols(double* __restrict__ dst, const double* __restrict__ X, const int* __restrict__ idx,
                                          int cnt, int ldx, int r0, int k) {
  for (int e = threadIdx.x; e < cnt * KC; e += NT) {
    const int a = e / KC, rho = e % KC;
    dst[e] = (r0 + rho < k) ? X[(long long)__ldg(idx + a) * ldx + r0 + rho] : 0.0;
  }
}

template <int KC>
__device__ __forceinline__ void store_cols(const double* __restrict__ src, double* __restrict__ X, const int* __restrict__ idx,
                                           int cnt, int ldx, int r0, int k) {
  for (int e = threadIdx.x; e < cnt * KC; e += NT) {
    const int a = e / KC, rho = e % KC;
    if (r0 + rho < k) X[(long long)__ldg(idx + a) * ldx + r0 + rho] = src[e];
  }
}

template <int KC>
__global__ void __launch_bounds__(NT) sweep_kernel(const BoxOp* __restrict__ ops, int kind, double* X0, double* X1,
                                                   int k) {
  extern __shared__ double sm[];
  const BoxOp op = ops[blockIdx.x];
  const int kb = op.kb, r = op.r, r0 = blockIdx.y * KC;
  double* xs = sm;                    // kb x KC
  double* xr = sm + kb * KC;          // r x KC
  double* yr = xr + r * KC;           // r x KC
  if (kind == SW_SOLVE_FWD || kind == SW_SOLVE_BWD) {
    load_cols<KC>(xs, X0, op.S, kb, k, r0, k);
    load_cols<KC>(xr, X0, op.R, r, k, r0, k);
    __syncthreads();
    if (kind == SW_SOLVE_FWD) {
      if (kb) slab_mm_any<KC, false>(xr, xs, kb, r, op.T, kb, -1.0, 1.0);   // x_R -= T^T x_S
      __syncthreads();
      slab_mm_any<KC, true>(yr, xr, r, r, op.L, r, 1.0, 0.0);               // y_R = L^-1 x_R
      __syncthreads();
      if (kb) slab_mm_any<KC, true>(xs, yr, r, kb, op.E, kb, -1.0, 1.0);    // x_S -= E y_R
    } else {
      if (kb) slab_mm_any<KC, false>(xr, xs, kb, r, op.E, kb, -1.0, 1.0);   // x_R -= E^T x_S
      __syncthreads();
      slab_mm_any<KC, false>(yr, xr, r, r, op.L, r, 1.0, 0.0);              // y_R = L^-T x_R
      __syncthreads();
      if (kb) slab_mm_any<KC, true>(xs, yr, r, kb, op.T, kb, -1.0, 1.0);    // x_S -= T y_R
    }
    __syncthreads();
    store_cols<KC>(xs, X0, op.S, kb, k, r0, k);
    store_cols<KC>(yr, X0, op.R, r, k, r0, k);
  } else if (kind == SW_AO_UP) {
    load_cols<KC>(xs, X0, op.S, kb, k, r0, k);
    load_cols<KC>(xr, X0, op.R, r, k, r0, k);
    __syncthreads();
    if (kb) slab_mm_any<KC, true>(xs, xr, r, kb, op.T, kb, 1.0, 1.0);       // x_S += T x_R
    __syncthreads();
    if (kb) slab_mm_any<KC, false>(yr, xs, kb, r, op.E, kb, 1.0, 0.0);      // y_R = X_SR^T x_S
    slab_mm_any<KC, false>(yr, xr, r, r, op.L, r, 1.0, kb ? 1.0 : 0.0);     //     + X_RR x_R (same thread owns y_R(j, rho))
    __syncthreads();
    store_cols<KC>(xs, X0, op.S, kb, k, r0, k);
    store_cols<KC>(yr, X1, op.R, r, k, r0, k);
  } else {   // SW_AO_DN: xs holds y_S, xr holds x_R, yr holds y_R
    load_cols<KC>(xs, X1, op.S, kb, k, r0, k);
    load_cols<KC>(xr, X0, op.R, r, k, r0, k);
    load_cols<KC>(yr, X1, op.R, r, k, r0, k);
    __syncthreads();
    if (kb) slab_mm_any<KC, true>(xs, xr, r, kb, op.E, kb, 1.0, 1.0);       // y_S += X_SR x_R
    __syncthreads();
    if (kb) slab_mm_any<KC, false>(yr, xs, kb, r, op.T, kb, 1.0, 1.0);      // y_R += T^T y_S
    __syncthreads();
    store_cols<KC>(xs, X1, op.S, kb, k, r0, k);
    store_cols<KC>(yr, X1, op.R, r, k, r0, k);
  }
}

// DMMA.8x8x4 version of slab_mm: C (rho x j) = A (rho x kk) B (kk x j) with A(rho, kk) =
// in[kk][rho] (shared memory) and B(kk, j) = M(kk, j) (global, read-only path).  Warp w owns
// the N-tiles w, w + 8, ... (8 columns each) for all KC/8 row tiles, two N-tiles at a time; the
// element (rho, j) of out is always written by the same thread (lane layout of the DMMA
// accumulator), so consecutive calls on the same out need no barrier.
template <int KC, bool TR>
__device__ __forceinline__ void slab_mm_mma(double* __restrict__ out, const double* __restrict__ in, int K, int N,
                                            const double* __restrict__ Mat, int ldm, double alpha, double beta) {
  constexpr int MT = KC / 8, NW = NT / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int ntiles = (N + 7) / 8;
  for (int nt0 = warp; nt0 < ntiles; nt0 += 2 * NW) {
    const int nt1 = nt0 + NW;
    const bool has1 = nt1 < ntiles;
    double acc[2][MT][2];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int m = 0; m < MT; ++m) { acc[u][m][0] = 0.0; acc[u][m][1] = 0.0; }
    const int jb0 = nt0 * 8 + g, jb1 = nt1 * 8 + g;
    auto ldb = [&](int kk, int jb) -> double {
      if (kk >= K || jb >= N) return 0.0;
      return TR ? __ldg(Mat + jb + (long long)kk * ldm) : __ldg(Mat + kk + (long long)jb * ldm);
    };
    // B fragments of the next k-step are fetched before the MMAs of this one (global latency)
    double nb0 = ldb(tq, jb0), nb1 = has1 ? ldb(tq, jb1) : 0.0;
    for (int k0 = 0; k0 < K; k0 += 4) {
      const int kk = k0 + tq;
      const bool kv = kk < K;
      double a[MT];
#pragma unroll
      for (int m = 0; m < MT; ++m) a[m] = kv ? in[kk * KC + m * 8 + g] : 0.0;
      const double b0 = nb0, b1 = nb1;
      nb0 = ldb(kk + 4, jb0);
      nb1 = has1 ? ldb(kk + 4, jb1) : 0.0;
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[0][m][0]), "+d"(acc[0][m][1]) : "d"(a[m]), "d"(b0));
        if (has1)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc[1][m][0]), "+d"(acc[1][m][1]) : "d"(a[m]), "d"(b1));
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (u == 1 && !has1) break;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = (u ? nt1 : nt0) * 8 + 2 * tq + h;
        if (j >= N) continue;
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          double* o = out + j * KC + m * 8 + g;
          *o = (beta == 0.0) ? alpha * acc[u][m][h] : fma(beta, *o, alpha * acc[u][m][h]);
        }
      }
    }
  }
}

template <int KC>
__global__ void __launch_bounds__(NT) sweep_mma_kernel(const BoxOp* __restrict__ ops, int kind, double* X0, double* X1,
                                                       int k) {
  extern __shared__ double sm[];
  const BoxOp op = ops[blockIdx.x];
  const int kb = op.kb, r = op.r, r0 = blockIdx.y * KC;
  double* xs = sm;
  double* xr = sm + kb * KC;
  double* yr = xr + r * KC;
  if (kind == SW_SOLVE_FWD || kind == SW_SOLVE_BWD) {
    load_cols<KC>(xs, X0, op.S, kb, k, r0, k);
    load_cols<KC>(xr, X0, op.R, r, k, r0, k);
    __syncthreads();
    if (kind == SW_SOLVE_FWD) {
      if (kb) slab_mm_mma<KC, false>(xr, xs, kb, r, op.T, kb, -1.0, 1.0);
      __syncthreads();
      slab_mm_mma<KC, true>(yr, xr, r, r, op.L, r, 1.0, 0.0);
      __syncthreads();
      if (kb) slab_mm_mma<KC, true>(xs, yr, r, kb, op.E, kb, -1.0, 1.0);
    } else {
      if (kb) slab_mm_mma<KC, false>(xr, xs, kb, r, op.E, kb, -1.0, 1.0);
      __syncthreads();
      slab_mm_mma<KC, false>(yr, xr, r, r, op.L, r, 1.0, 0.0);
      __syncthreads();
      if (kb) slab_mm_mma<KC, true>(xs, yr, r, kb, op.T, kb, -1.0, 1.0);
    }
    __syncthreads();
    store_cols<KC>(xs, X0, op.S, kb, k, r0, k);
    store_cols<KC>(yr, X0, op.R, r, k, r0, k);
  } else if (kind == SW_AO_UP) {
    load_cols<KC>(xs, X0, op.S, kb, k, r0, k);
    load_cols<KC>(xr, X0, op.R, r, k, r0, k);
    __syncthreads();
    if (kb) slab_mm_mma<KC, true>(xs, xr, r, kb, op.T, kb, 1.0, 1.0);
    __syncthreads();
    if (kb) slab_mm_mma<KC, false>(yr, xs, kb, r, op.E, kb, 1.0, 0.0);
    slab_mm_mma<KC, false>(yr, xr, r, r, op.L, r, 1.0, kb ? 1.0 : 0.0);
    __syncthreads();
    store_cols<KC>(xs, X0, op.S, kb, k, r0, k);
    store_cols<KC>(yr, X1, op.R, r, k, r0, k);
  } else {
    load_cols<KC>(xs, X1, op.S, kb, k, r0, k);
    load_cols<KC>(xr, X0, op.R, r, k, r0, k);
    load_cols<KC>(yr, X1, op.R, r, k, r0, k);
    __syncthreads();
    if (kb) slab_mm_mma<KC, true>(xs, xr, r, kb, op.E, kb, 1.0, 1.0);
    __syncthreads();
    if (kb) slab_mm_mma<KC, false>(yr, xs, kb, r, op.T, kb, 1.0, 1.0);
    __syncthreads();
    store_cols<KC>(xs, X1, op.S, kb, k, r0, k);
    store_cols<KC>(yr, X1, op.R, r, k, r0, k);
  }
}

// One right-hand side (k = 1): the box's x_S, x_R live in shared memory as plain vectors and
// every step is a GEMV laid out for coalesced reads of the box matrix (the 1-RHS sweep is
// bound by streaming T, L, E from HBM):
//   TR = false, out[j] = sum_kk in[kk] Mat[kk + j ldm]: a warp per output j, lanes over kk;
//   TR = true,  out[j] = sum_kk in[kk] Mat[j + kk ldm]: a thread per output j, loop over kk.
constexpr int NT1 = 128;
template <bool TR>
__device__ __forceinline__ void vec_mv(double* __restrict__ out, const double* __restrict__ in, int K, int N,
                                       const double* __restrict__ Mat, int ldm, double alpha, double beta) {
  if (!TR) {
    // a warp per 4 output columns, lanes over kk: 4 (x 2 unrolled) independent loads in flight
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j0 = 4 * warp; j0 < N; j0 += 4 * (NT1 / 32)) {
      const double* m[4];
      bool ok[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { ok[u] = j0 + u < N; m[u] = Mat + (long long)(ok[u] ? j0 + u : j0) * ldm; }
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      int kk = lane;
      for (; kk + 32 < K; kk += 64) {
        const double x0 = in[kk], x1 = in[kk + 32];
        double v[4], w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { v[u] = ok[u] ? __ldg(m[u] + kk) : 0.0; w[u] = ok[u] ? __ldg(m[u] + kk + 32) : 0.0; }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] = fma(x1, w[u], fma(x0, v[u], acc[u]));
      }
      for (; kk < K; kk += 32) {
        const double x0 = in[kk];
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] = fma(x0, ok[u] ? __ldg(m[u] + kk) : 0.0, acc[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        double a = acc[u];
#pragma unroll
        for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0 && ok[u]) out[j0 + u] = (beta == 0.0) ? alpha * a : fma(beta, out[j0 + u], alpha * a);
      }
    }
  } else {
    // a thread per output j (coalesced across the warp), 8 rows kk in flight
    for (int j = threadIdx.x; j < N; j += NT1) {
      double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      int kk = 0;
      for (; kk + 8 <= K; kk += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(Mat + j + (long long)(kk + u) * ldm);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] = fma(in[kk + u], v[u], acc[u]);
      }
      for (; kk < K; ++kk) acc[0] = fma(in[kk], __ldg(Mat + j + (long long)kk * ldm), acc[0]);
      const double a = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
      out[j] = (beta == 0.0) ? alpha * a : fma(beta, out[j], alpha * a);
    }
  }
}

__device__ __forceinline__ void load_vec(double* __restrict__ dst, const double* __restrict__ X, const int* __restrict__ idx,
                                         int cnt) {
  for (int e = threadIdx.x; e < cnt; e += NT1) dst[e] = X[__ldg(idx + e)];
}
__device__ __forceinline__ void store_vec(const double* __restrict__ src, double* __restrict__ X, const int* __restrict__ idx,
                                          int cnt) {
  for (int e = threadIdx.x; e < cnt; e += NT1) X[__ldg(idx + e)] = src[e];
}

__global__ void __launch_bounds__(NT1) sweep1_kernel(const BoxOp* __restrict__ ops, int kind, double* X0, double* X1) {
  extern __shared__ double sm[];
  const BoxOp op = ops[blockIdx.x];
  const int kb = op.kb, r = op.r;
  double* xs = sm;
  double* xr = sm + kb;
  double* yr = xr + r;
  if (kind == SW_SOLVE_FWD || kind == SW_SOLVE_BWD) {
    load_vec(xs, X0, op.S, kb);
    load_vec(xr, X0, op.R, r);
    __syncthreads();
    if (kind == SW_SOLVE_FWD) {
      if (kb) vec_mv<false>(xr, xs, kb, r, op.T, kb, -1.0, 1.0);   // x_R -= T^T x_S
      __syncthreads();
      vec_mv<true>(yr, xr, r, r, op.L, r, 1.0, 0.0);               // y_R = L^-1 x_R
      __syncthreads();
      if (kb) vec_mv<true>(xs, yr, r, kb, op.E, kb, -1.0, 1.0);    // x_S -= E y_R
    } else {
      if (kb) vec_mv<false>(xr, xs, kb, r, op.E, kb, -1.0, 1.0);   // x_R -= E^T x_S
      __syncthreads();
      vec_mv<false>(yr, xr, r, r, op.L, r, 1.0, 0.0);              // y_R = L^-T x_R
      __syncthreads();
      if (kb) vec_mv<true>(xs, yr, r, kb, op.T, kb, -1.0, 1.0);    // x_S -= T y_R
    }
    __syncthreads();
    store_vec(xs, X0, op.S, kb);
    store_vec(yr, X0, op.R, r);
  } else if (kind == SW_AO_UP) {
    load_vec(xs, X0, op.S, kb);
    load_vec(xr, X0, op.R, r);
    __syncthreads();
    if (kb) vec_mv<true>(xs, xr, r, kb, op.T, kb, 1.0, 1.0);       // x_S += T x_R
    __syncthreads();
    if (kb) vec_mv<false>(yr, xs, kb, r, op.E, kb, 1.0, 0.0);      // y_R = X_SR^T x_S
    __syncthreads();
    vec_mv<false>(yr, xr, r, r, op.L, r, 1.0, kb ? 1.0 : 0.0);     //     + X_RR x_R
    __syncthreads();
    store_vec(xs, X0, op.S, kb);
    store_vec(yr, X1, op.R, r);
  } else {   // SW_AO_DN: xs holds y_S, xr holds x_R, yr holds y_R
    load_vec(xs, X1, op.S, kb);
    load_vec(xr, X0, op.R, r);
    load_vec(yr, X1, op.R, r);
    __syncthreads();
    if (kb) vec_mv<true>(xs, xr, r, kb, op.E, kb, 1.0, 1.0);       // y_S += X_SR x_R
    __syncthreads();
    if (kb) vec_mv<false>(yr, xs, kb, r, op.T, kb, 1.0, 1.0);      // y_R += T^T y_S
    __syncthreads();
    store_vec(xs, X1, op.S, kb);
    store_vec(yr, X1, op.R, r);
  }
}

bool sweep_mma_on() {
  static const bool on = getenv("RSF_SWEEP_MMA") && getenv("RSF_SWEEP_MMA")[0] == '1';
  return on;
}

}  // namespace

int sweep_max_i() { return sweep_mma_on() ? SWEEP_MAX_I_MMA : SWEEP_MAX_I; }

void sweep_level(cudaStream_t s, const BoxOp* d_ops, int nops, int max_i, SweepKind kind, double* X0, double* X1,
                 int k) {
  if (nops == 0 || k <= 0) return;
  RSF_REQUIRE(max_i <= (k == 1 ? SWEEP1_MAX_I : sweep_max_i()), ST_EINVAL,
              "sweep_level: box too large for the fused kernel");
  static std::once_flag attr_once;
  std::call_once(attr_once, [&] {
    RSF_CUDA(cudaFuncSetAttribute(sweep_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    RSF_CUDA(cudaFuncSetAttribute(sweep_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    RSF_CUDA(cudaFuncSetAttribute(sweep_mma_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    RSF_CUDA(cudaFuncSetAttribute(sweep_mma_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  });
  static const bool k1_on = !(getenv("RSF_SWEEP1") && getenv("RSF_SWEEP1")[0] == '0');
  if (k == 1 && k1_on) {   // one right-hand side: GEMV steps (HBM stream of the box matrices)
    const size_t smem = (size_t)2 * max_i * sizeof(double);
    for (int o = 0; o < nops; o += 65535) {
      const unsigned nb = (unsigned)std::min(65535, nops - o);
      sweep1_kernel<<<nb, NT1, smem, s>>>(d_ops + o, (int)kind, X0, X1);
      count_launch();
    }
    RSF_LAUNCH_CHECK();
    return;
  }
  // shared memory: (kb + 2 r) * KC doubles <= 2 |I| * KC
  const int KC = (max_i <= 128) ? 32 : 16;
  const size_t smem = (size_t)2 * max_i * KC * sizeof(double);
  const unsigned gy = (unsigned)((k + KC - 1) / KC);
  const bool mma = sweep_mma_on();
  for (int o = 0; o < nops; o += 65535) {
    const unsigned nb = (unsigned)std::min(65535, nops - o);
    if (mma) {
      if (KC == 32) sweep_mma_kernel<32><<<dim3(nb, gy), NT, smem, s>>>(d_ops + o, (int)kind, X0, X1, k);
      else sweep_mma_kernel<16><<<dim3(nb, gy), NT, smem, s>>>(d_ops + o, (int)kind, X0, X1, k);
    } else {
      if (KC == 32) sweep_kernel<32><<<dim3(nb, gy), NT, smem, s>>>(d_ops + o, (int)kind, X0, X1, k);
      else sweep_kernel<16><<<dim3(nb, gy), NT, smem, s>>>(d_ops + o, (int)kind, X0, X1, k);
    }
    count_launch();
  }
  RSF_LAUNCH_CHECK();
}

}  // namespace rsf

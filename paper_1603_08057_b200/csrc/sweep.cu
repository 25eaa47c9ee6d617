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
      if (kb) slab_mm<KC, false>(xr, xs, kb, r, op.T, kb, -1.0, 1.0);   // x_R -= T^T x_S
      __syncthreads();
      slab_mm<KC, true>(yr, xr, r, r, op.L, r, 1.0, 0.0);               // y_R = L^-1 x_R
      __syncthreads();
      if (kb) slab_mm<KC, true>(xs, yr, r, kb, op.E, kb, -1.0, 1.0);    // x_S -= E y_R
    } else {
      if (kb) slab_mm<KC, false>(xr, xs, kb, r, op.E, kb, -1.0, 1.0);   // x_R -= E^T x_S
      __syncthreads();
      slab_mm<KC, false>(yr, xr, r, r, op.L, r, 1.0, 0.0);              // y_R = L^-T x_R
      __syncthreads();
      if (kb) slab_mm<KC, true>(xs, yr, r, kb, op.T, kb, -1.0, 1.0);    // x_S -= T y_R
    }
    __syncthreads();
    store_cols<KC>(xs, X0, op.S, kb, k, r0, k);
    store_cols<KC>(yr, X0, op.R, r, k, r0, k);
  } else if (kind == SW_AO_UP) {
    load_cols<KC>(xs, X0, op.S, kb, k, r0, k);
    load_cols<KC>(xr, X0, op.R, r, k, r0, k);
    __syncthreads();
    if (kb) slab_mm<KC, true>(xs, xr, r, kb, op.T, kb, 1.0, 1.0);       // x_S += T x_R
    __syncthreads();
    if (kb) slab_mm<KC, false>(yr, xs, kb, r, op.E, kb, 1.0, 0.0);      // y_R = X_SR^T x_S
    slab_mm<KC, false>(yr, xr, r, r, op.L, r, 1.0, kb ? 1.0 : 0.0);     //     + X_RR x_R (same thread owns y_R(j, rho))
    __syncthreads();
    store_cols<KC>(xs, X0, op.S, kb, k, r0, k);
    store_cols<KC>(yr, X1, op.R, r, k, r0, k);
  } else {   // SW_AO_DN: xs holds y_S, xr holds x_R, yr holds y_R
    load_cols<KC>(xs, X1, op.S, kb, k, r0, k);
    load_cols<KC>(xr, X0, op.R, r, k, r0, k);
    load_cols<KC>(yr, X1, op.R, r, k, r0, k);
    __syncthreads();
    if (kb) slab_mm<KC, true>(xs, xr, r, kb, op.E, kb, 1.0, 1.0);       // y_S += X_SR x_R
    __syncthreads();
    if (kb) slab_mm<KC, false>(yr, xs, kb, r, op.T, kb, 1.0, 1.0);      // y_R += T^T y_S
    __syncthreads();
    store_cols<KC>(xs, X1, op.S, kb, k, r0, k);
    store_cols<KC>(yr, X1, op.R, r, k, r0, k);
  }
}

}  // namespace

void sweep_level(cudaStream_t s, const BoxOp* d_ops, int nops, int max_i, SweepKind kind, double* X0, double* X1,
                 int k) {
  if (nops == 0 || k <= 0) return;
  RSF_REQUIRE(max_i <= SWEEP_MAX_I, ST_EINVAL, "sweep_level: box too large for the fused kernel");
  static std::once_flag attr_once;
  std::call_once(attr_once, [&] {
    RSF_CUDA(cudaFuncSetAttribute(sweep_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    RSF_CUDA(cudaFuncSetAttribute(sweep_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  });
  // shared memory: (kb + 2 r) * KC doubles <= 2 |I| * KC
  const int KC = (max_i <= 128) ? 32 : 16;
  const size_t smem = (size_t)2 * max_i * KC * sizeof(double);
  const unsigned gy = (unsigned)((k + KC - 1) / KC);
  for (int o = 0; o < nops; o += 65535) {
    const unsigned nb = (unsigned)std::min(65535, nops - o);
    if (KC == 32) sweep_kernel<32><<<dim3(nb, gy), NT, smem, s>>>(d_ops + o, (int)kind, X0, X1, k);
    else sweep_kernel<16><<<dim3(nb, gy), NT, smem, s>>>(d_ops + o, (int)kind, X0, X1, k);
    count_launch();
  }
  RSF_LAUNCH_CHECK();
}

}  // namespace rsf

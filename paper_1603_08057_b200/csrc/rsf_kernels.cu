// Element kernels of the factorization (see rsf_kernels.cuh).
#include <algorithm>

#include "rsf_kernels.cuh"

namespace rsf {

namespace {

constexpr int NT = 256;

template <class D>
DBuf<D> up(const std::vector<D>& v, cudaStream_t s) {
  DBuf<D> b(v.size(), s);
  b.upload(v);
  return b;
}

__global__ void assemble_id_kernel(const IdAsmDesc* __restrict__ descs, KParams kp, int which,
                                   const double* __restrict__ xs, const double* __restrict__ ys,
                                   double rin, double rout, int nr, int na) {
  const IdAsmDesc d = descs[blockIdx.y];
  const int m = d.m_near + nr * na;
  const long long tot = (long long)m * d.c;
  const double two_pi = 6.283185307179586;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    const int r = (int)(e % m), j = (int)(e / m);
    const int cj = __ldg(d.I + j);
    const double xj = xs[cj], yj = ys[cj];
    double px, py;
    if (r < d.m_near) {
      const int ri = __ldg(d.near + r);
      px = xs[ri]; py = ys[ri];
    } else {
      const int q = r - d.m_near;
      const int ring = q / na, a = q - ring * na;
      const double rad = d.h * (rin + (rout - rin) * (ring + 0.5) / nr);
      double sn, cs;
      sincos(two_pi * a / na, &sn, &cs);
      px = d.cx + rad * cs; py = d.cy + rad * sn;
    }
    const double dx = px - xj, dy = py - yj;
    d.A[e] = entry_xy(kp, which, dx, dy, false);
  }
}

__global__ void assemble_self_kernel(const SelfAsmDesc* __restrict__ descs, KParams kp, int which,
                                     const double* __restrict__ xs, const double* __restrict__ ys) {
  const SelfAsmDesc& d = descs[blockIdx.y];
  const int c = d.c;
  const long long tot = (long long)c * c;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    const int i = (int)(e % c), j = (int)(e / c);
    double v;
    int ci = -1, cj = -1;
    if (d.nch > 0) {
      for (int q = 0; q < d.nch; ++q) {
        if (i >= d.choff[q] && i < d.choff[q + 1]) ci = q;
        if (j >= d.choff[q] && j < d.choff[q + 1]) cj = q;
      }
    }
    if (ci >= 0 && ci == cj) {
      v = d.chB[ci][(long long)(j - d.choff[ci]) * d.chld[ci] + (i - d.choff[ci])];
    } else {
      const int a = __ldg(d.I + i), b = __ldg(d.I + j);
      const double dx = xs[a] - xs[b], dy = ys[a] - ys[b];
      v = entry_xy(kp, which, dx, dy, a == b);
    }
    d.B[e] = v;
  }
}

__global__ void permute_kernel(const PermDesc* __restrict__ descs) {
  const PermDesc d = descs[blockIdx.y];
  const long long tot = (long long)d.c * d.c;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    const int i = (int)(e % d.c), j = (int)(e / d.c);
    d.Bp[e] = d.B[(long long)__ldg(d.piv + j) * d.c + __ldg(d.piv + i)];
  }
}

__global__ void symmetrize_kernel(const SymDesc* __restrict__ descs) {
  const SymDesc d = descs[blockIdx.y];
  const long long tot = (long long)d.n * d.n;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    const int i = (int)(e % d.n), j = (int)(e / d.n);
    if (i > j) {
      double a = d.A[j * d.lda + i], b = d.A[i * d.lda + j];
      double v = 0.5 * (a + b);
      d.A[j * d.lda + i] = v;
      d.A[i * d.lda + j] = v;
    }
  }
}

__global__ void colcopy_kernel(double* __restrict__ dst, const double* __restrict__ src, int ldx, int M,
                               const int* __restrict__ dmap, const int* __restrict__ smap, long long count,
                               double alpha, double beta) {
  const long long tot = count * M;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    const long long t = e / M;
    const int i = (int)(e - t * M);
    const long long dc = dmap ? dmap[t] : t;
    const long long sc = smap ? smap[t] : t;
    double v = alpha * src[sc * ldx + i];
    if (beta != 0.0) v += beta * dst[dc * ldx + i];
    dst[dc * ldx + i] = v;
  }
}

__global__ void to_internal_kernel(const double* __restrict__ b, long long ld, int k,
                                   const int* __restrict__ perm, int n, double* __restrict__ X) {
  const long long tot = (long long)n * k;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    const int t = (int)(e / k), j = (int)(e - (long long)t * k);
    X[e] = b[(long long)j * ld + perm[t]];
  }
}

__global__ void to_external_kernel(const double* __restrict__ X, int k, const int* __restrict__ perm, int n,
                                   double* __restrict__ b, long long ld) {
  const long long tot = (long long)n * k;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    const int t = (int)(e / k), j = (int)(e - (long long)t * k);
    b[(long long)j * ld + perm[t]] = X[e];
  }
}

int gx(long long maxelems) {
  long long g = (maxelems + NT - 1) / NT;
  return (int)std::max<long long>(1, std::min<long long>(g, 512));
}

template <class D, class K, class... Args>
void launch_y(cudaStream_t s, const std::vector<D>& v, long long maxelems, K kern, Args... args) {
  if (v.empty() || maxelems <= 0) return;
  auto d = ring_up(v, s);
  for (size_t o = 0; o < v.size(); o += 65535) {
    int ny = (int)std::min<size_t>(65535, v.size() - o);
    kern<<<dim3(gx(maxelems), ny), NT, 0, s>>>(d.p + o, args...);
    count_launch();
    RSF_LAUNCH_CHECK();
  }
}

}  // namespace

void assemble_id(cudaStream_t s, const std::vector<IdAsmDesc>& d, const KParams& kp, int which,
                 const Opts& o, const double* xs, const double* ys, int nr, int na) {
  long long mx = 0;
  for (auto& x : d) mx = std::max(mx, (long long)(x.m_near + nr * na) * x.c);
  launch_y(s, d, mx, assemble_id_kernel, kp, which, xs, ys, o.r_in, o.r_out, nr, na);
}

void assemble_self(cudaStream_t s, const std::vector<SelfAsmDesc>& d, const KParams& kp, int which,
                   const double* xs, const double* ys) {
  long long mx = 0;
  for (auto& x : d) mx = std::max(mx, (long long)x.c * x.c);
  launch_y(s, d, mx, assemble_self_kernel, kp, which, xs, ys);
}

void permute_sym(cudaStream_t s, const std::vector<PermDesc>& d) {
  long long mx = 0;
  for (auto& x : d) mx = std::max(mx, (long long)x.c * x.c);
  launch_y(s, d, mx, permute_kernel);
}

void symmetrize(cudaStream_t s, const std::vector<SymDesc>& d) {
  long long mx = 0;
  for (auto& x : d) mx = std::max(mx, (long long)x.n * x.n);
  launch_y(s, d, mx, symmetrize_kernel);
}

void colcopy(cudaStream_t s, double* dst, const double* src, int ldx, int M, const int* dmap,
             const int* smap, long long count, double alpha, double beta) {
  if (count <= 0 || M <= 0) return;
  colcopy_kernel<<<gx(count * M), NT, 0, s>>>(dst, src, ldx, M, dmap, smap, count, alpha, beta);
  count_launch();
  RSF_LAUNCH_CHECK();
}

void to_internal(cudaStream_t s, const Tree& t, const double* b, long long ld, int k, double* X) {
  to_internal_kernel<<<gx((long long)t.n * k), NT, 0, s>>>(b, ld, k, t.d_perm.p, t.n, X);
  count_launch();
  RSF_LAUNCH_CHECK();
}

void to_external(cudaStream_t s, const Tree& t, const double* X, int k, double* b, long long ld) {
  to_external_kernel<<<gx((long long)t.n * k), NT, 0, s>>>(X, k, t.d_perm.p, t.n, b, ld);
  count_launch();
  RSF_LAUNCH_CHECK();
}

}  // namespace rsf

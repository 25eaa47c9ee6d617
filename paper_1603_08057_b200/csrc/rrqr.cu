// Blocked randomized rank-revealing QR truncated at the eps-rank (see rrqr.cuh).
#include <algorithm>
#include <mutex>
#include <climits>
#include <cmath>

#include <cooperative_groups.h>

#include "rrqr.cuh"

namespace cg = cooperative_groups;

namespace rsf {

namespace {

constexpr int NT = 256;
constexpr int SP = QR_NB + 8;   // sketch rows (block + oversampling)

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ uint4 philox10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k.x += 0x9E3779B9u; k.y += 0xBB67AE85u; }
    const unsigned hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const unsigned hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

struct RDesc {
  double* A; long long lda; int m, c;
  double* G;       // SP x m
  double* Y;       // SP x c
  double* Z;       // SP x c scratch (sketch CPQR)
  double* zn;      // c scratch (sketch column norms)
  double* nrm2;    // c: squared trailing column norms
  int* piv;
  int* sw;         // QR_NB swap targets
  double* ref;     // max column norm
  int* flag;       // [0] done, [1] k
  double* R11i;    // QR_NB x QR_NB
  const double* ref_in;
  double* ref_out;
  int J, nbp, id;
  double eps;
};

// ref = max_j ||A(:, j)||, piv = identity.  Grid (column blocks, problems): warp per column,
// the squared norms combined with an integer atomicMax (the bit patterns of non-negative
// doubles order like the values); ref2 must be zero on entry.
__global__ void ref_norms_kernel(const RDesc* __restrict__ d0, unsigned long long* __restrict__ ref2) {
  const RDesc d = d0[blockIdx.y];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double mx = 0.0;
  for (int j = blockIdx.x * (NT / 32) + warp; j < d.c; j += gridDim.x * (NT / 32)) {
    const double* a = d.A + (long long)j * d.lda;
    double s = 0.0;
    for (int r = lane; r < d.m; r += 32) s += a[r] * a[r];
    mx = fmax(mx, wsum(s));
  }
  if (lane == 0 && mx > 0.0) atomicMax(ref2 + blockIdx.y, (unsigned long long)__double_as_longlong(mx));
  for (int j = blockIdx.x * NT + threadIdx.x; j < d.c; j += gridDim.x * NT) d.piv[j] = j;
}
// per problem: the reference scale and the "nothing to factor" flag
__global__ void ref_finish_kernel(const RDesc* __restrict__ d0, const unsigned long long* __restrict__ ref2, int P) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const RDesc d = d0[i];
  const double v = __longlong_as_double((long long)ref2[i]);
  if (d.ref_out) *d.ref_out = sqrt(v);
  const double rf = d.ref_in ? *d.ref_in : sqrt(v);
  *d.ref = rf;
  // nothing to factor: an all-zero matrix, or every column already below the absolute threshold
  d.flag[0] = (v > 0.0 && rf > 0.0 && sqrt(v) > d.eps * rf) ? 0 : 1;
  d.flag[1] = 0;
  d.flag[2] = 0;
}

__global__ void gauss_kernel(const RDesc* __restrict__ d0, unsigned seed) {
  const RDesc d = d0[blockIdx.y];
  const long long tot = (long long)SP * d.m;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    const int r = (int)(e % SP), col = (int)(e / SP);
    uint4 x = philox10(make_uint4((unsigned)d.id, (unsigned)r, (unsigned)col, 0x51u), make_uint2(seed, 4u));
    const double u1 = ((double)(x.x >> 5) * 67108864.0 + (double)(x.y >> 6)) * (1.0 / 9007199254740992.0);
    const double u2 = ((double)(x.z >> 5) * 67108864.0 + (double)(x.w >> 6)) * (1.0 / 9007199254740992.0);
    d.G[e] = sqrt(-2.0 * log1p(-u1)) * cos(6.283185307179586 * u2);
  }
}

// greedy CPQR of a copy of the sketch Y(:, J:c) for nbp steps -> swap list
__global__ void __launch_bounds__(NT) sketch_cpqr_kernel(const RDesc* __restrict__ d0) {
  const RDesc d = d0[blockIdx.x];
  const int J = d.J, cr = d.c - J, nbp = d.nbp;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  __shared__ double redv[NT / 32];
  __shared__ int redi[NT / 32];
  __shared__ double sc[4];
  __shared__ int sp;
  double* Z = d.Z;
  double* zn = d.zn;
  for (long long e = tid; e < (long long)SP * cr; e += NT) Z[e] = d.Y[(long long)J * SP + e];
  __syncthreads();
  for (int j = warp; j < cr; j += NT / 32) {
    double v = (lane < SP) ? Z[(long long)j * SP + lane] : 0.0;
    double s = v * v;
    if (lane + 32 < SP) { double w = Z[(long long)j * SP + lane + 32]; s += w * w; }
    s = wsum(s);
    if (lane == 0) zn[j] = s;
  }
  __syncthreads();
  for (int t = 0; t < nbp; ++t) {
    double bv = -1.0;
    int bi = cr;
    for (int j = t + tid; j < cr; j += NT) {
      const double v = zn[j];
      if (v > bv) { bv = v; bi = j; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { redv[warp] = bv; redi[warp] = bi; }
    __syncthreads();
    if (tid == 0) {
      double v = redv[0]; int b = redi[0];
      for (int w = 1; w < NT / 32; ++w)
        if (redv[w] > v || (redv[w] == v && redi[w] < b)) { v = redv[w]; b = redi[w]; }
      if (b >= cr) b = t;
      sp = b;
      d.sw[t] = b;
    }
    __syncthreads();
    const int p = sp;
    if (p != t) {
      for (int r = tid; r < SP; r += NT) {
        double a = Z[(long long)t * SP + r];
        Z[(long long)t * SP + r] = Z[(long long)p * SP + r];
        Z[(long long)p * SP + r] = a;
      }
      if (tid == 0) { double a = zn[t]; zn[t] = zn[p]; zn[p] = a; }
    }
    __syncthreads();
    // Householder on Z(t:SP, t)
    double* x = Z + (long long)t * SP;
    if (warp == 0) {
      double s = 0.0;
      for (int r = t + 1 + lane; r < SP; r += 32) s += x[r] * x[r];
      s = wsum(s);
      if (lane == 0) {
        const double alpha = x[t];
        double tau = 0.0, beta = alpha, scale = 0.0;
        if (s != 0.0) {
          const double mu = sqrt(alpha * alpha + s);
          beta = (alpha >= 0.0) ? -mu : mu;
          tau = (beta - alpha) / beta;
          scale = 1.0 / (alpha - beta);
        }
        sc[0] = tau; sc[1] = beta; sc[2] = scale;
      }
    }
    __syncthreads();
    const double tau = sc[0], scale = sc[2];
    if (tau != 0.0)
      for (int r = t + 1 + tid; r < SP; r += NT) x[r] *= scale;
    __syncthreads();
    if (tid == 0) x[t] = sc[1];
    for (int j = t + 1 + warp; j < cr; j += NT / 32) {
      double* y = Z + (long long)j * SP;
      double dot = 0.0;
      for (int r = t + 1 + lane; r < SP; r += 32) dot += x[r] * y[r];
      dot = wsum(dot) + y[t];
      const double w = tau * dot;
      double ss = 0.0;
      for (int r = t + 1 + lane; r < SP; r += 32) {
        const double v = y[r] - w * x[r];
        y[r] = v;
        ss += v * v;
      }
      ss = wsum(ss);
      __syncwarp();
      if (lane == 0) { y[t] -= w; zn[j] = ss; }
    }
    __syncthreads();
  }
}

// Cluster version of the block pivot selection: the sketch columns Y(:, J:c) are
// distributed over the CL CTAs of a thread-block cluster and held in shared memory
// (SP x chunk each); every greedy step exchanges the CTAs' best candidates and the
// Householder vector of the winner through distributed shared memory, so one step
// costs two cluster barriers instead of a pass of one SM over the whole sketch in
// global memory.  Same greedy rule as sketch_cpqr_kernel (the column norms are summed in a
// different order, so near-ties may resolve differently).
constexpr int SK_NT = 512, SK_NW = SK_NT / 32;
constexpr int SK_MAXCOLS = 600;   // columns per CTA: (SPP + 1) * 600 * 8 B = 202 KB of shared memory
constexpr int SPP = SP + 1;       // padded shared-memory column stride (odd: conflict-free per-thread columns)

template <int CL>
__global__ void __launch_bounds__(SK_NT) sketch_cpqr_cl_kernel(const RDesc* __restrict__ d0) {
  extern __shared__ double sk_sm[];
  __shared__ double cand_v[CL];
  __shared__ int cand_i[CL];
  __shared__ double hv[SP];
  __shared__ double htau;
  __shared__ double redv[SK_NW];
  __shared__ int redi[SK_NW];
  __shared__ int chosen[QR_NB];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const RDesc d = d0[blockIdx.x / CL];
  const int J = d.J, cr = d.c - J, nbp = d.nbp;
  const int chunk = (cr + CL - 1) / CL;
  const int j0 = rank * chunk, nc = max(0, min(cr, j0 + chunk) - j0);
  double* Zs = sk_sm;               // SP x chunk, column-major with the padded stride SPP
  double* zn = Zs + SPP * chunk;    // squared trailing norms (-1: retired)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < SP * nc; e += SK_NT) {
    const int j = e / SP, r = e - j * SP;
    Zs[j * SPP + r] = d.Y[(long long)(J + j0) * SP + e];
  }
  __syncthreads();
  for (int j = tid; j < nc; j += SK_NT) {   // one thread per column
    const double* z = Zs + j * SPP;
    double s2 = 0.0;
    for (int r = 0; r < SP; ++r) s2 += z[r] * z[r];
    zn[j] = s2;
  }
  __syncthreads();
  for (int t = 0; t < nbp; ++t) {
    // local candidate: largest trailing norm, ties -> lowest global index
    double bv = -2.0;
    int bi = INT_MAX;
    for (int j = tid; j < nc; j += SK_NT) {
      const double v = zn[j];
      if (v > bv) { bv = v; bi = j0 + j; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { redv[warp] = bv; redi[warp] = bi; }
    __syncthreads();
    if (tid < CL) {
      double v = redv[0];
      int b = redi[0];
      for (int w = 1; w < SK_NW; ++w)
        if (redv[w] > v || (redv[w] == v && redi[w] < b)) { v = redv[w]; b = redi[w]; }
      double* rv = cluster.map_shared_rank(cand_v, tid);
      int* ri = cluster.map_shared_rank(cand_i, tid);
      rv[rank] = v;
      ri[rank] = b;
    }
    cluster.sync();
    double pv = cand_v[0];
    int p = cand_i[0];
    for (int r = 1; r < CL; ++r)
      if (cand_v[r] > pv || (cand_v[r] == pv && cand_i[r] < p)) { pv = cand_v[r]; p = cand_i[r]; }
    if (p >= cr) p = t;   // degenerate (no active column): keep the order
    const int owner = p / chunk;
    if (rank == owner && warp == 0) {
      // Householder reflector of Zs(t:SP, p): v = [1; x(t+1:)/(x_t - beta)], tau = (beta - x_t)/beta
      double* x = Zs + (p - j0) * SPP;
      double s2 = 0.0;
      for (int r = t + 1 + lane; r < SP; r += 32) s2 += x[r] * x[r];
      s2 = wsum(s2);
      const double alpha = x[t];
      double tau = 0.0, beta = alpha, scale = 0.0;
      if (s2 != 0.0) {
        const double mu = sqrt(alpha * alpha + s2);
        beta = (alpha >= 0.0) ? -mu : mu;
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      for (int r = lane; r < SP; r += 32) {
        const double v = (r < t) ? 0.0 : (r == t ? 1.0 : x[r] * scale);
        for (int q = 0; q < CL; ++q) cluster.map_shared_rank(hv, q)[r] = v;
      }
      if (lane < CL) *cluster.map_shared_rank(&htau, lane) = tau;
      if (lane == 0) zn[p - j0] = -1.0;   // retired
    }
    if (rank == 0 && tid == 0) chosen[t] = p;
    cluster.sync();
    // apply (I - tau v v^T) to the active local columns and recompute their trailing norms,
    // one thread per column (hv is read as a broadcast; the padded stride SPP keeps the
    // per-thread column accesses at two wavefronts per warp): a warp-per-column layout spends
    // most of its instructions in shuffle reductions over only SP = 40 rows
    const double tau = htau;
    for (int j = tid; j < nc; j += SK_NT) {
      if (zn[j] < 0.0) continue;
      double* z = Zs + j * SPP;
      double dot = 0.0;
      for (int r = t; r < SP; ++r) dot += z[r] * hv[r];
      const double w = tau * dot;
      double s2 = 0.0;
      for (int r = t; r < SP; ++r) {
        const double b = z[r] - w * hv[r];
        z[r] = b;
        if (r > t) s2 += b * b;
      }
      zn[j] = s2;
    }
    __syncthreads();
  }
  // chosen original indices -> sequential swap list (swap positions t and sw[t], t = 0..nbp-1)
  if (rank == 0 && tid == 0) {
    int mv_orig[2 * QR_NB], mv_pos[2 * QR_NB], nm = 0;   // moved columns: original index -> position
    auto pos_of = [&](int o) {
      for (int q = 0; q < nm; ++q) if (mv_orig[q] == o) return mv_pos[q];
      return o;
    };
    auto at_pos = [&](int ps) {   // original column currently at position ps
      for (int q = 0; q < nm; ++q) if (mv_pos[q] == ps) return mv_orig[q];
      for (int q = 0; q < nm; ++q) if (mv_orig[q] == ps) return -1;   // ps's original moved away
      return ps;
    };
    auto set_pos = [&](int o, int ps) {
      for (int q = 0; q < nm; ++q) if (mv_orig[q] == o) { mv_pos[q] = ps; return; }
      mv_orig[nm] = o; mv_pos[nm] = ps; ++nm;
    };
    for (int t = 0; t < nbp; ++t) {
      const int p = chosen[t];
      const int q = pos_of(p);
      int ot = at_pos(t);
      if (ot < 0) {   // search: the original column sitting at position t
        for (int k2 = 0; k2 < nm; ++k2) if (mv_pos[k2] == t) { ot = mv_orig[k2]; break; }
      }
      d.sw[t] = q;
      if (q != t) { set_pos(p, t); set_pos(ot, q); }
    }
  }
}

// Swap list of a block from the chosen original columns (positions relative to J), composed by
// one warp: a table of the (<= 2 QR_NB) positions the swaps touched, searched with a ballot per
// step, instead of one thread's linear scans over local-memory arrays.  sw[t]: the position
// swapped with t at step t (swap positions t and sw[t], t = 0..nbp-1, in order).
__device__ void compose_swaps_warp(const int* chosen, int nbp, int* sw, int* posv, int* origv, int lane) {
  int n = 0;   // table entries (uniform across the warp)
  auto find = [&](const int* keys, int key) -> int {   // entry index holding key, -1 if none
    int f = -1;
    for (int b = 0; b < n; b += 32) {
      const int e = b + lane;
      const unsigned m = __ballot_sync(0xffffffffu, e < n && keys[e] == key);
      if (m) { f = b + __ffs(m) - 1; break; }
    }
    return f;
  };
  for (int t = 0; t < nbp; ++t) {
    const int o = chosen[t];
    const int eo = find(origv, o);
    const int q = eo >= 0 ? posv[eo] : o;
    if (lane == 0) sw[t] = q;
    if (q != t) {
      const int et = find(posv, t);
      const int ot = et >= 0 ? origv[et] : t;
      // position t now holds o, position q holds ot
      if (lane == 0) {
        if (et >= 0) origv[et] = o; else { posv[n] = t; origv[n] = o; }
      }
      const int n1 = n + (et >= 0 ? 0 : 1);
      __syncwarp();
      const int eq = (eo >= 0) ? eo : -1;   // the entry of position q is the one that held o
      if (lane == 0) {
        if (eq >= 0) origv[eq] = ot; else { posv[n1] = q; origv[n1] = ot; }
      }
      n = n1 + (eq >= 0 ? 0 : 1);
      __syncwarp();
    }
  }
}

// Register-resident pivot selection (round 2): one sketch column (SP doubles) per thread in
// registers, columns over the CL CTAs of a cluster (<= 512 each).  Each step every CTA finds
// its best trailing norm, publishes the candidate COLUMN itself (not only its index) to every
// CTA through DSMEM, and after ONE cluster barrier every thread knows the winner and builds the
// Householder vector from the published column -- no second barrier to broadcast it.  Same
// greedy rule as sketch_cpqr_cl_kernel (largest trailing norm, ties to the lowest index).
constexpr int SR_NT = 512, SR_NW = SR_NT / 32;
template <int CL>
__global__ void __launch_bounds__(SR_NT, 1) sketch_cpqr_reg_kernel(const RDesc* __restrict__ d0) {
  __shared__ double xc[2][CL][SP];     // candidate columns, by rank
  __shared__ double xv[2][CL];         // candidate trailing norms (-2: none)
  __shared__ int xi[2][CL];            // candidate indices (block-relative)
  __shared__ double redv[SR_NW];
  __shared__ int redi[SR_NW];
  __shared__ double colbuf[SP];
  __shared__ int chosen[QR_NB], posv[2 * QR_NB], origv[2 * QR_NB];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const RDesc d = d0[blockIdx.x / CL];
  const int J = d.J, cr = d.c - J, nbp = d.nbp;
  const int chunk = (cr + CL - 1) / CL;
  const int j0 = rank * chunk, nc = max(0, min(cr, j0 + chunk) - j0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool mine = tid < nc;
  const int myc = j0 + tid;
  double z[SP];
  double zn = -2.0;
  if (mine) {
    const double* src = d.Y + (long long)(J + myc) * SP;
    zn = 0.0;
#pragma unroll
    for (int r = 0; r < SP; ++r) { z[r] = src[r]; zn += z[r] * z[r]; }
  } else {
#pragma unroll
    for (int r = 0; r < SP; ++r) z[r] = 0.0;
  }
  auto better = [](double ov, int oi, double bv, int bi) { return ov > bv || (ov == bv && oi < bi); };
  for (int t = 0; t < nbp; ++t) {
    const int buf = t & 1;
    // local candidate: largest trailing norm, ties -> lowest index (warp shuffles, then every warp
    // reduces the 16 warp results itself: one CTA barrier per step)
    double bv = (mine && zn > -1.0) ? zn : -2.0;
    int bi = (mine && zn > -1.0) ? myc : INT_MAX;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { redv[warp] = bv; redi[warp] = bi; }
    __syncthreads();
    bv = lane < SR_NW ? redv[lane] : -2.0;
    bi = lane < SR_NW ? redi[lane] : INT_MAX;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
    }
    // the warp holding the CTA's candidate (warp 0 when the CTA has none) publishes (norm, index,
    // column) to every rank
    const int ow = (bi == INT_MAX) ? 0 : (bi - j0) / 32;
    if (warp == ow) {
      if (bi != INT_MAX && myc == bi) {
#pragma unroll
        for (int r = 0; r < SP; ++r) colbuf[r] = z[r];
      }
      __syncwarp();
      for (int e = lane; e < CL * (SP + 1); e += 32) {
        const int q = e / (SP + 1), r = e - q * (SP + 1);
        if (r < SP) {
          cluster.map_shared_rank(&xc[0][0][0], q)[(buf * CL + rank) * SP + r] = colbuf[r];
        } else {
          cluster.map_shared_rank(&xv[0][0], q)[buf * CL + rank] = bv;
          cluster.map_shared_rank(&xi[0][0], q)[buf * CL + rank] = bi;
        }
      }
    }
    cluster.sync();
    double pv = xv[buf][0];
    int p = xi[buf][0], wr = 0;
#pragma unroll
    for (int r = 1; r < CL; ++r)
      if (better(xv[buf][r], xi[buf][r], pv, p)) { pv = xv[buf][r]; p = xi[buf][r]; wr = r; }
    if (p >= cr || pv < -1.0) p = t;   // degenerate (no active column): keep the order
    if (rank == 0 && tid == 0) chosen[t] = p;
    if (pv < -1.0) continue;           // nothing left to reflect (uniform over the cluster)
    // Householder reflector of the winner's rows t..SP-1 (every thread, from the published copy):
    // its trailing norm^2 is the published pv (rows >= t), so mu = sqrt(pv)
    const double* xw = &xc[buf][wr][0];
    const double alpha = xw[t];
    double tau = 0.0, scale = 0.0;
    if (pv > alpha * alpha) {
      const double mu = sqrt(pv);
      const double beta = (alpha >= 0.0) ? -mu : mu;
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    if (mine && myc == p) zn = -2.0;   // retired
    if (mine && zn > -1.0) {
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int r = 0; r < SP; ++r) {
        if (r < t) continue;
        const double hv = (r == t) ? 1.0 : xw[r] * scale;
        if (r & 1) d1 += z[r] * hv; else d0 += z[r] * hv;
      }
      const double w = tau * (d0 + d1);
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int r = 0; r < SP; ++r) {
        if (r < t) continue;
        const double hv = (r == t) ? 1.0 : xw[r] * scale;
        z[r] -= w * hv;
        if (r > t) { if (r & 1) s1 += z[r] * z[r]; else s0 += z[r] * z[r]; }
      }
      zn = s0 + s1;
    }
  }
  if (rank != 0) return;
  __syncthreads();
  if (warp == 0) compose_swaps_warp(chosen, nbp, d.sw, posv, origv, lane);
}

template <int CL>
void launch_sk_reg(cudaStream_t s, const RDesc* dd, int na) {
  static std::once_flag attr_once;
  std::call_once(attr_once, [&] {
    if (CL > 8) RSF_CUDA(cudaFuncSetAttribute(sketch_cpqr_reg_kernel<CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  });
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(na * CL));
  cfg.blockDim = dim3(SR_NT);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  RSF_CUDA(cudaLaunchKernelEx(&cfg, sketch_cpqr_reg_kernel<CL>, dd));
  count_launch();
}

// register pivot selection when the widest trailing sketch fits in <= 16 CTAs x 512 columns
bool launch_sketch_reg(cudaStream_t s, const RDesc* dd, int na, int crmax) {
  static const bool on = !(getenv("RSF_SKETCH_REG") && getenv("RSF_SKETCH_REG")[0] == '0');
  if (!on || crmax <= 0 || crmax > 16 * SR_NT) return false;
  int CL = 1;
  while ((crmax + CL - 1) / CL > SR_NT) CL *= 2;
  switch (CL) {
    case 1: launch_sk_reg<1>(s, dd, na); break;
    case 2: launch_sk_reg<2>(s, dd, na); break;
    case 4: launch_sk_reg<4>(s, dd, na); break;
    case 8: launch_sk_reg<8>(s, dd, na); break;
    default: launch_sk_reg<16>(s, dd, na); break;
  }
  return true;
}

// apply the swap list to A (m rows), Y (SP rows) and piv
// The block's column swaps (positions J + t and J + sw[t], t = 0..nbp-1, in order).  Rows are
// independent: every thread applies the whole swap sequence to its rows of A, so the CTAs of
// one problem split its rows (grid.x) with no barrier; CTA 0 also swaps Y's rows and piv.
__global__ void apply_swaps_kernel(const RDesc* __restrict__ d0) {
  const RDesc d = d0[blockIdx.y];
  __shared__ int sw[QR_NB];
  if (threadIdx.x < d.nbp) sw[threadIdx.x] = d.J + d.sw[threadIdx.x];
  __syncthreads();
  for (long long r = blockIdx.x * (long long)NT + threadIdx.x; r < d.m; r += (long long)gridDim.x * NT)
    for (int t = 0; t < d.nbp; ++t) {
      const int a = d.J + t, b = sw[t];
      if (a != b) {
        double* ca = d.A + (long long)a * d.lda + r;
        double* cb = d.A + (long long)b * d.lda + r;
        const double v = *ca; *ca = *cb; *cb = v;
      }
    }
  if (blockIdx.x != 0) return;
  for (int r = threadIdx.x; r < SP; r += NT)
    for (int t = 0; t < d.nbp; ++t) {
      const int a = d.J + t, b = sw[t];
      if (a != b) {
        double* ya = d.Y + (long long)a * SP + r;
        double* yb = d.Y + (long long)b * SP + r;
        const double v = *ya; *ya = *yb; *yb = v;
      }
    }
  if (threadIdx.x == 0)
    for (int t = 0; t < d.nbp; ++t) {
      const int a = d.J + t, b = sw[t];
      if (a != b) { const int v = d.piv[a]; d.piv[a] = d.piv[b]; d.piv[b] = v; }
    }
}

// The same column swaps with the sequence composed first: thread 0 lists the affected columns
// (the block's positions J..J+nbp-1 and their swap targets, <= 2 QR_NB) and which original
// column ends up in each; every CTA then moves its 64-row slab of those columns through shared
// memory -- coalesced column reads, all loads in flight at once -- instead of nbp dependent
// read-modify-write swaps per row.  The sketch columns and pivots are swapped as before.
constexpr int SW_ROWS = 64;
__global__ void __launch_bounds__(NT) apply_swaps_rows_kernel(const RDesc* __restrict__ d0) {
  const RDesc d = d0[blockIdx.y];
  // cols[q]: original column of slot q; cur[q]: the column it moves to.  Slots 0..nbp-1 are the
  // block positions J+q, slots QR_NB+t the swap targets outside the block (first occurrence);
  // every slot replays the swap sequence on its own position (no serial composition)
  __shared__ int cols[2 * QR_NB], cur[2 * QR_NB];
  __shared__ double buf[2 * QR_NB][SW_ROWS + 1];
  if (threadIdx.x < 2 * QR_NB) {
    const int q = threadIdx.x, J = d.J, nbp = d.nbp;
    int col = -1;
    if (q < QR_NB) {
      if (q < nbp) col = J + q;
    } else {
      const int t = q - QR_NB;
      if (t < nbp) {
        const int b = J + d.sw[t];
        bool first = b >= J + nbp;
        for (int t2 = 0; t2 < t && first; ++t2) first = (J + d.sw[t2]) != b;
        if (first) col = b;
      }
    }
    int pos = col;
    if (col >= 0)
      for (int t = 0; t < nbp; ++t) {
        const int a = J + t, b = J + d.sw[t];
        if (pos == a) pos = b; else if (pos == b) pos = a;
      }
    cols[q] = col;      // data of original column col ...
    cur[q] = pos;       // ... ends up in column pos
  }
  __syncthreads();
  const int nc = 2 * QR_NB;
  for (long long r0 = (long long)blockIdx.x * SW_ROWS; r0 < d.m; r0 += (long long)gridDim.x * SW_ROWS) {
    const int rows = (int)min((long long)SW_ROWS, d.m - r0);
    for (int e = threadIdx.x; e < nc * SW_ROWS; e += NT) {
      const int rr = e % SW_ROWS, q = e / SW_ROWS;
      if (rr < rows && cols[q] >= 0 && cur[q] != cols[q]) buf[q][rr] = d.A[(long long)cols[q] * d.lda + r0 + rr];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nc * SW_ROWS; e += NT) {
      const int rr = e % SW_ROWS, q = e / SW_ROWS;
      if (rr < rows && cols[q] >= 0 && cur[q] != cols[q]) d.A[(long long)cur[q] * d.lda + r0 + rr] = buf[q][rr];
    }
    __syncthreads();
  }
  if (blockIdx.x != 0) return;
  for (int r = threadIdx.x; r < SP; r += NT)
    for (int t = 0; t < d.nbp; ++t) {
      const int a = d.J + t, b = d.J + d.sw[t];
      if (a != b) {
        double* ya = d.Y + (long long)a * SP + r;
        double* yb = d.Y + (long long)b * SP + r;
        const double v = *ya; *ya = *yb; *yb = v;
      }
    }
  if (threadIdx.x == 0)
    for (int t = 0; t < d.nbp; ++t) {
      const int a = d.J + t, b = d.J + d.sw[t];
      if (a != b) { const int v = d.piv[a]; d.piv[a] = d.piv[b]; d.piv[b] = v; }
    }
}

// squared norms of the trailing columns A(j1:m, j) for j >= j1 (warp per column, many CTAs)
__global__ void trail_norm_kernel(const RDesc* __restrict__ d0) {
  const RDesc d = d0[blockIdx.y];
  const int j1 = d.J + d.nbp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = j1 + blockIdx.x * (NT / 32) + warp; j < d.c; j += gridDim.x * (NT / 32)) {
    const double* a = d.A + (long long)j * d.lda;
    double s = 0.0;
    for (int r = j1 + lane; r < d.m; r += 32) s += a[r] * a[r];
    s = wsum(s);
    if (lane == 0) d.nrm2[j] = s;
  }
}

// smallest k' in [J, j1] with max trailing column norm <= eps * ref (exact, from R and nrm2)
__global__ void __launch_bounds__(NT) rank_kernel(const RDesc* __restrict__ d0) {
  const RDesc d = d0[blockIdx.x];
  if (d.flag[0]) return;   // finished at an earlier block (checks are deferred, see rrqr_batched)
  const int J = d.J, nbp = d.nbp, j1 = J + nbp;
  __shared__ double red[QR_NB + 1][NT / 32];
  double mx[QR_NB + 1];
#pragma unroll
  for (int q = 0; q <= QR_NB; ++q) mx[q] = 0.0;
  for (int j = J + threadIdx.x; j < d.c; j += NT) {
    const double* a = d.A + (long long)j * d.lda;
    if (j < j1) {
      double acc = 0.0;   // sum_{r=k'}^{j} R(r,j)^2 for k' = j, j-1, ..., J
      for (int r = j; r >= J; --r) {
        acc += a[r] * a[r];
        const int q = r - J;
        mx[q] = fmax(mx[q], acc);
      }
    } else {
      double acc = d.nrm2[j];
      mx[nbp] = fmax(mx[nbp], acc);
      for (int r = j1 - 1; r >= J; --r) {
        acc += a[r] * a[r];
        const int q = r - J;
        mx[q] = fmax(mx[q], acc);
      }
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q <= QR_NB; ++q) {
    double v = mx[q];
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) red[q][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double thr = d.eps * (*d.ref);
    int k = -1;
    for (int q = 0; q <= nbp; ++q) {
      double v = 0.0;
      for (int w = 0; w < NT / 32; ++w) v = fmax(v, red[q][w]);
      if (sqrt(v) <= thr) { k = J + q; break; }
    }
    if (k < 0 && j1 >= min(d.m, d.c)) k = j1;
    if (k >= 0) { d.flag[0] = 1; d.flag[1] = k; d.flag[2] = j1; }
  }
}

// The same rank test, parallel over columns: a warp per column j holds the panel rows J + lane
// (coalesced), a suffix scan over the lanes gives sum_{r >= J+q} of the squares for every q at
// once (rows r <= j only inside the panel: below the diagonal are Householder vectors), and the
// per-q maxima over the columns go to mxb by an atomic max on the IEEE bit patterns (exact and
// order-independent for non-negative doubles, so the result is deterministic).  rank_finish_kernel
// applies the threshold and resets mxb for the next block.  (The one-CTA-per-problem rank_kernel
// above kept 33 maxima in a dynamically indexed local array: 280-byte stack, uncoalesced reads.)
__global__ void __launch_bounds__(NT) rank_cols_kernel(const RDesc* __restrict__ d0, unsigned long long* mxb) {
  const RDesc d = d0[blockIdx.y];
  if (d.flag[0]) return;
  const int J = d.J, nbp = d.nbp, j1 = J + nbp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ double red[NT / 32][QR_NB + 1];
  double mq = 0.0, mb = 0.0;   // running max of this lane's q = lane, and of q = nbp (trailing only)
  for (int j = J + blockIdx.x * (NT / 32) + warp; j < d.c; j += gridDim.x * (NT / 32)) {
    const double* a = d.A + (long long)j * d.lda;
    const int r = J + lane;
    const double x = (lane < nbp && (j >= j1 || r <= j)) ? a[r] : 0.0;
    double sfx = x * x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double t = __shfl_down_sync(0xffffffffu, sfx, o);
      if (lane + o < 32) sfx += t;
    }
    const double base = (j >= j1) ? d.nrm2[j] : 0.0;
    if (lane < nbp) mq = fmax(mq, base + sfx);
    mb = fmax(mb, base);
  }
  red[warp][lane] = mq;
  if (lane == 0) red[warp][QR_NB] = mb;
  __syncthreads();
  if (threadIdx.x <= QR_NB && threadIdx.x <= nbp) {
    const int q = threadIdx.x == nbp ? QR_NB : threadIdx.x;
    double v = 0.0;
    for (int w = 0; w < NT / 32; ++w) v = fmax(v, red[w][q]);
    atomicMax(mxb + (long long)d.id * (QR_NB + 1) + q, (unsigned long long)__double_as_longlong(v));
  }
}

__global__ void rank_finish_kernel(const RDesc* __restrict__ d0, unsigned long long* mxb) {
  const RDesc d = d0[blockIdx.x];
  unsigned long long* m = mxb + (long long)d.id * (QR_NB + 1);
  if (threadIdx.x == 0 && !d.flag[0]) {
    const int J = d.J, nbp = d.nbp, j1 = J + nbp;
    const double thr = d.eps * (*d.ref);
    int k = -1;
    for (int q = 0; q <= nbp; ++q) {
      const double v = __longlong_as_double((long long)m[q == nbp ? QR_NB : q]);
      if (sqrt(v) <= thr) { k = J + q; break; }
    }
    if (k < 0 && j1 >= min(d.m, d.c)) k = j1;
    if (k >= 0) { d.flag[0] = 1; d.flag[1] = k; d.flag[2] = j1; }
  }
  __syncthreads();
  for (int q = threadIdx.x; q <= QR_NB; q += blockDim.x) m[q] = 0ull;
}

// inverse of the upper-triangular block R(J:j1, J:j1) -> R11i (ld QR_NB)
__global__ void r11_inv_kernel(const RDesc* __restrict__ d0) {
  const RDesc d = d0[blockIdx.x];
  __shared__ double S[QR_NB * QR_NB];
  const int nb = d.nbp;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e % nb, j = e / nb;
    S[e] = (i <= j) ? d.A[(long long)(d.J + j) * d.lda + d.J + i] : 0.0;
  }
  __syncthreads();
  if (threadIdx.x < nb) {
    const int c = threadIdx.x;   // column c of the inverse: back substitution
    double x[QR_NB];
#pragma unroll
    for (int i = 0; i < QR_NB; ++i) x[i] = 0.0;
    for (int i = c; i >= 0; --i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int l = i + 1; l <= c; ++l) s -= S[l * nb + i] * x[l];
      x[i] = s / S[i * nb + i];
    }
    for (int i = 0; i < QR_NB; ++i) d.R11i[c * QR_NB + i] = (i <= c && i < nb) ? x[i] : 0.0;
  }
}

template <class D>
DBuf<D> upd(const std::vector<D>& v, cudaStream_t s) {
  DBuf<D> b(std::max<size_t>(v.size(), 1), s);
  b.upload(v);
  return b;
}

// ----------------------------------------------------------------- trsm helpers
constexpr int TB = 64;
struct DInvDesc { const double* U; long long ldu; int nb; double* out; };   // out ld TB
__global__ void upper_inv64_kernel(const DInvDesc* __restrict__ d0) {
  const DInvDesc d = d0[blockIdx.x];
  __shared__ double S[TB * TB];
  const int nb = d.nb;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int i = e % nb, j = e / nb;
    S[e] = (i <= j) ? d.U[(long long)j * d.ldu + i] : 0.0;
  }
  __syncthreads();
  if (threadIdx.x < nb) {
    const int c = threadIdx.x;
    for (int i = c; i >= 0; --i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int l = i + 1; l <= c; ++l) s -= S[l * nb + i] * d.out[c * TB + l];
      d.out[c * TB + i] = s / S[i * nb + i];
    }
    for (int i = c + 1; i < TB; ++i) d.out[c * TB + i] = 0.0;
  }
}

template <int CL>
void launch_cl(cudaStream_t s, const RDesc* dd, int na, int chunk) {
  static std::once_flag attr_once;
  std::call_once(attr_once, [&] {
    RSF_CUDA(cudaFuncSetAttribute(sketch_cpqr_cl_kernel<CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
    if (CL > 8) RSF_CUDA(cudaFuncSetAttribute(sketch_cpqr_cl_kernel<CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  });
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(na * CL));
  cfg.blockDim = dim3(SK_NT);
  cfg.dynamicSmemBytes = (size_t)(SPP + 1) * chunk * sizeof(double);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  RSF_CUDA(cudaLaunchKernelEx(&cfg, sketch_cpqr_cl_kernel<CL>, dd));
  count_launch();
}

// cluster pivot selection when the widest trailing sketch fits in <= 16 CTAs' shared memory
bool launch_sketch_cluster(cudaStream_t s, const RDesc* dd, int na, int crmax) {
  static const bool on = !(getenv("RSF_SKETCH_CLUSTER") && getenv("RSF_SKETCH_CLUSTER")[0] == '0');
  if (!on || crmax <= 0) return false;
  int CL = 1;
  while (CL < 16 && (crmax + CL - 1) / CL > SK_MAXCOLS) CL *= 2;
  const int chunk = (crmax + CL - 1) / CL;
  if (chunk > SK_MAXCOLS) return false;
  switch (CL) {
    case 1: launch_cl<1>(s, dd, na, chunk); break;
    case 2: launch_cl<2>(s, dd, na, chunk); break;
    case 4: launch_cl<4>(s, dd, na, chunk); break;
    case 8: launch_cl<8>(s, dd, na, chunk); break;
    default: launch_cl<16>(s, dd, na, chunk); break;
  }
  return true;
}

}  // namespace

void trsm_upper_batched(cudaStream_t s, const std::vector<TrsmProb>& probs) {
  if (probs.empty()) return;
  const int P = (int)probs.size();
  std::vector<long long> ioff(P), woff(P);
  long long it = 0, wt = 0;
  int maxblk = 0;
  std::vector<DInvDesc> dv;
  for (int i = 0; i < P; ++i) {
    const int nblk = (probs[i].k + TB - 1) / TB;
    ioff[i] = it; it += (long long)nblk * TB * TB;
    woff[i] = wt; wt += (long long)TB * probs[i].nrhs;
    maxblk = std::max(maxblk, nblk);
  }
  DBuf<double> inv(std::max<long long>(it, 1), s), W(std::max<long long>(wt, 1), s);
  for (int i = 0; i < P; ++i) {
    const auto& p = probs[i];
    const int nblk = (p.k + TB - 1) / TB;
    for (int b = 0; b < nblk; ++b) {
      const int r0 = b * TB, rb = std::min(TB, p.k - r0);
      dv.push_back(DInvDesc{p.U + (long long)r0 * p.ldu + r0, p.ldu, rb, inv.p + ioff[i] + (long long)b * TB * TB});
    }
  }
  if (!dv.empty()) {
    auto dd = ring_up(dv, s);
    for (size_t o = 0; o < dv.size(); o += 65535) {
      unsigned nb = (unsigned)std::min<size_t>(65535, dv.size() - o);
      upper_inv64_kernel<<<nb, 64, 0, s>>>(dd.p + o);
      count_launch();
      RSF_LAUNCH_CHECK();
    }
  }
  for (int st = 0; st < maxblk; ++st) {
    GemmBatch g1(false, false), g2(false, false);
    std::vector<CopyProb> cp;
    for (int i = 0; i < P; ++i) {
      const auto& p = probs[i];
      const int nblk = (p.k + TB - 1) / TB;
      const int b = nblk - 1 - st;
      if (b < 0 || p.nrhs <= 0) continue;
      const int r0 = b * TB, rb = std::min(TB, p.k - r0), r1 = r0 + rb;
      if (r1 < p.k) {   // B_b -= U(b, r1:k) X(r1:k)
        GemmDesc a = gdesc(rb, p.nrhs, p.k - r1);
        a.A = p.U + (long long)r1 * p.ldu + r0; a.lda = (int)p.ldu;
        a.B = p.B + r1; a.ldb = (int)p.ldb;
        a.C = p.B + r0; a.ldc = (int)p.ldb;
        a.alpha = -1.0; a.beta = 1.0;
        g1.add(a);
      }
      GemmDesc c = gdesc(rb, p.nrhs, rb);   // W = Uinv_bb B_b
      c.A = inv.p + ioff[i] + (long long)b * TB * TB; c.lda = TB;
      c.B = p.B + r0; c.ldb = (int)p.ldb;
      c.C = W.p + woff[i]; c.ldc = rb;
      g2.add(c);
      cp.push_back(CopyProb{W.p + woff[i], rb, p.B + r0, p.ldb, rb, p.nrhs, 1.0});
    }
    g1.run(s);
    g2.run(s);
    copy_batched(s, cp);
  }
}

RRQRResult rrqr_batched(cudaStream_t s, const std::vector<RRQRProb>& probs, double eps,
                        unsigned long long seed) {
  RRQRResult res;
  const int P = (int)probs.size();
  res.k.assign(P, 0);
  res.done.assign(P, 0);
  if (P == 0) return res;
  // workspaces
  std::vector<long long> goff(P), yoff(P), coff(P), voff(P), woff(P);
  long long gt = 0, yt = 0, ct = 0, vt = 0, wt = 0;
  for (int i = 0; i < P; ++i) {
    goff[i] = gt; gt += (long long)SP * probs[i].m;
    yoff[i] = yt; yt += (long long)SP * probs[i].c;
    coff[i] = ct; ct += probs[i].c;
    voff[i] = vt; vt += (long long)probs[i].m * QR_NB;
    woff[i] = wt; wt += (long long)QR_NB * probs[i].c;
  }
  DBuf<double> Y(yt, s), Z(yt, s), zn(ct, s), nrm2(ct, s), V(vt, s), W(wt, s), W2(wt, s), Wt(wt, s);
  DBuf<double> Tsc((size_t)P * QR_NB * QR_NB, s), R11i((size_t)P * QR_NB * QR_NB, s), ref(P, s);
  DBuf<int> sw((size_t)P * QR_NB, s), flag((size_t)3 * P, s);
  DBuf<unsigned long long> mxb((size_t)P * (QR_NB + 1), s);   // per-problem maxima of the rank test
  RSF_CUDA(cudaMemsetAsync(mxb.p, 0, (size_t)P * (QR_NB + 1) * sizeof(unsigned long long), s));
  std::vector<RDesc> base(P);
  for (int i = 0; i < P; ++i) {
    const auto& p = probs[i];
    RDesc d{};
    d.A = p.A; d.lda = p.lda; d.m = p.m; d.c = p.c;
    d.Y = Y.p + yoff[i]; d.Z = Z.p + yoff[i]; d.zn = zn.p + coff[i]; d.nrm2 = nrm2.p + coff[i];
    d.piv = p.piv; d.sw = sw.p + (long long)i * QR_NB; d.ref = ref.p + i; d.flag = flag.p + 3 * i;
    d.R11i = R11i.p + (long long)i * QR_NB * QR_NB;
    d.id = i; d.eps = eps;
    d.ref_in = p.ref_in; d.ref_out = p.ref_out;
    base[i] = d;
  }
  {
    DBuf<double> G(gt, s);
    for (int i = 0; i < P; ++i) base[i].G = G.p + goff[i];
    auto db = ring_up(base, s);
    {
      DBuf<unsigned long long> ref2(P, s);
      RSF_CUDA(cudaMemsetAsync(ref2.p, 0, P * sizeof(unsigned long long), s));
      long long cmax = 1, work = 0;
      for (auto& p : probs) { cmax = std::max<long long>(cmax, p.c); work = std::max<long long>(work, (long long)p.m * p.c); }
      // column blocks of 8 columns; enough CTAs per problem that ~1 MB of A goes to each
      const long long gx = std::max<long long>(1, std::min<long long>((cmax + 7) / 8, (work + (1 << 17) - 1) >> 17));
      ref_norms_kernel<<<dim3((unsigned)std::min<long long>(gx, 4096), P), NT, 0, s>>>(db.p, ref2.p);
      ref_finish_kernel<<<(P + 127) / 128, 128, 0, s>>>(db.p, ref2.p, P);
      count_launch();
    }
    long long mx = 0;
    for (auto& p : probs) mx = std::max(mx, (long long)SP * p.m);
    gauss_kernel<<<dim3((unsigned)std::min<long long>(1024, (mx + NT - 1) / NT), P), NT, 0, s>>>(
        db.p, (unsigned)(seed & 0xffffffffu));
    count_launch(2);
    RSF_LAUNCH_CHECK();
    GemmBatch gy(false, false);   // Y = G A
    for (int i = 0; i < P; ++i) {
      GemmDesc g = gdesc(SP, probs[i].c, probs[i].m);
      g.A = base[i].G; g.lda = SP; g.B = probs[i].A; g.ldb = (int)probs[i].lda; g.C = base[i].Y; g.ldc = SP;
      gy.add(g);
    }
    gy.run(s);
    for (int i = 0; i < P; ++i) base[i].G = nullptr;
  }
  std::vector<int> hflag = flag.to_host(3 * P);
  std::vector<int> active;
  for (int i = 0; i < P; ++i) {
    if (hflag[3 * i]) { res.k[i] = 0; res.done[i] = 0; }
    else active.push_back(i);
  }
  // The rank test of a block is read back only every `every` blocks (and at a problem's last
  // block): finished problems run a few more (harmless) blocks -- the later panels touch rows and
  // columns past the rank only, rank_kernel ignores them -- in exchange for 1/every host syncs.
  static const int every = getenv("RSF_RRQR_CHECK") ? std::max(1, atoi(getenv("RSF_RRQR_CHECK"))) : 4;
  for (int J = 0; !active.empty(); J += QR_NB) {
    {
      std::vector<int> keep;   // problems whose columns are exhausted were finished at the previous block
      for (int i : active) if (J < std::min(probs[i].m, probs[i].c)) keep.push_back(i);
      if (keep.size() != active.size()) {
        hflag = flag.to_host(3 * P);
        for (int i : active)
          if (J >= std::min(probs[i].m, probs[i].c)) { res.k[i] = hflag[3 * i + 1]; res.done[i] = hflag[3 * i + 2]; }
        active.swap(keep);
        if (active.empty()) break;
      }
    }
    std::vector<RDesc> dv;
    for (int i : active) {
      RDesc d = base[i];
      d.J = J;
      d.nbp = std::min(QR_NB, std::min(probs[i].m, probs[i].c) - J);
      dv.push_back(d);
    }
    auto dd = ring_up(dv, s);
    const unsigned na = (unsigned)dv.size();
    int crmax = 0;
    for (auto& d : dv) crmax = std::max(crmax, d.c - d.J);
    if (!launch_sketch_reg(s, dd.p, (int)na, crmax) && !launch_sketch_cluster(s, dd.p, (int)na, crmax)) {
      sketch_cpqr_kernel<<<na, NT, 0, s>>>(dd.p);
      count_launch();
    }
    {
      int mmax = 0;
      for (auto& d : dv) mmax = std::max(mmax, d.m);
      static const bool old_swaps = getenv("RSF_SWAPS_OLD") && getenv("RSF_SWAPS_OLD")[0] == '1';
      if (old_swaps)
        apply_swaps_kernel<<<dim3((unsigned)std::max(1, std::min(64, (mmax + NT - 1) / NT)), na), NT, 0, s>>>(dd.p);
      else
        apply_swaps_rows_kernel<<<dim3((unsigned)std::max(1, std::min(512, (mmax + SW_ROWS - 1) / SW_ROWS)), na), NT, 0,
                                  s>>>(dd.p);
      count_launch();
    }
    RSF_LAUNCH_CHECK();
    std::vector<PanelStep> ps;
    for (size_t a = 0; a < dv.size(); ++a) {
      const int i = active[a];
      const auto& p = probs[i];
      PanelStep st;
      st.A = p.A + (long long)J * p.lda + J; st.lda = p.lda;
      st.rows = p.m - J; st.ncol = dv[a].nbp; st.c2 = p.c - J - dv[a].nbp;
      st.V = V.p + voff[i];
      st.T = p.Tws ? p.Tws + (long long)(J / QR_NB) * QR_NB * QR_NB : Tsc.p + (long long)i * QR_NB * QR_NB;
      st.W = W.p + woff[i]; st.W2 = W2.p + woff[i];
      ps.push_back(st);
    }
    panel_step_batched(s, ps);
    int maxc = 0;
    for (auto& d : dv) maxc = std::max(maxc, d.c - d.J - d.nbp);
    if (maxc > 0) {
      trail_norm_kernel<<<dim3((unsigned)std::min(256, (maxc + 7) / 8), na), NT, 0, s>>>(dd.p);
      count_launch();
    }
    {
      static const bool old_rank = getenv("RSF_RANK_OLD") && getenv("RSF_RANK_OLD")[0] == '1';
      if (old_rank) {
        rank_kernel<<<na, NT, 0, s>>>(dd.p);
        count_launch();
      } else {
        int cmax = 0;
        for (auto& d : dv) cmax = std::max(cmax, d.c - d.J);
        rank_cols_kernel<<<dim3((unsigned)std::max(1, std::min(512, (cmax + 7) / 8)), na), NT, 0, s>>>(dd.p, mxb.p);
        rank_finish_kernel<<<na, 64, 0, s>>>(dd.p, mxb.p);
        count_launch(2);
      }
    }
    RSF_LAUNCH_CHECK();
    bool last = false;
    for (size_t a = 0; a < dv.size(); ++a) last |= (J + dv[a].nbp >= std::min(dv[a].m, dv[a].c));
    const bool check = last || ((J / QR_NB) % every == every - 1);
    std::vector<int> next;
    std::vector<RDesc> cont;
    if (check) {
      hflag = flag.to_host(3 * P);
      for (size_t a = 0; a < dv.size(); ++a) {
        const int i = active[a];
        if (hflag[3 * i]) {
          res.k[i] = hflag[3 * i + 1];
          res.done[i] = hflag[3 * i + 2];
        } else {
          next.push_back(i);
          cont.push_back(dv[a]);
        }
      }
    } else {
      next = active;
      cont = dv;
    }
    if (!cont.empty()) {   // sketch downdate: Y2 -= Y1 R11^-1 R12
      auto dc = ring_up(cont, s);
      r11_inv_kernel<<<(unsigned)cont.size(), 64, 0, s>>>(dc.p);
      count_launch();
      RSF_LAUNCH_CHECK();
      GemmBatch g1(false, false), g2(false, false);
      for (auto& d : cont) {
        const int j1 = d.J + d.nbp, rest = d.c - j1;
        if (rest <= 0) continue;
        const int i = d.id;
        GemmDesc a = gdesc(d.nbp, rest, d.nbp);   // Wt = R11^-1 R12
        a.A = d.R11i; a.lda = QR_NB; a.B = d.A + (long long)j1 * d.lda + d.J; a.ldb = (int)d.lda;
        a.C = Wt.p + woff[i]; a.ldc = QR_NB;
        g1.add(a);
        GemmDesc b = gdesc(SP, rest, d.nbp);      // Y2 -= Y1 Wt
        b.A = d.Y + (long long)d.J * SP; b.lda = SP; b.B = Wt.p + woff[i]; b.ldb = QR_NB;
        b.C = d.Y + (long long)j1 * SP; b.ldc = SP; b.alpha = -1.0; b.beta = 1.0;
        g2.add(b);
      }
      g1.run(s);
      g2.run(s);
    }
    active.swap(next);
  }
  // T = R11^-1 R12
  std::vector<TrsmProb> tp;
  std::vector<CopyProb> cp;
  for (int i = 0; i < P; ++i) {
    const auto& p = probs[i];
    const int k = res.k[i];
    if (!p.T || k == 0 || k >= p.c) continue;
    cp.push_back(CopyProb{p.A + (long long)k * p.lda, p.lda, p.T, p.ldt, k, p.c - k, 1.0});
    tp.push_back(TrsmProb{p.A, p.lda, p.T, p.ldt, k, p.c - k});
  }
  copy_batched(s, cp);
  trsm_upper_batched(s, tp);
  return res;
}

}  // namespace rsf

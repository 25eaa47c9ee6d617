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

#include "dense.cuh"
#include "peel.cuh"
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

// dst rows [r0, r0+k) of a (cap x n) X'-matrix <- src (k x n)
__global__ void rowblock_copy_kernel(double* dst, long long ldd, int r0, const double* src, int k, int n) {
  const long long tot = (long long)n * k;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    const long long t = e / k;
    const int j = (int)(e - t * k);
    dst[t * ldd + r0 + j] = src[e];
  }
}

// transpose: Q (ni x c, ld ni) <- Y' block (c x ni, ld ldy)
struct TrDesc { const double* Y; long long ldy; double* Q; int ni, c; };
__global__ void transpose_kernel(const TrDesc* __restrict__ descs) {
  __shared__ double tile[32][33];
  const TrDesc d = descs[blockIdx.z];
  const int tilesN = (d.ni + 31) / 32, tilesC = (d.c + 31) / 32;
  for (int tb = blockIdx.x; tb < tilesN * tilesC; tb += gridDim.x) {
    const int tn = tb % tilesN, tc = tb / tilesN;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
    for (int yy = ty; yy < 32; yy += 8) {
      const int t = tn * 32 + yy, j = tc * 32 + tx;
      tile[yy][tx] = (t < d.ni && j < d.c) ? d.Y[(long long)t * d.ldy + j] : 0.0;
    }
    __syncthreads();
    for (int yy = ty; yy < 32; yy += 8) {
      const int j = tc * 32 + yy, t = tn * 32 + tx;
      if (t < d.ni && j < d.c) d.Q[(long long)j * d.ni + t] = tile[tx][yy];
    }
    __syncthreads();
  }
}

// U (ni x k, ld ni) <- Q_R E_k padded: identity, then the CPQR reflectors in reverse
struct URDesc { double* U; int ni, q, k; const double* Rv; const double* tau; };
__global__ void form_qr_columns_kernel(const URDesc* __restrict__ descs) {
  const URDesc d = descs[blockIdx.x];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (long long e = tid; e < (long long)d.ni * d.k; e += NT) {
    const int r = (int)(e % d.ni), c = (int)(e / d.ni);
    d.U[e] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int i = d.k - 1; i >= 0; --i) {
    const double tau = d.tau[i];
    if (tau != 0.0) {
      const double* v = d.Rv + (long long)i * d.q;   // v(i) = 1, v(r>i) = Rv(r, i)
      for (int j = i + warp; j < d.k; j += NT / 32) {
        double* y = d.U + (long long)j * d.ni;
        double dot = 0.0;
        for (int r = i + 1 + lane; r < d.q; r += 32) dot += v[r] * y[r];
#pragma unroll
        for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        dot += y[i];
        const double w = tau * dot;
        for (int r = i + 1 + lane; r < d.q; r += 32) y[r] -= w * v[r];
        __syncwarp();
        if (lane == 0) y[i] -= w;
      }
    }
    __syncthreads();
  }
}

// E' (k x n): 1 where t - leafbegin[t] == e0 + j
__global__ void extract_probe_kernel(double* X, int k, int n, const int* __restrict__ lb, int e0) {
  const long long tot = (long long)n * k;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    const int t = (int)(e / k), j = (int)(e % k);
    X[e] = (t - lb[t] == e0 + j) ? 1.0 : 0.0;
  }
}

// per-block partial sums of diag entries H'(t - lb[t] - e0, t) and of their magnitudes
__global__ void extract_diag_kernel(const double* H, int k, int n, const int* __restrict__ lb, int e0,
                                    double* part, double* parta) {
  __shared__ double s1[NT], s2[NT];
  double a = 0.0, b = 0.0;
  for (int t = blockIdx.x * NT + threadIdx.x; t < n; t += gridDim.x * NT) {
    const int j = t - lb[t] - e0;
    if (j >= 0 && j < k) {
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
struct GOp {
  const Fact& F;
  const Fact* Fi;
  cudaStream_t s;
  DBuf<double> A, B, tmp;
  int kcap = 0;
  double columns = 0;
  GOp(const Fact& f, const Fact* fi) : F(f), Fi(fi), s(f.ctx->stream) {}
  void reserve(int k) {
    if (k <= kcap) return;
    kcap = k;
    const size_t n = F.n();
    A.alloc(n * k, s);
    if (Fi) B.alloc(n * k, s);
    tmp.alloc((size_t)std::max<long long>(F.tmp_cols, 1) * k, s);
  }
  // Y = G X (X preserved), X and Y are k x n
  void apply(const double* X, double* Y, int k) {
    reserve(k);
    const size_t bytes = (size_t)F.n() * k * sizeof(double);
    columns += k;
    if (!Fi) {
      RSF_CUDA(cudaMemcpyAsync(Y, X, bytes, cudaMemcpyDeviceToDevice, s));
      solve_internal(F, Y, k, tmp.p);
      return;
    }
    RSF_CUDA(cudaMemcpyAsync(A.p, X, bytes, cudaMemcpyDeviceToDevice, s));
    apply_only_internal(*Fi, A.p, B.p, k);          // B = F_i X
    solve_internal(F, B.p, k, tmp.p);               // B = F^-1 F_i X
    RSF_CUDA(cudaMemcpyAsync(A.p, X, bytes, cudaMemcpyDeviceToDevice, s));
    solve_internal(F, A.p, k, tmp.p);               // A = F^-1 X
    apply_only_internal(*Fi, A.p, Y, k);            // Y = F_i F^-1 X
    const long long nn = (long long)F.n() * k;
    axpby_kernel<<<gxx(nn), NT, 0, s>>>(Y, B.p, 0.5, 0.5, nn);
    count_launch();
    RSF_LAUNCH_CHECK();
  }
};

// ----------------------------------------------------------------- G^(m) storage
struct PairLR {
  int i, j;          // level-box indices
  int ib, ni, jb, nj;
  int kij = 0;
  long long uoff = -1, moff = -1;
  int rev = -1;      // index of the pair (j, i)
};

struct PeelLevel {
  std::vector<PairLR> pairs;
  DBuf<double> U, M;
  GemmBatch g1, g2, g3;
  long long tcols = 0;   // temp columns per probe column
  bool empty() const { return g1.empty(); }
  // Y' -= G^(m) X'   (X', Y' are k x n; tmp has k * tcols doubles)
  void subtract(cudaStream_t s, const double* X, double* Y, int k, double* tmp) const {
    if (g1.empty()) return;
    g1.run(s, const_cast<double*>(X), tmp, k, k);
    g2.run(s, nullptr, tmp, k, k);
    g3.run(s, Y, tmp, k, k);
  }
};

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

double peel(const Fact& F, const Fact* Fi, const Opts& o, int trace_id, PeelDiag* diag) {
  const double t0 = now_s();
  cudaStream_t s = F.ctx->stream;
  const Tree& t = *F.tree;
  const int n = t.n, L = t.L;
  const unsigned long long seed = o.seed;
  GOp G(F, Fi);
  std::vector<PeelLevel> peeled(L + 1);
  long long max_tcols = 0;
  PeelDiag pd;
  pd.cols.assign(L + 1, 0);
  pd.rank_max.assign(L + 1, 0);
  int prev_rank = -1;
  const int kb = std::max(16, o.probe_block);

  auto residual = [&](const double* W, double* Y, int k, int upto) {
    G.apply(W, Y, k);
    DBuf<double> tmp((size_t)std::max<long long>(max_tcols, 1) * k, s);
    for (int m = 1; m < upto; ++m) peeled[m].subtract(s, W, Y, k, tmp.p);
  };

  for (int lev = 1; lev <= L; ++lev) {
    const std::vector<int>& nodes = t.levels[lev];
    const int nb = (int)nodes.size();
    // ordered sibling pairs (Def. sibs)
    std::vector<PairLR> pairs;
    std::unordered_map<int, std::vector<int>> fam;
    for (int b = 0; b < nb; ++b) fam[t.parent[nodes[b]]].push_back(b);
    for (int b = 0; b < nb; ++b) {
      const auto& sib = fam[t.parent[nodes[b]]];
      for (int c : sib) {
        if (c == b) continue;
        PairLR p;
        p.i = b; p.j = c;
        p.ib = t.begin[nodes[b]]; p.ni = t.end[nodes[b]] - p.ib;
        p.jb = t.begin[nodes[c]]; p.nj = t.end[nodes[c]] - p.jb;
        pairs.push_back(p);
      }
    }
    if (pairs.empty()) continue;
    {
      std::unordered_map<long long, int> idx;
      for (int q = 0; q < (int)pairs.size(); ++q) idx[(long long)pairs[q].i * nb + pairs[q].j] = q;
      for (auto& p : pairs) p.rev = idx[(long long)p.j * nb + p.i];
    }
    std::vector<int> hq(n, -1);
    int maxni = 0;
    for (int b = 0; b < nb; ++b) {
      const int nd = nodes[b];
      for (int x = t.begin[nd]; x < t.end[nd]; ++x) hq[x] = t.quad[nd];
      maxni = std::max(maxni, t.end[nd] - t.begin[nd]);
    }
    DBuf<int> qmap = up(hq, s);
    const int cmax = maxni + o.oversample;
    int c = (prev_rank < 0) ? o.peel_start : (int)std::ceil(0.7 * prev_rank) + o.oversample;
    c = std::min(std::max(c, o.oversample + 8), cmax);
    c = (c + 7) / 8 * 8;
    int cap = 0, have = 0;
    DBuf<double> Yg[4];
    std::vector<int> kp(pairs.size(), 0);
    // QR factors of the final sketches (kept when they fit one batch)
    DBuf<double> Qws, Tws, Rout, tau;
    std::vector<long long> qoff(pairs.size()), toffv(pairs.size()), roff(pairs.size()), tauoff(pairs.size());
    while (true) {
      if (c > cap) {   // grow the sketch buffers (keep computed rows)
        int ncap = c;
        for (int g = 0; g < 4; ++g) {
          DBuf<double> nbuf((size_t)ncap * n, s);
          if (have > 0) {   // keep the computed rows [0, have)
            std::vector<CopyProb> cp{CopyProb{Yg[g].p, cap, nbuf.p, ncap, have, n, 1.0}};
            copy_batched(s, cp);
          }
          Yg[g] = std::move(nbuf);
        }
        cap = ncap;
      }
      // new probe columns [have, c) for every group
      for (int g = 0; g < 4; ++g) {
        for (int c0 = have; c0 < c; c0 += kb) {
          const int k = std::min(kb, c - c0);
          DBuf<double> W((size_t)n * k, s), Y((size_t)n * k, s);
          gen_probes(s, W.p, k, n, t.d_perm.p, qmap.p, g, c0, lev, trace_id, seed);
          residual(W.p, Y.p, k, lev);
          rowblock_copy_kernel<<<gxx((long long)n * k), NT, 0, s>>>(Yg[g].p, cap, c0, Y.p, k, n);
          count_launch();
          RSF_LAUNCH_CHECK();
        }
      }
      have = c;
      // sketches Y_ij = Y_{quad(j)}(I_i, 0:c) -> QR -> truncated CPQR (ranks)
      long long qtot = 0, ttot = 0, rtot = 0, tautot = 0;
      for (size_t q = 0; q < pairs.size(); ++q) {
        const auto& p = pairs[q];
        const int qq = std::min(p.ni, c);
        qoff[q] = qtot; qtot += (long long)p.ni * c;
        toffv[q] = ttot; ttot += (long long)((qq + QR_NB - 1) / QR_NB) * QR_NB * QR_NB;
        roff[q] = rtot; rtot += (long long)qq * c;
        tauoff[q] = tautot; tautot += std::max(qq, 1);
      }
      Qws.alloc(qtot, s);
      Tws.alloc(std::max<long long>(ttot, 1), s);
      Rout.alloc(std::max<long long>(rtot, 1), s);
      tau.alloc(std::max<long long>(tautot * 2, 1), s);
      {
        std::vector<TrDesc> td;
        std::vector<QRProb> qp;
        for (size_t q = 0; q < pairs.size(); ++q) {
          const auto& p = pairs[q];
          const int gj = t.quad[nodes[p.j]];
          td.push_back(TrDesc{Yg[gj].p + (long long)p.ib * cap, cap, Qws.p + qoff[q], p.ni, c});
          qp.push_back(QRProb{Qws.p + qoff[q], p.ni, p.ni, c, Tws.p + toffv[q], tau.p + tautot + tauoff[q]});
        }
        auto dtd = up(td, s);
        for (size_t o2 = 0; o2 < td.size(); o2 += 65535) {
          unsigned nz = (unsigned)std::min<size_t>(65535, td.size() - o2);
          transpose_kernel<<<dim3(64, 1, nz), NT, 0, s>>>(dtd.p + o2);
          count_launch();
          RSF_LAUNCH_CHECK();
        }
        geqrf_batched(s, qp, true);
        std::vector<CPQRProb> cp;
        DBuf<int> dpv((size_t)c * pairs.size(), s), dk(pairs.size(), s);
        long long wtot = 0;
        std::vector<long long> wo(pairs.size(), -1);
        for (size_t q = 0; q < pairs.size(); ++q) {
          const int qq = std::min(pairs[q].ni, c);
          if ((size_t)qq * c * 8 + (72 + 2 * (size_t)c + 64) * 8 > 200 * 1024) { wo[q] = wtot; wtot += (long long)qq * c; }
        }
        DBuf<double> W(std::max<long long>(wtot, 1), s);
        for (size_t q = 0; q < pairs.size(); ++q) {
          const auto& p = pairs[q];
          CPQRProb pr;
          pr.R = Qws.p + qoff[q]; pr.ldr = p.ni; pr.q = std::min(p.ni, c); pr.c = c;
          pr.W = wo[q] >= 0 ? W.p + wo[q] : nullptr;
          pr.T = nullptr; pr.piv = dpv.p + (long long)q * c;
          pr.Rout = Rout.p + roff[q]; pr.tau = tau.p + tauoff[q];
          cp.push_back(pr);
        }
        cpqr_id_batched(s, cp, o.eps_peel, dk.p, false);
        kp = dk.to_host(pairs.size());
      }
      int mr = 0;
      for (int v : kp) mr = std::max(mr, v);
      if (mr <= c - o.oversample || c >= cmax) {
        pd.rank_max[lev] = mr;
        break;
      }
      int nc = (mr >= c - 1) ? 2 * c : std::max(c + 8, (int)std::ceil(1.25 * mr) + o.oversample);
      nc = std::min((nc + 7) / 8 * 8, (cmax + 7) / 8 * 8);
      c = std::max(nc, c + 8);
    }
    pd.cols[lev] = c;
    prev_rank = pd.rank_max[lev];

    // ---- U_ij = Q [Q_R E_k ; 0]
    PeelLevel& PL = peeled[lev];
    long long utot = 0;
    for (size_t q = 0; q < pairs.size(); ++q) {
      pairs[q].kij = kp[q];
      pairs[q].uoff = utot;
      utot += (long long)pairs[q].ni * kp[q];
    }
    PL.U.alloc(std::max<long long>(utot, 1), s);
    {
      std::vector<URDesc> ud;
      std::vector<QApplyProb> ap;
      for (size_t q = 0; q < pairs.size(); ++q) {
        const auto& p = pairs[q];
        if (p.kij == 0) continue;
        ud.push_back(URDesc{PL.U.p + p.uoff, p.ni, std::min(p.ni, c), p.kij, Rout.p + roff[q], tau.p + tauoff[q]});
        ap.push_back(QApplyProb{Qws.p + qoff[q], p.ni, p.ni, c, Tws.p + toffv[q], PL.U.p + p.uoff, p.ni, p.kij});
      }
      if (!ud.empty()) {
        auto dud = up(ud, s);
        for (size_t o2 = 0; o2 < ud.size(); o2 += 65535) {
          unsigned nz = (unsigned)std::min<size_t>(65535, ud.size() - o2);
          form_qr_columns_kernel<<<nz, NT, 0, s>>>(dud.p + o2);
          count_launch();
          RSF_LAUNCH_CHECK();
        }
        ormqr_batched(s, ap, false);
      }
    }
    Qws.release(); Tws.release(); Rout.release(); tau.release();

    // ---- cores M_ij (Eq. lowrankapprox) via normal equations of the Gaussian sketches
    {
      const size_t P = pairs.size();
      std::vector<long long> woff(P), a1off(P), poff(P), b2off(P), g1off(P), g2off(P), t1off(P), t2off(P), moff(P);
      long long wt = 0, a1t = 0, pt = 0, b2t = 0, g1t = 0, g2t = 0, t1t = 0, t2t = 0, mt = 0;
      std::vector<long long> boxw(nb, -1);
      for (int b = 0; b < nb; ++b) { boxw[b] = wt; wt += (long long)c * (t.end[nodes[b]] - t.begin[nodes[b]]); }
      for (size_t q = 0; q < P; ++q) {
        const auto& p = pairs[q];
        const int k1 = p.kij, k2 = pairs[p.rev].kij;
        a1off[q] = a1t; a1t += (long long)c * k1;
        poff[q] = pt; pt += (long long)c * c;
        b2off[q] = b2t; b2t += (long long)k2 * c;
        g1off[q] = g1t; g1t += (long long)k1 * k1;
        g2off[q] = g2t; g2t += (long long)k2 * k2;
        t1off[q] = t1t; t1t += (long long)k1 * c;
        t2off[q] = t2t; t2t += (long long)k1 * k2;
        moff[q] = mt; mt += (long long)k1 * k2;
      }
      DBuf<double> Wb(std::max<long long>(wt, 1), s), A1(std::max<long long>(a1t, 1), s), Pm(std::max<long long>(pt, 1), s),
          B2(std::max<long long>(b2t, 1), s), G1(std::max<long long>(g1t, 1), s), G1i(std::max<long long>(g1t, 1), s),
          G2(std::max<long long>(g2t, 1), s), G2i(std::max<long long>(g2t, 1), s), T1(std::max<long long>(t1t, 1), s),
          T2(std::max<long long>(t2t, 1), s), T3(std::max<long long>(t2t, 1), s);
      PL.M.alloc(std::max<long long>(mt, 1), s);
      // probes of every box: W_b^T as (c x n_b), the same Philox entries as in the sketches
      for (int b = 0; b < nb; ++b) {
        const int nd = nodes[b];
        const int ni = t.end[nd] - t.begin[nd];
        probes_kernel<<<gxx((long long)ni * c), NT, 0, s>>>(Wb.p + boxw[b], c, t.begin[nd], t.end[nd], t.d_perm.p,
                                                            nullptr, 0, 0, lev, trace_id,
                                                            (unsigned)(seed & 0xffffffffull), c);
        count_launch();
      }
      RSF_LAUNCH_CHECK();
      GemmBatch ga1(false, false), gp(false, true), gb2(true, true), gg1(true, false), gg2(false, true);
      std::vector<PotrfProb> pp;
      std::vector<int> ppq;
      for (size_t q = 0; q < P; ++q) {
        const auto& p = pairs[q];
        const int k1 = p.kij, k2 = pairs[p.rev].kij;
        if (k1 == 0 || k2 == 0) continue;
        const double* Wi = Wb.p + boxw[p.i];
        const double* Wj = Wb.p + boxw[p.j];
        const int gj = t.quad[nodes[p.j]];
        GemmDesc a = gdesc(c, k1, p.ni);            // A1 = W_i^T U_ij
        a.A = Wi; a.lda = c; a.B = PL.U.p + p.uoff; a.ldb = p.ni; a.C = A1.p + a1off[q]; a.ldc = c;
        ga1.add(a);
        GemmDesc b = gdesc(c, c, p.ni);             // P = W_i^T Y_ij   (Y_ij^T stored c x ni)
        b.A = Wi; b.lda = c; b.B = Yg[gj].p + (long long)p.ib * cap; b.ldb = cap; b.C = Pm.p + poff[q]; b.ldc = c;
        gp.add(b);
        GemmDesc d = gdesc(k2, c, p.nj);            // B2 = U_ji^T W_j
        d.A = PL.U.p + pairs[p.rev].uoff; d.lda = p.nj; d.B = Wj; d.ldb = c; d.C = B2.p + b2off[q]; d.ldc = k2;
        gb2.add(d);
        GemmDesc e = gdesc(k1, k1, c);              // G1 = A1^T A1
        e.A = A1.p + a1off[q]; e.lda = c; e.B = A1.p + a1off[q]; e.ldb = c; e.C = G1.p + g1off[q]; e.ldc = k1;
        gg1.add(e);
        GemmDesc f = gdesc(k2, k2, c);              // G2 = B2 B2^T
        f.A = B2.p + b2off[q]; f.lda = k2; f.B = B2.p + b2off[q]; f.ldb = k2; f.C = G2.p + g2off[q]; f.ldc = k2;
        gg2.add(f);
        pp.push_back(PotrfProb{G1.p + g1off[q], k1, k1, G1i.p + g1off[q], k1});
        pp.push_back(PotrfProb{G2.p + g2off[q], k2, k2, G2i.p + g2off[q], k2});
        ppq.push_back((int)q);
        pd.flops += 2.0 * c * k1 * p.ni + 2.0 * c * c * p.ni + 2.0 * k2 * c * p.nj;
      }
      ga1.run(s);
      gp.run(s);
      gb2.run(s);
      gg1.run(s);
      gg2.run(s);
      DBuf<double> ls(std::max<size_t>(pp.size(), 1), s);
      DBuf<int> inf(std::max<size_t>(pp.size(), 1), s);
      potrf_batched(s, pp, ls.p, inf.p);
      {
        auto hi = inf.to_host(pp.size());
        for (size_t x = 0; x < hi.size(); ++x)
          if (hi[x]) throw Error(ST_ENUMERIC, "peeling: rank-deficient sketch product at level " + std::to_string(lev));
      }
      GemmBatch m1(true, false), m2(false, true), m3(false, false), m4(true, false), m5(false, true), m6(false, false);
      for (size_t q : ppq) {
        const auto& p = pairs[q];
        const int k1 = p.kij, k2 = pairs[p.rev].kij;
        GemmDesc a = gdesc(k1, c, c);     // T1 = A1^T P
        a.A = A1.p + a1off[q]; a.lda = c; a.B = Pm.p + poff[q]; a.ldb = c; a.C = T1.p + t1off[q]; a.ldc = k1;
        m1.add(a);
        GemmDesc b = gdesc(k1, k2, c);    // T2 = T1 B2^T
        b.A = T1.p + t1off[q]; b.lda = k1; b.B = B2.p + b2off[q]; b.ldb = k2; b.C = T2.p + t2off[q]; b.ldc = k1;
        m2.add(b);
        GemmDesc d = gdesc(k1, k2, k1);   // T3 = L1^-1 T2
        d.A = G1i.p + g1off[q]; d.lda = k1; d.B = T2.p + t2off[q]; d.ldb = k1; d.C = T3.p + t2off[q]; d.ldc = k1;
        m3.add(d);
        GemmDesc e = gdesc(k1, k2, k1);   // T2 = L1^-T T3
        e.A = G1i.p + g1off[q]; e.lda = k1; e.B = T3.p + t2off[q]; e.ldb = k1; e.C = T2.p + t2off[q]; e.ldc = k1;
        m4.add(e);
        GemmDesc f = gdesc(k1, k2, k2);   // T3 = T2 L2^-T
        f.A = T2.p + t2off[q]; f.lda = k1; f.B = G2i.p + g2off[q]; f.ldb = k2; f.C = T3.p + t2off[q]; f.ldc = k1;
        m5.add(f);
        GemmDesc g = gdesc(k1, k2, k2);   // M = T3 L2^-1
        g.A = T3.p + t2off[q]; g.lda = k1; g.B = G2i.p + g2off[q]; g.ldb = k2; g.C = PL.M.p + moff[q]; g.ldc = k1;
        m6.add(g);
        pairs[q].moff = moff[q];
      }
      m1.run(s); m2.run(s); m3.run(s); m4.run(s); m5.run(s); m6.run(s);
    }
    for (int g = 0; g < 4; ++g) Yg[g].release();

    // ---- subtraction batches for G^(lev):  Y'(I_i) -= sum_j X'(I_j) U_ji M_ij^T U_ij^T
    //      (one final GEMM per row box i over its concatenated [U_ij1 | U_ij2 | ...])
    PL.pairs = pairs;
    PL.g1.reset(false, false);
    PL.g2.reset(false, true);
    PL.g3.reset(false, true);
    long long tc = 0;
    std::vector<long long> t1o(pairs.size(), -1), t2o(pairs.size(), -1);
    for (size_t q = 0; q < pairs.size(); ++q) {
      const auto& p = PL.pairs[q];
      const int k1 = p.kij, k2 = PL.pairs[p.rev].kij;
      if (k1 > 0 && k2 > 0) { t1o[q] = tc; tc += k2; }
    }
    for (size_t q = 0; q < pairs.size(); ++q)
      if (PL.pairs[q].kij > 0) { t2o[q] = tc; tc += PL.pairs[q].kij; }
    for (size_t q = 0; q < pairs.size(); ++q) {
      const auto& p = PL.pairs[q];
      const int k1 = p.kij, k2 = PL.pairs[p.rev].kij;
      if (k1 == 0) continue;
      if (k2 > 0) {
        GemmDesc a = gdesc(-1, k2, p.nj);                 // t1 = X'(I_j) U_ji
        a.selA = 1; a.offA = p.jb; a.B = PL.U.p + PL.pairs[p.rev].uoff; a.ldb = p.nj; a.selC = 2; a.offC = t1o[q];
        PL.g1.add(a);
      }
      GemmDesc b = gdesc(-1, k1, k2);                     // t2 = t1 M_ij^T  (zero if k2 == 0)
      b.selA = 2; b.offA = k2 > 0 ? t1o[q] : 0; b.B = k2 > 0 ? PL.M.p + p.moff : PL.M.p; b.ldb = k1;
      b.selC = 2; b.offC = t2o[q];
      PL.g2.add(b);
    }
    for (size_t q = 0; q < pairs.size();) {
      size_t e = q;
      int ksum = 0;
      while (e < pairs.size() && PL.pairs[e].i == PL.pairs[q].i) { ksum += PL.pairs[e].kij; ++e; }
      if (ksum > 0) {
        size_t f = q;
        while (PL.pairs[f].kij == 0) ++f;
        const auto& p = PL.pairs[f];
        GemmDesc d = gdesc(-1, p.ni, ksum);               // Y'(I_i) -= [t2 ...] [U_ij ...]^T
        d.selA = 2; d.offA = t2o[f]; d.B = PL.U.p + p.uoff; d.ldb = p.ni; d.selC = 1; d.offC = p.ib;
        d.alpha = -1.0; d.beta = 1.0;
        PL.g3.add(d);
      }
      q = e;
    }
    PL.tcols = tc;
    max_tcols = std::max(max_tcols, tc);
    for (GemmBatch* g : {&PL.g1, &PL.g2, &PL.g3})
      if (!g->empty()) g->finalize(s);
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
  double tr = 0.0, tra = 0.0;
  const int GB = 256;
  for (int e0 = 0; e0 < nL; e0 += kb) {
    const int k = std::min(kb, nL - e0);
    DBuf<double> E((size_t)n * k, s), H((size_t)n * k, s), part(GB, s), parta(GB, s);
    extract_probe_kernel<<<gxx((long long)n * k), NT, 0, s>>>(E.p, k, n, dlb.p, e0);
    count_launch();
    RSF_LAUNCH_CHECK();
    residual(E.p, H.p, k, L + 1);
    extract_diag_kernel<<<GB, NT, 0, s>>>(H.p, k, n, dlb.p, e0, part.p, parta.p);
    count_launch();
    RSF_LAUNCH_CHECK();
    auto hp = part.to_host(GB), ha = parta.to_host(GB);
    for (int i = 0; i < GB; ++i) { tr += hp[i]; tra += ha[i]; }
  }
  pd.nL = nL;
  pd.cancellation = tr != 0.0 ? tra / std::fabs(tr) : INFINITY;
  pd.applies = G.columns;
  RSF_CUDA(cudaStreamSynchronize(s));
  pd.seconds = now_s() - t0;
  if (diag) *diag = pd;
  return tr;
}

void fill_peel_diag(const PeelDiag& d, rsf_peel_diag* out) {
  std::memset(out, 0, sizeof(*out));
  out->levels = (int)d.cols.size() - 1;
  for (size_t l = 0; l < d.cols.size() && l < 32; ++l) {
    out->cols[l] = d.cols[l];
    out->rank_max[l] = d.rank_max[l];
  }
  out->nL = d.nL;
  out->cancellation = d.cancellation;
  out->applies = d.applies;
  out->seconds = d.seconds;
}

// ----------------------------------------------------------------- Alg. 1
EvalResult mle_eval(Ctx& ctx, const double* xy, const double* z, int n, const KParams& kp, int p,
                    const int* theta, double eps, int leaf, const Opts& o) {
  EvalResult R;
  const long long l0 = g_launches;
  const double T0 = now_s();
  cudaStream_t s = ctx.stream;
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
  t = now_s();
  auto F = factor(ctx, tree, kp, W_SIGMA, eps, o);
  R.t_factor = now_s() - t;
  R.fdiag = F->diag;
  R.L = tree->L;
  R.n0 = F->n0;
  R.flops_factor = F->diag.flops_id + F->diag.flops_elim + F->diag.flops_top;
  R.logdet = F->logdet;
  // u = F^-1 z (k = 1), q0 = z^T u
  t = now_s();
  DBuf<double> zt(n, s), u(n, s), tmp((size_t)std::max<long long>(F->tmp_cols, 1), s);
  to_internal(s, *tree, dz, n, 1, zt.p);
  RSF_CUDA(cudaMemcpyAsync(u.p, zt.p, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  solve_internal(*F, u.p, 1, tmp.p);
  R.quad = ddot(s, zt.p, u.p, n);
  R.ell = -0.5 * R.quad - 0.5 * R.logdet - 0.5 * n * std::log(2.0 * M_PI);
  R.t_solve = now_s() - t;
  double trinv = NAN, utu = NAN;
  for (int i = 0; i < p; ++i) {
    const int w = theta[i];
    double q, tr;
    if (w == W_SIGMA2 || w == W_NUGGET) {   // reading R-G
      if (std::isnan(trinv)) {
        t = now_s();
        trinv = peel(*F, nullptr, o, 100, &R.pd[i]);
        R.t_peel += now_s() - t;
        utu = ddot(s, u.p, u.p, n);
      } else {
        R.pd[i] = R.pd[0];
      }
      if (w == W_NUGGET) { q = utu; tr = trinv; }
      else { q = (R.quad - kp.nugget * utu) / kp.sigma2; tr = (n - kp.nugget * trinv) / kp.sigma2; }
    } else {
      t = now_s();
      auto Fi = factor(ctx, tree, kp, w, eps, o);
      R.t_compress += now_s() - t;
      R.flops_factor += Fi->diag.flops_id + Fi->diag.flops_elim;
      t = now_s();
      DBuf<double> x(n, s), y(n, s);
      RSF_CUDA(cudaMemcpyAsync(x.p, u.p, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
      apply_only_internal(*Fi, x.p, y.p, 1);
      q = ddot(s, u.p, y.p, n);
      R.t_solve += now_s() - t;
      t = now_s();
      tr = peel(*F, Fi.get(), o, i, &R.pd[i]);
      R.t_peel += now_s() - t;
    }
    R.q[i] = q;
    R.trace[i] = tr;
    R.grad[i] = 0.5 * q - 0.5 * tr;
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

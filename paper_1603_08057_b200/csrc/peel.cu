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

// U (ni x k, ld ni) <- [I_k; 0]
struct EyeDesc { double* U; int ni, k; };
__global__ void eye_kernel(const EyeDesc* __restrict__ descs) {
  const EyeDesc d = descs[blockIdx.y];
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < (long long)d.ni * d.k; e += (long long)gridDim.x * NT) {
    const int r = (int)(e % d.ni), c = (int)(e / d.ni);
    d.U[e] = (r == c) ? 1.0 : 0.0;
  }
}

// Y_k (n_i x k, ld n_i) <- probe columns piv[0:k] of the sketch rows of box i,
// read from the column chunks of Y_g (chunk c holds probe columns [c*kb, ...), X' layout)
struct GatherDesc { double* Yk; const int* piv; int ib, ni, k; };
__global__ void gather_cols_kernel(const GatherDesc* __restrict__ descs, double* const* __restrict__ chunks,
                                   const int* __restrict__ chw, int kb) {
  const GatherDesc d = descs[blockIdx.y];
  const long long tot = (long long)d.ni * d.k;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    const int t = (int)(e % d.ni), j = (int)(e / d.ni);
    const int col = __ldg(d.piv + j), ch = col / kb, w = __ldg(chw + ch);
    d.Yk[e] = chunks[ch][(long long)(d.ib + t) * w + (col - ch * kb)];
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
    RSF_PHASE("p.G_apply", s);
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
  std::vector<DBuf<double>> Ubufs;
  GemmBatch g1, g2, g3;
  std::vector<GemmBatch> g3s;
  long long tcols = 0;   // temp columns per probe column
  bool empty() const { return g1.empty(); }
  // Y' -= G^(m) X'   (X', Y' are k x n; tmp has k * tcols doubles)
  void subtract(cudaStream_t s, const double* X, double* Y, int k, double* tmp) const {
    if (g2.empty()) return;
    g1.run(s, const_cast<double*>(X), tmp, k, k);
    g2.run(s, nullptr, tmp, k, k);
    for (const auto& g : g3s) g.run(s, Y, tmp, k, k);
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
  const unsigned seed32 = (unsigned)(seed & 0xffffffffull);
  GOp G(F, Fi);
  std::vector<PeelLevel> peeled(L + 1);
  long long max_tcols = 0;
  PeelDiag pd;
  pd.cols.assign(L + 1, 0);
  pd.rank_max.assign(L + 1, 0);
  int prev_rank = -1;
  const int kb = std::max(16, o.probe_block);
  const double budget = 24.0 * (1ull << 30);   // bytes of transient per-batch buffers

  auto residual = [&](const double* W, double* Y, int k, int upto) {
    G.apply(W, Y, k);
    DBuf<double> tmp((size_t)std::max<long long>(max_tcols, 1) * k, s);
    RSF_PHASE("p.subtract", s);
    for (int m = 1; m < upto; ++m) peeled[m].subtract(s, W, Y, k, tmp.p);
  };

  for (int lev = 1; lev <= L; ++lev) {
    const std::vector<int>& nodes = t.levels[lev];
    const int nb = (int)nodes.size();
    // ordered sibling pairs (Def. sibs), grouped by the probe group quad(j)
    std::vector<PairLR> pairs;
    std::unordered_map<int, std::vector<int>> fam;
    for (int b = 0; b < nb; ++b) fam[t.parent[nodes[b]]].push_back(b);
    for (int b = 0; b < nb; ++b) {
      for (int c2 : fam[t.parent[nodes[b]]]) {
        if (c2 == b) continue;
        PairLR p;
        p.i = b; p.j = c2;
        p.ib = t.begin[nodes[b]]; p.ni = t.end[nodes[b]] - p.ib;
        p.jb = t.begin[nodes[c2]]; p.nj = t.end[nodes[c2]] - p.jb;
        pairs.push_back(p);
      }
    }
    if (pairs.empty()) continue;
    const size_t P = pairs.size();
    {
      std::unordered_map<long long, int> idx;
      for (int q = 0; q < (int)P; ++q) idx[(long long)pairs[q].i * nb + pairs[q].j] = q;
      for (auto& p : pairs) p.rev = idx[(long long)p.j * nb + p.i];
    }
    std::vector<std::vector<int>> grp(4);
    for (size_t q = 0; q < P; ++q) grp[t.quad[nodes[pairs[q].j]]].push_back((int)q);
    std::vector<int> gorder = {0, 1, 2, 3};
    std::stable_sort(gorder.begin(), gorder.end(), [&](int a2, int b2) { return grp[a2].size() > grp[b2].size(); });
    std::vector<int> hq(n, -1);
    int maxni = 0;
    for (int b = 0; b < nb; ++b) {
      const int nd = nodes[b];
      for (int x = t.begin[nd]; x < t.end[nd]; ++x) hq[x] = t.quad[nd];
      maxni = std::max(maxni, t.end[nd] - t.begin[nd]);
    }
    DBuf<int> qmap = up(hq, s);
    const int cmax = ((maxni + o.oversample) + 7) / 8 * 8;
    // initial width: level 1 from the factor's level-1 skeleton sizes (ranks of Sigma's
    // off-diagonal blocks at eps_fact); deeper levels from the previous level's ranks (R-M)
    int hint = o.peel_start;
    if (prev_rank < 0 && F.levels.size() > 1)
      for (int kk : F.levels[1].k) hint = std::max(hint, kk);
    int c = (prev_rank < 0) ? (int)std::ceil(0.6 * hint) : prev_rank + o.oversample;
    c = std::min(std::max(c, o.oversample + 8), cmax);
    c = (c + 7) / 8 * 8;

    PeelLevel& PL = peeled[lev];
    std::vector<DBuf<double>> keep;          // U, A1, P buffers of this level
    std::vector<double*> Up(P, nullptr), A1p(P, nullptr), Pp(P, nullptr);
    std::vector<int> kp(P, 0);
    int mr = 0;
    while (true) {
      keep.clear();
      bool fail = false;
      mr = 0;
      for (int g : gorder) {
        if (grp[g].empty()) continue;
        // sketch Y_g = (G - sum_{m<l} G^(m)) W_g in column chunks
        std::vector<DBuf<double>> ych;
        std::vector<int> ycs, ykk;
        for (int c0 = 0; c0 < c; c0 += kb) {
          const int k = std::min(kb, c - c0);
          DBuf<double> W((size_t)n * k, s), Y((size_t)n * k, s);
          gen_probes(s, W.p, k, n, t.d_perm.p, qmap.p, g, c0, lev, trace_id, seed);
          residual(W.p, Y.p, k, lev);
          ych.push_back(std::move(Y));
          ycs.push_back(c0);
          ykk.push_back(k);
        }
        // pair batches under the byte budget
        const std::vector<int>& gq = grp[g];
        size_t q0 = 0;
        while (q0 < gq.size() && !fail) {
          size_t q1 = q0;
          double bytes = 0;
          while (q1 < gq.size()) {
            const auto& p = pairs[gq[q1]];
            const double bb = 8.0 * (3.0 * p.ni * (double)c + 3.0 * (double)c * c);
            if (q1 > q0 && bytes + bb > budget) break;
            bytes += bb;
            ++q1;
          }
          const size_t B = q1 - q0;
          // per pair: W_i^T (c x n_i), P = W_i^T Y_ij (c x c), Pc (RRQR copy)
          std::vector<long long> wo(B), po(B);
          long long wt = 0, pt = 0;
          for (size_t x = 0; x < B; ++x) {
            const auto& p = pairs[gq[q0 + x]];
            wo[x] = wt; wt += (long long)c * p.ni;
            po[x] = pt; pt += (long long)c * c;
          }
          DBuf<double> Wi(wt, s), Pb(pt, s), Pc(pt, s);
          DBuf<int> dpv((size_t)c * B, s);
          std::vector<int> kk;
          {
            RSF_PHASE("p.sketch_rank", s);
            GemmBatch gp(false, true);   // P_ij(:, chunk cols) = W_i^T (Y_chunk(:, I_i))^T
            for (size_t x = 0; x < B; ++x) {
              const auto& p = pairs[gq[q0 + x]];
              // W_i^T: the same Philox entries as in the sketches
              probes_kernel<<<gxx((long long)p.ni * c), NT, 0, s>>>(Wi.p + wo[x], c, p.ib, p.ib + p.ni, t.d_perm.p,
                                                                  nullptr, 0, 0, lev, trace_id, seed32, c);
              count_launch();
              for (size_t ci = 0; ci < ych.size(); ++ci) {
                GemmDesc d = gdesc(c, ykk[ci], p.ni);
                d.A = Wi.p + wo[x]; d.lda = c;
                d.B = ych[ci].p + (long long)p.ib * ykk[ci]; d.ldb = ykk[ci];
                d.C = Pb.p + po[x] + (long long)ycs[ci] * c; d.ldc = c;
                gp.add(d);
              }
              pd.flops += 2.0 * c * (double)c * p.ni;
            }
            RSF_LAUNCH_CHECK();
            gp.run(s);
            RSF_CUDA(cudaMemcpyAsync(Pc.p, Pb.p, pt * sizeof(double), cudaMemcpyDeviceToDevice, s));
            // rank and column pivots of Y_ij from its Gaussian row sketch P_ij (R-N)
            std::vector<RRQRProb> rp;
            for (size_t x = 0; x < B; ++x)
              rp.push_back(RRQRProb{Pc.p + po[x], c, c, c, dpv.p + (long long)x * c, nullptr, nullptr, 0});
            RRQRResult rr = rrqr_batched(s, rp, o.eps_peel,
                                         seed ^ (0xD1B54A32D192ED03ull * (unsigned long long)(lev + 64 * (trace_id + 1))));
            kk = rr.k;
          }
          for (size_t x = 0; x < B; ++x) mr = std::max(mr, kk[x]);
          if (mr > c - o.oversample && c < cmax) { fail = true; break; }
          // U_ij = orth(Y_ij(:, piv[0:k])): preconditioned CholeskyQR2
          //   U0 = Y_k R11^-1 (R11 from the sketch RRQR; W_i^T U0 has orthonormal columns),
          //   then twice U <- U chol(U^T U)^-T
          long long ut = 0, at = 0, kt = 0, rt = 0;
          std::vector<long long> uo(B), ao(B), ko(B), ro(B);
          for (size_t x = 0; x < B; ++x) {
            const auto& p = pairs[gq[q0 + x]];
            uo[x] = ut; ut += (long long)p.ni * kk[x];
            ao[x] = at; at += (long long)c * kk[x];
            ko[x] = kt; kt += (long long)kk[x] * kk[x];
          }
          DBuf<double> Ub(std::max<long long>(ut, 1), s), Ab(std::max<long long>(at, 1), s);
          {
            RSF_PHASE("p.form_U", s);
            DBuf<double> Yk(std::max<long long>(ut, 1), s), U0(std::max<long long>(ut, 1), s);
            DBuf<double> Ri(std::max<long long>(kt, 1), s), G1(std::max<long long>(kt, 1), s), G1i(std::max<long long>(kt, 1), s);
            // gather Y_k from the chunks
            std::vector<double*> chp;
            std::vector<int> chw;
            for (size_t ci = 0; ci < ych.size(); ++ci) { chp.push_back(ych[ci].p); chw.push_back(ykk[ci]); }
            DBuf<double*> dchp = up(chp, s);
            DBuf<int> dchw = up(chw, s);
            std::vector<GatherDesc> gd;
            std::vector<EyeDesc> ed;
            std::vector<TrsmProb> tp;
            long long mx = 0;
            for (size_t x = 0; x < B; ++x) {
              const auto& p = pairs[gq[q0 + x]];
              if (kk[x] == 0) continue;
              gd.push_back(GatherDesc{Yk.p + uo[x], dpv.p + (long long)x * c, p.ib, p.ni, kk[x]});
              ed.push_back(EyeDesc{Ri.p + ko[x], kk[x], kk[x]});
              tp.push_back(TrsmProb{Pc.p + po[x], c, Ri.p + ko[x], kk[x], kk[x], kk[x]});
              mx = std::max(mx, (long long)p.ni * kk[x]);
            }
            if (!gd.empty()) {
              auto dg = up(gd, s);
              for (size_t o2 = 0; o2 < gd.size(); o2 += 65535) {
                unsigned nz = (unsigned)std::min<size_t>(65535, gd.size() - o2);
                gather_cols_kernel<<<dim3(gxx(mx), nz), NT, 0, s>>>(dg.p + o2, dchp.p, dchw.p, kb);
                count_launch();
              }
              auto de = up(ed, s);
              for (size_t o2 = 0; o2 < ed.size(); o2 += 65535) {
                unsigned nz = (unsigned)std::min<size_t>(65535, ed.size() - o2);
                eye_kernel<<<dim3(gxx(mx), nz), NT, 0, s>>>(de.p + o2);
                count_launch();
              }
              RSF_LAUNCH_CHECK();
              trsm_upper_batched(s, tp);                 // Ri = R11^-1
              GemmBatch g0(false, false);
              for (size_t x = 0; x < B; ++x) {
                const auto& p = pairs[gq[q0 + x]];
                if (kk[x] == 0) continue;
                GemmDesc d = gdesc(p.ni, kk[x], kk[x]);   // U0 = Y_k R11^-1
                d.A = Yk.p + uo[x]; d.lda = p.ni; d.B = Ri.p + ko[x]; d.ldb = kk[x]; d.C = U0.p + uo[x]; d.ldc = p.ni;
                g0.add(d);
              }
              g0.run(s);
              for (int pass = 0; pass < 2; ++pass) {
                double* src = pass == 0 ? U0.p : Yk.p;   // U1 lives in Yk, U in Ub
                double* dst = pass == 0 ? Yk.p : Ub.p;
                GemmBatch gg(true, false), gu(false, true);
                std::vector<PotrfProb> pp;
                for (size_t x = 0; x < B; ++x) {
                  const auto& p = pairs[gq[q0 + x]];
                  if (kk[x] == 0) continue;
                  GemmDesc d = gdesc(kk[x], kk[x], p.ni);     // Gram = U^T U
                  d.A = src + uo[x]; d.lda = p.ni; d.B = src + uo[x]; d.ldb = p.ni; d.C = G1.p + ko[x]; d.ldc = kk[x];
                  gg.add(d);
                  pp.push_back(PotrfProb{G1.p + ko[x], kk[x], kk[x], G1i.p + ko[x], kk[x]});
                  GemmDesc e = gdesc(p.ni, kk[x], kk[x]);     // U <- U L^-T
                  e.A = src + uo[x]; e.lda = p.ni; e.B = G1i.p + ko[x]; e.ldb = kk[x]; e.C = dst + uo[x]; e.ldc = p.ni;
                  gu.add(e);
                  pd.flops += 4.0 * p.ni * (double)kk[x] * kk[x];
                }
                gg.run(s);
                DBuf<double> ls(std::max<size_t>(pp.size(), 1), s);
                DBuf<int> inf(std::max<size_t>(pp.size(), 1), s);
                potrf_batched(s, pp, ls.p, inf.p);
                auto hi = inf.to_host(pp.size());
                for (int v : hi)
                  if (v) throw Error(ST_ENUMERIC, "peeling: CholeskyQR of the skeleton sketch columns failed at level " +
                                                      std::to_string(lev));
                gu.run(s);
              }
              GemmBatch ga(false, false);
              for (size_t x = 0; x < B; ++x) {
                const auto& p = pairs[gq[q0 + x]];
                if (kk[x] == 0) continue;
                GemmDesc d = gdesc(c, kk[x], p.ni);            // A1 = W_i^T U_ij
                d.A = Wi.p + wo[x]; d.lda = c; d.B = Ub.p + uo[x]; d.ldb = p.ni; d.C = Ab.p + ao[x]; d.ldc = c;
                ga.add(d);
              }
              ga.run(s);
            }
          }
          for (size_t x = 0; x < B; ++x) {
            const int q = gq[q0 + x];
            kp[q] = kk[x];
            Up[q] = Ub.p + uo[x];
            A1p[q] = Ab.p + ao[x];
            Pp[q] = Pb.p + po[x];
          }
          keep.push_back(std::move(Ub));
          keep.push_back(std::move(Ab));
          keep.push_back(std::move(Pb));
          q0 = q1;
        }
        if (fail) break;
      }
      if (!fail) break;
      int nc = (mr >= c - 1) ? (int)std::ceil(1.4 * c) : std::max(c + 8, (int)std::ceil(1.1 * mr) + o.oversample);
      c = std::max(std::min((nc + 7) / 8 * 8, cmax), c + 8);
    }
    pd.cols[lev] = c;
    pd.rank_max[lev] = mr;
    prev_rank = mr;

    // ---- cores M_ij = (A1_ij)^+ P_ij (A1_ji^T)^+   (Eq. lowrankapprox; U_ji^T W_j = A1_ji^T)
    DBuf<double> Mbuf;
    std::vector<long long> moff(P, -1);
    {
      RSF_PHASE("p.cores", s);
      std::vector<long long> g1o(P), t1o(P), t2o(P);
      long long g1t = 0, t1t = 0, t2t = 0, mt = 0;
      for (size_t q = 0; q < P; ++q) {
        const int k1 = kp[q], k2 = kp[pairs[q].rev];
        g1o[q] = g1t; g1t += (long long)k1 * k1;
        t1o[q] = t1t; t1t += (long long)k1 * c;
        t2o[q] = t2t; t2t += (long long)k1 * k2;
        if (k1 > 0 && k2 > 0) { moff[q] = mt; mt += (long long)k1 * k2; }
      }
      DBuf<double> G1(std::max<long long>(g1t, 1), s), G1i(std::max<long long>(g1t, 1), s),
          T1(std::max<long long>(t1t, 1), s), T2(std::max<long long>(t2t, 1), s), T3(std::max<long long>(t2t, 1), s);
      Mbuf.alloc(std::max<long long>(mt, 1), s);
      GemmBatch gg(true, false);
      std::vector<PotrfProb> pp;
      for (size_t q = 0; q < P; ++q) {
        const int k1 = kp[q];
        if (k1 == 0) continue;
        GemmDesc e = gdesc(k1, k1, c);              // G1 = A1^T A1
        e.A = A1p[q]; e.lda = c; e.B = A1p[q]; e.ldb = c; e.C = G1.p + g1o[q]; e.ldc = k1;
        gg.add(e);
        pp.push_back(PotrfProb{G1.p + g1o[q], k1, k1, G1i.p + g1o[q], k1});
      }
      gg.run(s);
      DBuf<double> ls(std::max<size_t>(pp.size(), 1), s);
      DBuf<int> inf(std::max<size_t>(pp.size(), 1), s);
      potrf_batched(s, pp, ls.p, inf.p);
      {
        auto hi = inf.to_host(pp.size());
        for (size_t x = 0; x < hi.size(); ++x)
          if (hi[x]) throw Error(ST_ENUMERIC, "peeling: rank-deficient sketch product at level " + std::to_string(lev));
      }
      GemmBatch m1(true, false), m2(false, false), m3(false, false), m4(true, false), m5(false, true), m6(false, false);
      for (size_t q = 0; q < P; ++q) {
        const int k1 = kp[q], rq = pairs[q].rev, k2 = kp[rq];
        if (moff[q] < 0) continue;
        const double* L1i = G1i.p + g1o[q];
        const double* L2i = G1i.p + g1o[rq];
        GemmDesc a = gdesc(k1, c, c);     // T1 = A1_ij^T P_ij
        a.A = A1p[q]; a.lda = c; a.B = Pp[q]; a.ldb = c; a.C = T1.p + t1o[q]; a.ldc = k1;
        m1.add(a);
        GemmDesc b = gdesc(k1, k2, c);    // T2 = T1 A1_ji
        b.A = T1.p + t1o[q]; b.lda = k1; b.B = A1p[rq]; b.ldb = c; b.C = T2.p + t2o[q]; b.ldc = k1;
        m2.add(b);
        GemmDesc d = gdesc(k1, k2, k1);   // T3 = L1^-1 T2
        d.A = L1i; d.lda = k1; d.B = T2.p + t2o[q]; d.ldb = k1; d.C = T3.p + t2o[q]; d.ldc = k1;
        m3.add(d);
        GemmDesc e = gdesc(k1, k2, k1);   // T2 = L1^-T T3
        e.A = L1i; e.lda = k1; e.B = T3.p + t2o[q]; e.ldb = k1; e.C = T2.p + t2o[q]; e.ldc = k1;
        m4.add(e);
        GemmDesc f = gdesc(k1, k2, k2);   // T3 = T2 L2^-T
        f.A = T2.p + t2o[q]; f.lda = k1; f.B = L2i; f.ldb = k2; f.C = T3.p + t2o[q]; f.ldc = k1;
        m5.add(f);
        GemmDesc g2 = gdesc(k1, k2, k2);  // M = T3 L2^-1
        g2.A = T3.p + t2o[q]; g2.lda = k1; g2.B = L2i; g2.ldb = k2; g2.C = Mbuf.p + moff[q]; g2.ldc = k1;
        m6.add(g2);
        pd.flops += 2.0 * k1 * (double)c * c + 2.0 * k1 * (double)k2 * c;
      }
      m1.run(s); m2.run(s); m3.run(s); m4.run(s); m5.run(s); m6.run(s);
    }
    // keep U (persistent) and M; drop A1 / P
    std::vector<DBuf<double>> Ukeep;
    for (size_t x = 0; x < keep.size(); x += 3) Ukeep.push_back(std::move(keep[x]));
    keep.clear();

    // ---- subtraction batches for G^(lev):  Y'(I_i) -= sum_j X'(I_j) U_ji M_ij^T U_ij^T
    //      one final GEMM per (row box i, U buffer) over its concatenated [U_ij1 | U_ij2 | ...]
    for (size_t q = 0; q < P; ++q) { pairs[q].kij = kp[q]; pairs[q].moff = moff[q]; }
    PL.pairs = pairs;
    PL.U = DBuf<double>();
    PL.M = std::move(Mbuf);
    PL.Ubufs = std::move(Ukeep);
    PL.g1.reset(false, false);
    PL.g2.reset(false, true);
    PL.g3.reset(false, true);
    long long tc = 0;
    std::vector<long long> t1o(P, -1), t2o(P, -1);
    for (size_t q = 0; q < P; ++q) {
      const int k1 = kp[q], k2 = kp[pairs[q].rev];
      if (k1 > 0 && k2 > 0) { t1o[q] = tc; tc += k2; }
    }
    // t2 columns grouped by row box i (pairs are generated in row-box order)
    for (size_t q = 0; q < P; ++q)
      if (kp[q] > 0) { t2o[q] = tc; tc += kp[q]; }
    for (size_t q = 0; q < P; ++q) {
      const auto& p = PL.pairs[q];
      const int k1 = kp[q], k2 = kp[p.rev];
      if (k1 == 0) continue;
      if (k2 > 0) {
        GemmDesc a = gdesc(-1, k2, p.nj);                 // t1 = X'(I_j) U_ji
        a.selA = 1; a.offA = p.jb; a.B = Up[p.rev]; a.ldb = p.nj; a.selC = 2; a.offC = t1o[q];
        PL.g1.add(a);
      }
      GemmDesc b = gdesc(-1, k1, k2);                     // t2 = t1 M_ij^T  (zero if k2 == 0)
      b.selA = 2; b.offA = k2 > 0 ? t1o[q] : 0; b.B = k2 > 0 ? PL.M.p + moff[q] : PL.M.p; b.ldb = k1;
      b.selC = 2; b.offC = t2o[q];
      PL.g2.add(b);
    }
    // Y'(I_i) -= t2 U_ij^T: one GEMM per row box i when its U_ij are contiguous, else per pair
    // (pairs of one row box live in different group buffers, so they are never contiguous;
    //  the per-pair GEMMs of one row box are issued in separate batches to avoid races)
    {
      std::vector<std::vector<int>> byrow(nb);
      for (size_t q = 0; q < P; ++q) if (kp[q] > 0) byrow[pairs[q].i].push_back((int)q);
      size_t maxdeg = 0;
      for (auto& v : byrow) maxdeg = std::max(maxdeg, v.size());
      PL.g3s.clear();
      for (size_t r = 0; r < maxdeg; ++r) {
        PL.g3s.emplace_back(false, true);
        for (int b = 0; b < nb; ++b) {
          if (r >= byrow[b].size()) continue;
          const int q = byrow[b][r];
          const auto& p = PL.pairs[q];
          GemmDesc d = gdesc(-1, p.ni, kp[q]);
          d.selA = 2; d.offA = t2o[q]; d.B = Up[q]; d.ldb = p.ni; d.selC = 1; d.offC = p.ib;
          d.alpha = -1.0; d.beta = 1.0;
          PL.g3s.back().add(d);
        }
      }
    }
    PL.tcols = tc;
    max_tcols = std::max(max_tcols, tc);
    for (GemmBatch* g : {&PL.g1, &PL.g2})
      if (!g->empty()) g->finalize(s);
    for (auto& g : PL.g3s) if (!g.empty()) g.finalize(s);
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

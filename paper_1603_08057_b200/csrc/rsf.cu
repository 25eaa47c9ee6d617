// Recursive skeletonization factorization F ~ Sigma (PAPER §2) and
// the apply-only compression of Sigma_i (reading R-F), level by level over the
// quadtree with every box of a level in one batched launch per step:
//
//   per level l = L..1:
//     near lists N_b + proxy annulus Gamma_b            (host schedule)
//     A_b = [K(N_b,I_b); K(Gamma_b,I_b)]                 assemble_id      (a4)
//     R_b = qr(A_b); (S,R,T) = cpqr-ID(R_b, eps)         geqrf + cpqr     (a5, Def. id)
//     B_b (self block), Bp = B(piv,piv)                  assemble_self / permute
//     X_SR, X_RR; L = chol(X_RR); E = X_SR L^-T; B_SS -= E E^T      (a6)
//   top: B_0 = [modified B_SS ; original cross blocks], C = chol(B_0)  (a7)
//
// Operators act on X' = (n x k RHS block)^T in tree order, one
// batched GEMM launch per (level, step); descriptors are built here once.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <mutex>
#include <numeric>
#include <unordered_set>

#include "dense.cuh"
#include "rsf_impl.cuh"
#include "rrqr.cuh"
#include "rsf_kernels.cuh"

namespace rsf {

namespace {

constexpr int N_RINGS = 4, N_ANGLES = 64;   // n_prox = 256, R-C
constexpr long long CHUNK_ELEMS = 1ll << 28; // max doubles of ID matrices per launch group
// |I| <= SMALL_C: exact greedy CPQR, one CTA per box (shared memory, global workspace when the
// block does not fit); larger boxes: the blocked randomized RRQR (RSF_SMALL_C overrides)
static const int SMALL_C = getenv("RSF_SMALL_C") ? atoi(getenv("RSF_SMALL_C")) : 128;

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

inline GemmDesc tri(GemmDesc d, int t) { d.btri = t; return d; }   // triangular op(B)

}  // namespace

cudaStream_t& stream_override() { static thread_local cudaStream_t s = nullptr; return s; }

namespace {

struct BRef {
  const double* Bp = nullptr;   // permuted self block of a processed node (B_SS at top-left)
  int ld = 0;
  int k = 0;
};

}  // namespace

// per-level phase names for RSF_PROFILE=1 (diagnostics)
static const char* lvname(const char* op, int lev) {
  static std::vector<std::string> names;
  static std::mutex mu;
  if (!phase_names_on()) return op;
  std::lock_guard<std::mutex> lk(mu);
  const std::string key = std::string(op) + ".L" + std::to_string(lev);
  for (size_t i = 0; i < names.size(); ++i) if (names[i] == key) return names[i].c_str();
  if (names.empty()) names.reserve(4096);   // stable c_str() pointers
  if (names.size() >= 4096) return op;
  names.push_back(key);
  return names.back().c_str();
}

std::unique_ptr<Fact> factor(Ctx& ctx, std::shared_ptr<Tree> tree, const KParams& kp, int which,
                             double eps, const Opts& opts, bool solve_only) {
  RSF_REQUIRE(eps > 0.0, ST_EINVAL, "eps must be > 0");
  const double t0 = now_s();
  cudaStream_t s = ctx_stream(ctx);
  auto F = std::make_unique<Fact>();
  F->ctx = &ctx;
  F->which = which;
  F->solve_only = solve_only && which == W_SIGMA;
  F->kp = kp;
  F->eps = eps;
  F->opts = opts;
  F->tree = tree;
  const Tree& t = *tree;
  const int L = t.L;
  const int nnodes = (int)t.lev.size();
  const bool sig = (which == W_SIGMA);
  F->levels.resize(L + 1);

  std::vector<std::vector<int>> Snode(nnodes);   // skeletons of processed nodes
  std::vector<BRef> bref(nnodes);
  DBuf<double> Bp_prev;
  double logdet = 0.0;

  for (int lev = L; lev >= 1; --lev) {
    RSF_PHASE(lvname(sig ? "fS" : "fI", lev), s);
    Level& LV = F->levels[lev];
    LV.lev = lev;
    const std::vector<int>& nodes = t.levels[lev];
    const int nb = (int)nodes.size();
    LV.nbox = nb;
    LV.node = nodes;
    std::unordered_map<int, int> boxof;
    boxof.reserve(nb * 2);
    for (int b = 0; b < nb; ++b) boxof[nodes[b]] = b;

    // ---- active sets I_b (leaf: its points; parent: children's skeletons)
    std::vector<std::vector<int>> I(nb);
    std::vector<std::array<int, 5>> choff(nb);
    std::vector<int> nch(nb, 0);
    for (int b = 0; b < nb; ++b) {
      const int nd = nodes[b];
      if (t.is_leaf(nd)) {
        I[b].resize(t.end[nd] - t.begin[nd]);
        std::iota(I[b].begin(), I[b].end(), t.begin[nd]);
      } else {
        choff[b][0] = 0;
        for (int q = 0; q < 4; ++q) {
          const int ch = t.child[nd][q];
          if (ch < 0) continue;
          I[b].insert(I[b].end(), Snode[ch].begin(), Snode[ch].end());
          choff[b][++nch[b]] = (int)I[b].size();
        }
      }
    }
    // ---- near lists (R-C, R-E): active DOFs outside b within r_near * h of its center
    std::vector<std::vector<int>> N(nb);
    {
    RSF_PHASE("f.near_host", s);
    for (int b = 0; b < nb; ++b) {
      const int nd = nodes[b];
      const double cx = t.cx(nd), cy = t.cy(nd), h = t.h(nd);
      const double rad = opts.r_near * h, rad2 = rad * rad;
      const int side = 1 << lev;
      std::vector<int> seen;
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          if (!dx && !dy) continue;
          const int nx = t.ix[nd] + dx, ny = t.iy[nd] + dy;
          if (nx < 0 || ny < 0 || nx >= side || ny >= side) continue;
          const std::vector<int>* cand = nullptr;
          std::vector<int> leafpts;
          int id = t.find(lev, nx, ny);
          if (id >= 0) {
            cand = &I[boxof[id]];
          } else {
            for (int l2 = lev - 1; l2 >= 0; --l2) {
              int a = t.find(l2, nx >> (lev - l2), ny >> (lev - l2));
              if (a < 0) continue;
              if (t.is_leaf(a) && std::find(seen.begin(), seen.end(), a) == seen.end()) {
                seen.push_back(a);
                leafpts.resize(t.end[a] - t.begin[a]);
                std::iota(leafpts.begin(), leafpts.end(), t.begin[a]);
                cand = &leafpts;
              }
              break;
            }
          }
          if (!cand) continue;
          for (int p : *cand) {
            const double ddx = t.hx[p] - cx, ddy = t.hy[p] - cy;
            if (ddx * ddx + ddy * ddy < rad2) N[b].push_back(p);
          }
        }
    }

    }
    // ---- interpolative decompositions, in chunks of boxes
    std::vector<int> cvec(nb), kvec(nb, 0);
    std::vector<std::vector<int>> piv(nb);
    std::vector<long long> tfoff(nb);   // T (ld c) offsets in Tfull
    long long tftot = 0;
    for (int b = 0; b < nb; ++b) {
      cvec[b] = (int)I[b].size();
      tfoff[b] = tftot;
      tftot += (long long)cvec[b] * cvec[b];
    }
    DBuf<double> Tfull(std::max<long long>(tftot, 1), s);
    int b0 = 0;
    while (b0 < nb) {
      long long tot = 0;
      int b1 = b0;
      while (b1 < nb) {
        long long e = (long long)(N[b1].size() + N_RINGS * N_ANGLES) * cvec[b1];
        if (b1 > b0 && tot + e > CHUNK_ELEMS) break;
        tot += e;
        ++b1;
      }
      // device index lists
      std::vector<int> hI, hN;
      std::vector<long long> ioff(b1 - b0), noff(b1 - b0), aoff(b1 - b0);
      long long at = 0;
      for (int b = b0; b < b1; ++b) {
        ioff[b - b0] = hI.size();
        hI.insert(hI.end(), I[b].begin(), I[b].end());
        noff[b - b0] = hN.size();
        hN.insert(hN.end(), N[b].begin(), N[b].end());
        aoff[b - b0] = at;
        at += (long long)(N[b].size() + N_RINGS * N_ANGLES) * cvec[b];
      }
      DBuf<int> dI(std::max<size_t>(hI.size(), 1), s), dN(std::max<size_t>(hN.size(), 1), s);
      dI.upload(hI);
      dN.upload(hN);
      DBuf<double> A(std::max<long long>(at, 1), s);
      std::vector<IdAsmDesc> ad;
      std::vector<QRProb> qp;
      std::vector<CPQRProb> cp;
      long long wtot = 0;
      std::vector<long long> woff(b1 - b0, -1);
      for (int b = b0; b < b1; ++b) {
        const int m = (int)N[b].size() + N_RINGS * N_ANGLES, c = cvec[b];
        const int q = std::min(m, c);
        if (c <= SMALL_C && (size_t)q * c * 8 + (72 + 2 * (size_t)c + 64) * 8 > 200 * 1024) {
          woff[b - b0] = wtot;
          wtot += (long long)q * c;
        }
      }
      DBuf<double> Wcp(std::max<long long>(wtot, 1), s);
      DBuf<int> dpiv(std::max<size_t>(hI.size(), 1), s);
      std::vector<int> big, sm;   // boxes on the blocked randomized RRQR path / greedy smem path
      for (int b = b0; b < b1; ++b) {
        const int nd = nodes[b];
        const int m = (int)N[b].size() + N_RINGS * N_ANGLES, c = cvec[b];
        IdAsmDesc d;
        d.A = A.p + aoff[b - b0];
        d.m_near = (int)N[b].size();
        d.c = c;
        d.near = dN.p + noff[b - b0];
        d.I = dI.p + ioff[b - b0];
        d.cx = t.cx(nd); d.cy = t.cy(nd); d.h = t.h(nd);
        ad.push_back(d);
        if (c > SMALL_C) {
          big.push_back(b);
        } else {
          sm.push_back(b);
          qp.push_back(QRProb{A.p + aoff[b - b0], m, m, c, nullptr, nullptr});
          CPQRProb p;
          p.R = A.p + aoff[b - b0]; p.ldr = m; p.q = std::min(m, c); p.c = c;
          p.W = woff[b - b0] >= 0 ? Wcp.p + woff[b - b0] : nullptr;
          p.T = Tfull.p + tfoff[b];
          p.piv = dpiv.p + ioff[b - b0];
          p.Rout = nullptr; p.tau = nullptr;
          cp.push_back(p);
          F->diag.flops_id += 2.0 * m * (double)c * c - (2.0 / 3.0) * (double)c * c * c + (4.0 / 3.0) * (double)c * c * c;
        }
      }
      { RSF_PHASE("f.assemble_id", s); assemble_id(s, ad, kp, which, opts, t.xs.p, t.ys.p, N_RINGS, N_ANGLES); }
      std::vector<int> hk(b1 - b0, 0);
      if (!cp.empty()) {
        DBuf<int> dks(cp.size(), s);
        { RSF_PHASE("f.geqrf", s); geqrf_batched(s, qp, false); }
        { RSF_PHASE("f.cpqr", s); cpqr_id_batched(s, cp, eps, dks.p, true); }
        std::vector<int> h = dks.to_host(cp.size());
        for (size_t q = 0; q < sm.size(); ++q) hk[sm[q] - b0] = h[q];
      }
      if (!big.empty()) {
        RSF_PHASE("f.rrqr", s);
        std::vector<RRQRProb> rp;
        for (int b : big) {
          const int m = (int)N[b].size() + N_RINGS * N_ANGLES, c = cvec[b];
          rp.push_back(RRQRProb{A.p + aoff[b - b0], m, m, c, dpiv.p + ioff[b - b0], nullptr, Tfull.p + tfoff[b], c});
        }
        RRQRResult rr = rrqr_batched(s, rp, eps, opts.seed ^ (0x9E3779B97F4A7C15ull * (unsigned long long)(lev + 17 * (which + 2))));
        for (size_t q = 0; q < big.size(); ++q) {
          const int b = big[q];
          const int m = (int)N[b].size() + N_RINGS * N_ANGLES, c = cvec[b];
          hk[b - b0] = rr.k[q];
          F->diag.flops_id += 2.0 * m * (double)c * rr.done[q] + (double)rr.k[q] * rr.k[q] * (c - rr.k[q]);
        }
      }
      std::vector<int> hp = dpiv.to_host(hI.size());
      for (int b = b0; b < b1; ++b) {
        kvec[b] = hk[b - b0];
        piv[b].assign(hp.begin() + ioff[b - b0], hp.begin() + ioff[b - b0] + cvec[b]);
        const double kk = kvec[b];
        if (cvec[b] <= SMALL_C) F->diag.flops_id += kk * kk * (cvec[b] - kk);
      }
      b0 = b1;
    }

    // ---- skeleton / redundant sets
    LV.c = cvec;
    LV.k = kvec;
    LV.r.resize(nb);
    LV.soff.resize(nb);
    LV.roff.resize(nb);
    std::vector<int> hS, hR, hpiv;
    std::vector<long long> poff(nb), bsz(nb);
    long long btot = 0;
    for (int b = 0; b < nb; ++b) {
      const int c = cvec[b], k = kvec[b];
      LV.r[b] = c - k;
      LV.soff[b] = hS.size();
      LV.roff[b] = hR.size();
      Snode[nodes[b]].clear();
      for (int j = 0; j < k; ++j) { hS.push_back(I[b][piv[b][j]]); Snode[nodes[b]].push_back(I[b][piv[b][j]]); }
      for (int j = k; j < c; ++j) hR.push_back(I[b][piv[b][j]]);
      poff[b] = hpiv.size();
      hpiv.insert(hpiv.end(), piv[b].begin(), piv[b].end());
      bsz[b] = btot;
      btot += (long long)c * c;
    }
    LV.rtot = hR.size();
    LV.S.alloc(std::max<size_t>(hS.size(), 1), s);
    LV.S.upload(hS);
    LV.R.alloc(std::max<size_t>(hR.size(), 1), s);
    LV.R.upload(hR);
    {
      static const bool fused_on0 = !(getenv("RSF_FUSED") && std::string(getenv("RSF_FUSED")) == "0");
      static const bool stack_on = !(getenv("RSF_STACKED") && std::string(getenv("RSF_STACKED")) == "0");
      int mi = 0;
      for (int b = 0; b < nb; ++b) mi = std::max(mi, cvec[b]);
      LV.stacked = !sig && stack_on && !(fused_on0 && mi <= sweep_max_i());
      if (LV.stacked) {
        std::vector<int> hSR;
        LV.sroff.resize(nb);
        for (int b = 0; b < nb; ++b) {
          LV.sroff[b] = hSR.size();
          hSR.insert(hSR.end(), hS.begin() + LV.soff[b], hS.begin() + LV.soff[b] + kvec[b]);
          hSR.insert(hSR.end(), hR.begin() + LV.roff[b], hR.begin() + LV.roff[b] + (cvec[b] - kvec[b]));
        }
        LV.SR.alloc(std::max<size_t>(hSR.size(), 1), s);
        LV.SR.upload(hSR);
      }
    }

    // ---- self blocks and permutation
    std::vector<int> hIall;
    std::vector<long long> iall(nb);
    for (int b = 0; b < nb; ++b) { iall[b] = hIall.size(); hIall.insert(hIall.end(), I[b].begin(), I[b].end()); }
    DBuf<int> dIall(std::max<size_t>(hIall.size(), 1), s), dpv(std::max<size_t>(hpiv.size(), 1), s);
    dIall.upload(hIall);
    dpv.upload(hpiv);
    DBuf<double> Bcur(std::max<long long>(btot, 1), s), Bp(std::max<long long>(btot, 1), s);
    {
      std::vector<SelfAsmDesc> sd;
      for (int b = 0; b < nb; ++b) {
        SelfAsmDesc d{};
        d.B = Bcur.p + bsz[b];
        d.c = cvec[b];
        d.I = dIall.p + iall[b];
        d.nch = 0;
        const int nd = nodes[b];
        if (sig && !t.is_leaf(nd)) {
          d.nch = nch[b];
          int qi = 0;
          for (int q = 0; q < 4; ++q) {
            const int ch = t.child[nd][q];
            if (ch < 0) continue;
            d.chB[qi] = bref[ch].Bp;
            d.chld[qi] = bref[ch].ld;
            ++qi;
          }
          for (int q = 0; q <= d.nch; ++q) d.choff[q] = choff[b][q];
        }
        sd.push_back(d);
      }
      RSF_PHASE("f.self_perm", s);
      assemble_self(s, sd, kp, which, t.xs.p, t.ys.p);
      std::vector<PermDesc> pd;
      for (int b = 0; b < nb; ++b) pd.push_back(PermDesc{Bcur.p + bsz[b], Bp.p + bsz[b], cvec[b], dpv.p + poff[b]});
      permute_sym(s, pd);
    }
    Bcur.release();
    Bp_prev.release();   // children's blocks consumed

    // ---- sparsify + eliminate
    long long ttot = 0, ltot = 0;
    LV.toff.resize(nb);
    LV.loff.resize(nb);
    LV.eoff.resize(nb);
    for (int b = 0; b < nb; ++b) {
      const long long k = kvec[b], r = LV.r[b];
      LV.toff[b] = ttot; LV.eoff[b] = ttot; ttot += k * r;
      LV.loff[b] = ltot; ltot += r * r;
    }
    LV.T.alloc(std::max<long long>(ttot, 1), s);
    if (LV.stacked) {
      long long et = 0;
      LV.eloff.resize(nb);
      for (int b = 0; b < nb; ++b) { LV.eloff[b] = et; et += (long long)cvec[b] * LV.r[b]; }
      LV.EL.alloc(std::max<long long>(et, 1), s);
    } else {
      LV.E.alloc(std::max<long long>(ttot, 1), s);
    }
    // L is needed by apply / sample only; a solve-only factor (Alg. 1) keeps L^-1
    if (!(sig && solve_only) && !LV.stacked) LV.L.alloc(std::max<long long>(ltot, 1), s);
    if (sig) LV.Linv.alloc(std::max<long long>(ltot, 1), s);
    {
      GemmBatch e1(false, false), e2(false, false), e3(true, false);
      std::vector<CopyProb> tcopy;
      for (int b = 0; b < nb; ++b) {
        const int c = cvec[b], k = kvec[b], r = LV.r[b];
        double* B = Bp.p + bsz[b];
        const double* Tf = Tfull.p + tfoff[b];
        if (k > 0 && r > 0) {
          GemmDesc d1 = gdesc(k, r, k);      // X_SR = B_SR - B_SS T
          d1.A = B; d1.lda = c; d1.B = Tf; d1.ldb = c; d1.C = B + (long long)k * c; d1.ldc = c;
          d1.alpha = -1.0; d1.beta = 1.0;
          e1.add(d1);
          GemmDesc d2 = gdesc(r, r, k);      // X_RR -= B_RS T
          d2.A = B + k; d2.lda = c; d2.B = Tf; d2.ldb = c; d2.C = B + (long long)k * c + k; d2.ldc = c;
          d2.alpha = -1.0; d2.beta = 1.0;
          e2.add(d2);
          GemmDesc d3 = gdesc(r, r, k);      // X_RR -= T^T X_SR
          d3.A = Tf; d3.lda = c; d3.B = B + (long long)k * c; d3.ldb = c; d3.C = B + (long long)k * c + k; d3.ldc = c;
          d3.alpha = -1.0; d3.beta = 1.0;
          e3.add(d3);
          tcopy.push_back(CopyProb{Tf, c, LV.T.p + LV.toff[b], k, k, r, 1.0});
        }
        F->diag.flops_elim += sig ? (3.0 * k * k * r + 5.0 * k * (double)r * r + (double)r * r * r / 3.0)
                                  : (2.0 * k * k * r + 4.0 * k * (double)r * r);
      }
      { RSF_PHASE("f.elim_gemm", s); e1.run(s); e2.run(s); e3.run(s); }
      copy_batched(s, tcopy);
      if (sig) {
        std::vector<PotrfProb> pp;
        std::vector<int> pbox;
        for (int b = 0; b < nb; ++b) {
          const int c = cvec[b], k = kvec[b], r = LV.r[b];
          if (r == 0) continue;
          pp.push_back(PotrfProb{Bp.p + bsz[b] + (long long)k * c + k, c, r, LV.Linv.p + LV.loff[b], r});
          pbox.push_back(b);
        }
        DBuf<double> lsum(std::max<size_t>(pp.size(), 1), s);
        DBuf<int> info(std::max<size_t>(pp.size(), 1), s);
        { RSF_PHASE("f.potrf", s); potrf_batched(s, pp, lsum.p, info.p); }
        std::vector<double> hl = lsum.to_host(pp.size());
        std::vector<int> hi = info.to_host(pp.size());
        for (size_t i = 0; i < pp.size(); ++i) {
          if (hi[i] != 0)
            throw Error(ST_ENUMERIC, "Cholesky of X_RR failed at level " + std::to_string(lev) + ", box " +
                                         std::to_string(pbox[i]) + " (node " + std::to_string(nodes[pbox[i]]) +
                                         "), column " + std::to_string(hi[i] - 1));
          logdet += 2.0 * hl[i];
        }
        std::vector<CopyProb> lc;
        GemmBatch e4(false, true), e5(false, true);
        for (int b = 0; b < nb; ++b) {
          const int c = cvec[b], k = kvec[b], r = LV.r[b];
          if (r == 0) continue;
          double* B = Bp.p + bsz[b];
          if (!solve_only) lc.push_back(CopyProb{B + (long long)k * c + k, c, LV.L.p + LV.loff[b], r, r, r, 1.0});
          if (k == 0) continue;
          GemmDesc d4 = gdesc(k, r, r);      // E = X_SR L^-T
          d4.btri = 2;
          d4.A = B + (long long)k * c; d4.lda = c; d4.B = LV.Linv.p + LV.loff[b]; d4.ldb = r;
          d4.C = LV.E.p + LV.eoff[b]; d4.ldc = k;
          e4.add(d4);
          GemmDesc d5 = gdesc(k, k, r);      // B_SS -= E E^T
          d5.A = LV.E.p + LV.eoff[b]; d5.lda = k; d5.B = LV.E.p + LV.eoff[b]; d5.ldb = k;
          d5.C = B; d5.ldc = c; d5.alpha = -1.0; d5.beta = 1.0;
          e5.add(d5);
        }
        RSF_PHASE("f.elim_gemm", s);
        copy_batched(s, lc);
        e4.run(s);
        e5.run(s);
      } else {
        std::vector<SymDesc> sy;
        std::vector<CopyProb> lc;
        for (int b = 0; b < nb; ++b) {
          const int c = cvec[b], k = kvec[b], r = LV.r[b];
          if (r == 0) continue;
          double* B = Bp.p + bsz[b];
          sy.push_back(SymDesc{B + (long long)k * c + k, c, r});
          if (LV.stacked) {   // [X_SR; X_RR] = the columns R of the pivoted block, as they are
            lc.push_back(CopyProb{B + (long long)k * c, c, LV.EL.p + LV.eloff[b], c, c, r, 1.0});
            continue;
          }
          lc.push_back(CopyProb{B + (long long)k * c + k, c, LV.L.p + LV.loff[b], r, r, r, 1.0});
          if (k > 0) lc.push_back(CopyProb{B + (long long)k * c, c, LV.E.p + LV.eoff[b], k, k, r, 1.0});
        }
        symmetrize(s, sy);
        copy_batched(s, lc);
      }
    }
    F->diag.bytes_factor += 8.0 * (sig ? (2.0 * ttot + (solve_only ? 1.0 : 2.0) * ltot) : (2.0 * ttot + ltot));
    F->diag.level_boxes.push_back(nb);
    long long Isum = 0, Ssum = 0;
    int Imax = 0;
    for (int b = 0; b < nb; ++b) { Isum += cvec[b]; Ssum += kvec[b]; Imax = std::max(Imax, cvec[b]); }
    if (sig) F->diag.bytes_solve += 2.0 * 8.0 * (2.0 * ttot + ltot) + 2.0 * 16.0 * (double)Isum;
    F->diag.level_I.push_back((int)Isum);
    F->diag.level_S.push_back((int)Ssum);
    F->diag.level_maxI.push_back(Imax);

    for (int b = 0; b < nb; ++b) bref[nodes[b]] = BRef{Bp.p + bsz[b], cvec[b], kvec[b]};
    Bp_prev = std::move(Bp);

    // ---- sweep descriptors for this level
    long long tcol = 0;
    std::vector<long long> tc(nb);
    for (int b = 0; b < nb; ++b) { tc[b] = tcol; tcol += LV.r[b]; }
    F->tmp_cols = std::max(F->tmp_cols, tcol);
    LV.fs1.reset(false, false); LV.fs2.reset(false, true); LV.fs3.reset(false, true);
    LV.bs2.reset(false, false); LV.bs3.reset(false, false); LV.bs4.reset(false, true);
    LV.up1.reset(false, true); LV.up2.reset(false, false); LV.up3.reset(false, false);
    LV.dn1.reset(false, true); LV.dn2.reset(false, true); LV.dn4.reset(false, false);
    LV.ao1.reset(false, true); LV.ao2a.reset(false, false); LV.ao2b.reset(false, false);
    LV.ao3.reset(false, true); LV.ao4.reset(false, false);
    for (int b = 0; b < nb; ++b) {
      const int k = kvec[b], r = LV.r[b];
      if (r == 0) continue;
      const int* Sb = LV.S.p + LV.soff[b];
      const int* Rb = LV.R.p + LV.roff[b];
      const double* Tb = LV.T.p + LV.toff[b];
      const double* Lb = LV.L.p ? LV.L.p + LV.loff[b] : nullptr;
      const double* Eb = LV.E.p ? LV.E.p + LV.eoff[b] : nullptr;
      auto mk = [&](int N, int K, int selA, const int* mapA, long long offA, const double* Bm, int ldb,
                    int selC, const int* mapC, long long offC, double alpha, double beta) {
        GemmDesc d = gdesc(-1, N, K);
        d.selA = selA; d.mapA = mapA; d.offA = offA;
        d.B = Bm; d.ldb = ldb;
        d.selC = selC; d.mapC = mapC; d.offC = offC;
        d.alpha = alpha; d.beta = beta;
        return d;
      };
      if (sig) {
        const double* Lib = LV.Linv.p + LV.loff[b];
        if (k > 0) LV.fs1.add(mk(r, k, 1, Sb, 0, Tb, k, 1, Rb, 0, -1.0, 1.0));
        LV.fs2.add(tri(mk(r, r, 1, Rb, 0, Lib, r, 2, nullptr, tc[b], 1.0, 0.0), 2));
        if (k > 0) LV.fs3.add(mk(k, r, 2, nullptr, tc[b], Eb, k, 1, Sb, 0, -1.0, 1.0));
        if (k > 0) LV.bs2.add(mk(r, k, 1, Sb, 0, Eb, k, 2, nullptr, tc[b], -1.0, 1.0));
        LV.bs3.add(tri(mk(r, r, 2, nullptr, tc[b], Lib, r, 1, Rb, 0, 1.0, 0.0), 1));
        if (k > 0) LV.bs4.add(mk(k, r, 1, Rb, 0, Tb, k, 1, Sb, 0, -1.0, 1.0));
        if (solve_only) continue;
        if (k > 0) LV.up1.add(mk(k, r, 1, Rb, 0, Tb, k, 1, Sb, 0, 1.0, 1.0));
        LV.up2.add(tri(mk(r, r, 1, Rb, 0, Lb, r, 2, nullptr, tc[b], 1.0, 0.0), 1));
        if (k > 0) LV.up3.add(mk(r, k, 1, Sb, 0, Eb, k, 2, nullptr, tc[b], 1.0, 1.0));
        if (k > 0) LV.dn1.add(mk(k, r, 1, Rb, 0, Eb, k, 1, Sb, 0, 1.0, 1.0));
        LV.dn2.add(tri(mk(r, r, 1, Rb, 0, Lb, r, 2, nullptr, tc[b], 1.0, 0.0), 2));
        if (k > 0) LV.dn4.add(mk(r, k, 1, Sb, 0, Tb, k, 1, Rb, 0, 1.0, 1.0));
      } else if (LV.stacked) {
        // X0 = x (modified), X1 = y;  y_R = [X_SR; X_RR]^T [x_S; x_R] in one GEMM (K = |I_b|)
        const int* SRb = LV.SR.p + LV.sroff[b];
        const double* ELb = LV.EL.p + LV.eloff[b];
        const int c = k + r;
        if (k > 0) LV.ao1.add(mk(k, r, 1, Rb, 0, Tb, k, 1, Sb, 0, 1.0, 1.0));
        LV.ao2a.add(mk(r, c, 1, SRb, 0, ELb, c, 2, Rb, 0, 1.0, 0.0));
        if (k > 0) LV.ao3.add(mk(k, r, 1, Rb, 0, ELb, c, 2, Sb, 0, 1.0, 1.0));
        if (k > 0) LV.ao4.add(mk(r, k, 2, Sb, 0, Tb, k, 2, Rb, 0, 1.0, 1.0));
      } else {
        // X0 = x (modified), X1 = y
        if (k > 0) LV.ao1.add(mk(k, r, 1, Rb, 0, Tb, k, 1, Sb, 0, 1.0, 1.0));
        if (k > 0) LV.ao2a.add(mk(r, k, 1, Sb, 0, Eb, k, 2, Rb, 0, 1.0, 0.0));
        LV.ao2b.add(mk(r, r, 1, Rb, 0, Lb, r, 2, Rb, 0, 1.0, k > 0 ? 1.0 : 0.0));
        if (k > 0) LV.ao3.add(mk(k, r, 1, Rb, 0, Eb, k, 2, Sb, 0, 1.0, 1.0));
        if (k > 0) LV.ao4.add(mk(r, k, 2, Sb, 0, Tb, k, 2, Rb, 0, 1.0, 1.0));
      }
    }
    for (GemmBatch* g : {&LV.fs1, &LV.fs2, &LV.fs3, &LV.bs2, &LV.bs3, &LV.bs4, &LV.up1, &LV.up2, &LV.up3,
                         &LV.dn1, &LV.dn2, &LV.dn4, &LV.ao1, &LV.ao2a, &LV.ao2b, &LV.ao3, &LV.ao4})
      if (!g->empty()) g->finalize(s);
    // fused small-box sweeps for the solve (Sigma) and the apply-only operator (Sigma_i)
    {
      static const bool fused_on = !(getenv("RSF_FUSED") && std::string(getenv("RSF_FUSED")) == "0");
      LV.max_i = 0;
      for (int b = 0; b < nb; ++b) LV.max_i = std::max(LV.max_i, cvec[b]);
      LV.fused = fused_on && LV.max_i <= sweep_max_i();
      LV.fused1 = fused_on && LV.max_i <= SWEEP1_MAX_I && (sig || !LV.stacked);
      if (LV.fused || LV.fused1) {
        std::vector<BoxOp> ops;
        for (int b = 0; b < nb; ++b) {
          if (LV.r[b] == 0) continue;
          BoxOp op;
          op.S = LV.S.p + LV.soff[b]; op.R = LV.R.p + LV.roff[b];
          op.kb = kvec[b]; op.r = LV.r[b];
          op.T = LV.T.p + LV.toff[b];
          op.L = sig ? LV.Linv.p + LV.loff[b] : LV.L.p + LV.loff[b];
          op.E = LV.E.p + LV.eoff[b];
          ops.push_back(op);
        }
        LV.nops = (int)ops.size();
        LV.ops.alloc(std::max<size_t>(ops.size(), 1), s);
        LV.ops.upload(ops);
      }
    }
  }

  // ---- top (level 0, R-Y): B_0 and its dense Cholesky
  {
    RSF_PHASE("f.top", s);
    const int root = t.levels[0][0];
    std::vector<int> I0;
    std::array<int, 5> co{};
    int nc = 0;
    SelfAsmDesc d{};
    if (t.is_leaf(root)) {
      I0.resize(t.n);
      std::iota(I0.begin(), I0.end(), 0);
    } else {
      co[0] = 0;
      for (int q = 0; q < 4; ++q) {
        const int ch = t.child[root][q];
        if (ch < 0) continue;
        I0.insert(I0.end(), Snode[ch].begin(), Snode[ch].end());
        if (sig) { d.chB[nc] = bref[ch].Bp; d.chld[nc] = bref[ch].ld; }
        co[++nc] = (int)I0.size();
      }
    }
    const int n0 = (int)I0.size();
    F->n0 = n0;
    F->I0.alloc(std::max(n0, 1), s);
    F->I0.upload(I0);
    F->tmp_cols = std::max<long long>(F->tmp_cols, n0);
    if (n0 > 0) {
      F->C.alloc((size_t)n0 * n0, s);
      d.B = F->C.p;
      d.c = n0;
      d.I = F->I0.p;
      d.nch = sig ? nc : 0;
      for (int q = 0; q <= nc; ++q) d.choff[q] = co[q];
      assemble_self(s, {d}, kp, which, t.xs.p, t.ys.p);
      if (sig) {
        F->Cinv.alloc((size_t)n0 * n0, s);
        DBuf<double> lsum(1, s);
        DBuf<int> info(1, s);
        potrf_batched(s, {PotrfProb{F->C.p, n0, n0, F->Cinv.p, n0}}, lsum.p, info.p);
        double hl = lsum.to_host(1)[0];
        int hi = info.to_host(1)[0];
        if (hi != 0)
          throw Error(ST_ENUMERIC, "Cholesky of the top block failed (level 0, size " + std::to_string(n0) +
                                       ", column " + std::to_string(hi - 1) + ")");
        logdet += 2.0 * hl;
        F->diag.flops_top = (double)n0 * n0 * n0 / 3.0;
      }
      F->diag.bytes_factor += 8.0 * (double)n0 * n0 * (sig && !solve_only ? 2 : 1);
      if (sig) F->diag.bytes_solve += 2.0 * 8.0 * (double)n0 * n0;
    }
    Bp_prev.release();
    auto mk = [&](int N, int K, int selA, const int* mapA, const double* Bm, int ldb, int selC,
                  const int* mapC, double beta) {
      GemmDesc g = gdesc(-1, N, K);
      g.selA = selA; g.mapA = mapA; g.B = Bm; g.ldb = ldb; g.selC = selC; g.mapC = mapC; g.beta = beta;
      return g;
    };
    F->top_s1.reset(false, true); F->top_s2.reset(false, false);
    F->top_a1.reset(false, false); F->top_a2.reset(false, true);
    F->top_q1.reset(false, true); F->top_ao.reset(false, false);
    if (n0 > 0) {
      const int* m0 = F->I0.p;
      if (sig) {
        F->top_s1.add(tri(mk(n0, n0, 1, m0, F->Cinv.p, n0, 2, nullptr, 0.0), 2));   // tmp = X(I0) Cinv^T
        F->top_s2.add(tri(mk(n0, n0, 2, nullptr, F->Cinv.p, n0, 1, m0, 0.0), 1));   // X(I0) = tmp Cinv
        if (!solve_only) {
          F->top_a1.add(tri(mk(n0, n0, 1, m0, F->C.p, n0, 2, nullptr, 0.0), 1));      // tmp = X(I0) C
          F->top_a2.add(tri(mk(n0, n0, 2, nullptr, F->C.p, n0, 1, m0, 0.0), 2));      // X(I0) = tmp C^T
          F->top_q1.add(tri(mk(n0, n0, 1, m0, F->C.p, n0, 2, nullptr, 0.0), 2));      // tmp = X(I0) C^T
        } else {
          F->C.release();
        }
      } else {
        F->top_ao.add(mk(n0, n0, 1, m0, F->C.p, n0, 2, m0, 0.0));           // Y(I0) = X(I0) B0
      }
      for (GemmBatch* g : {&F->top_s1, &F->top_s2, &F->top_a1, &F->top_a2, &F->top_q1, &F->top_ao})
        if (!g->empty()) g->finalize(s);
    }
  }
  F->logdet = logdet;
  RSF_CUDA(cudaStreamSynchronize(s));
  F->diag.t_factor = now_s() - t0;
  return F;
}

// ------------------------------------------------------------------ operators
void solve_internal(const Fact& F, double* X, int k, double* tmp) {
  RSF_REQUIRE(F.which == W_SIGMA, ST_EINVAL, "solve needs a Sigma factor");
  cudaStream_t s = op_stream(F);
  const int L = F.tree->L;
  for (int lev = L; lev >= 1; --lev) {
    const Level& LV = F.levels[lev];
    RSF_PHASE(lvname("sv", lev), s);
    if (LV.sweep1(k)) { sweep_level(s, LV.ops.p, LV.nops, LV.max_i, SW_SOLVE_FWD, X, nullptr, k); continue; }
    LV.fs1.run(s, X, tmp, k, k);
    LV.fs2.run(s, X, tmp, k, k);
    LV.fs3.run(s, X, tmp, k, k);
    colcopy(s, X, tmp, k, k, LV.R.p, nullptr, LV.rtot);
  }
  {
    RSF_PHASE("sv.top", s);
    F.top_s1.run(s, X, tmp, k, k);
    F.top_s2.run(s, X, tmp, k, k);
  }
  for (int lev = 1; lev <= L; ++lev) {
    const Level& LV = F.levels[lev];
    RSF_PHASE(lvname("sv", lev), s);
    if (LV.sweep1(k)) { sweep_level(s, LV.ops.p, LV.nops, LV.max_i, SW_SOLVE_BWD, X, nullptr, k); continue; }
    colcopy(s, tmp, X, k, k, nullptr, LV.R.p, LV.rtot);
    LV.bs2.run(s, X, tmp, k, k);
    LV.bs3.run(s, X, tmp, k, k);
    LV.bs4.run(s, X, tmp, k, k);
  }
}

// F = L L^T with L = M_L ... M_1 C: the two halves of the solve
// x <- L^-1 x (forward sweeps, then C^-1) and x <- L^-T x (C^-T, then backward sweeps)
void solve_half_fwd(const Fact& F, double* X, int k, double* tmp) {
  RSF_REQUIRE(F.which == W_SIGMA, ST_EINVAL, "solve needs a Sigma factor");
  cudaStream_t s = op_stream(F);
  for (int lev = F.tree->L; lev >= 1; --lev) {
    const Level& LV = F.levels[lev];
    RSF_PHASE(lvname("sv", lev), s);
    if (LV.sweep1(k)) { sweep_level(s, LV.ops.p, LV.nops, LV.max_i, SW_SOLVE_FWD, X, nullptr, k); continue; }
    LV.fs1.run(s, X, tmp, k, k);
    LV.fs2.run(s, X, tmp, k, k);
    LV.fs3.run(s, X, tmp, k, k);
    colcopy(s, X, tmp, k, k, LV.R.p, nullptr, LV.rtot);
  }
  if (F.n0 > 0) {
    RSF_PHASE("sv.top", s);
    F.top_s1.run(s, X, tmp, k, k);                        // tmp = X(I0) C^-T
    colcopy(s, X, tmp, k, k, F.I0.p, nullptr, F.n0);      // X(I0) = tmp
  }
}

void solve_half_bwd(const Fact& F, double* X, int k, double* tmp) {
  RSF_REQUIRE(F.which == W_SIGMA, ST_EINVAL, "solve needs a Sigma factor");
  cudaStream_t s = op_stream(F);
  if (F.n0 > 0) {
    RSF_PHASE("sv.top", s);
    colcopy(s, tmp, X, k, k, nullptr, F.I0.p, F.n0);      // tmp = X(I0)
    F.top_s2.run(s, X, tmp, k, k);                        // X(I0) = tmp C^-1
  }
  for (int lev = 1; lev <= F.tree->L; ++lev) {
    const Level& LV = F.levels[lev];
    RSF_PHASE(lvname("sv", lev), s);
    if (LV.sweep1(k)) { sweep_level(s, LV.ops.p, LV.nops, LV.max_i, SW_SOLVE_BWD, X, nullptr, k); continue; }
    colcopy(s, tmp, X, k, k, nullptr, LV.R.p, LV.rtot);
    LV.bs2.run(s, X, tmp, k, k);
    LV.bs3.run(s, X, tmp, k, k);
    LV.bs4.run(s, X, tmp, k, k);
  }
}

static void down_sweep(const Fact& F, double* X, int k, double* tmp) {
  cudaStream_t s = op_stream(F);
  for (int lev = 1; lev <= F.tree->L; ++lev) {
    const Level& LV = F.levels[lev];
    LV.dn1.run(s, X, tmp, k, k);
    LV.dn2.run(s, X, tmp, k, k);
    colcopy(s, X, tmp, k, k, LV.R.p, nullptr, LV.rtot);
    LV.dn4.run(s, X, tmp, k, k);
  }
}

void apply_internal(const Fact& F, double* X, int k, double* tmp) {
  RSF_REQUIRE(F.which == W_SIGMA && !F.solve_only, ST_EINVAL, "apply_internal needs a full Sigma factor");
  cudaStream_t s = op_stream(F);
  for (int lev = F.tree->L; lev >= 1; --lev) {
    const Level& LV = F.levels[lev];
    LV.up1.run(s, X, tmp, k, k);
    LV.up2.run(s, X, tmp, k, k);
    LV.up3.run(s, X, tmp, k, k);
    colcopy(s, X, tmp, k, k, LV.R.p, nullptr, LV.rtot);
  }
  F.top_a1.run(s, X, tmp, k, k);
  F.top_a2.run(s, X, tmp, k, k);
  down_sweep(F, X, k, tmp);
}

void sqrt_internal(const Fact& F, double* X, int k, double* tmp) {
  RSF_REQUIRE(F.which == W_SIGMA && !F.solve_only, ST_EINVAL, "sample needs a full Sigma factor");
  cudaStream_t s = op_stream(F);
  if (F.n0 > 0) {
    F.top_q1.run(s, X, tmp, k, k);
    colcopy(s, X, tmp, k, k, F.I0.p, nullptr, F.n0);
  }
  down_sweep(F, X, k, tmp);
}

void apply_only_internal(const Fact& F, double* X, double* Y, int k) {
  RSF_REQUIRE(F.which != W_SIGMA, ST_EINVAL, "apply_only needs a Sigma_i compression");
  cudaStream_t s = op_stream(F);
  const int L = F.tree->L;
  for (int lev = L; lev >= 1; --lev) {
    const Level& LV = F.levels[lev];
    RSF_PHASE(lvname("ao", lev), s);
    if (LV.sweep1(k)) { sweep_level(s, LV.ops.p, LV.nops, LV.max_i, SW_AO_UP, X, Y, k); continue; }
    LV.ao1.run(s, X, Y, k, k);
    LV.ao2a.run(s, X, Y, k, k);
    LV.ao2b.run(s, X, Y, k, k);
  }
  {
    RSF_PHASE("ao.top", s);
    F.top_ao.run(s, X, Y, k, k);
  }
  for (int lev = 1; lev <= L; ++lev) {
    const Level& LV = F.levels[lev];
    RSF_PHASE(lvname("ao", lev), s);
    if (LV.sweep1(k)) { sweep_level(s, LV.ops.p, LV.nops, LV.max_i, SW_AO_DN, X, Y, k); continue; }
    LV.ao3.run(s, X, Y, k, k);
    LV.ao4.run(s, X, Y, k, k);
  }
}

}  // namespace rsf

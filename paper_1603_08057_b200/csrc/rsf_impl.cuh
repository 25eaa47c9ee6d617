// Internal data structures of librsf: context, quadtree, factor handle.
#pragma once
#include <array>
#include <memory>
#include <unordered_map>

#include "comm.cuh"
#include "common.cuh"
#include "covariance.cuh"
#include "gemm.cuh"
#include "sweep.cuh"

namespace rsf {

struct Opts {
  double eps_peel = 1e-6;
  int oversample = 8;        // c in (r + c) (R-K)
  int probe_block = 512;     // max probe columns per G-apply chunk
  int peel_start = 64;       // initial probe columns per group at level 1 (R-M adaptivity)
  int max_depth = 30;
  double r_near = 1.8, r_in = 1.75, r_out = 2.45;   // R-C (in units of the box half-width)
  unsigned long long seed = 1603080570ull;
  int strong = 0;            // peeling admissibility: 0 weak, 1 strong (next row f4)
  int peel_f32 = 0;          // peeled levels stored in FP32 (FP64 arithmetic), DESIGN.md §7g
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = 0;
  std::vector<cudaStream_t> aux;   // streams of the concurrent trace jobs of gp_mle_eval (created lazily)
  bool own_stream = false;
  Comm comm;                        // rank group of a sharded evaluation (world 1: none)
  std::vector<Comm> job_comms;      // one split communicator per trace job (its group's ranks)
  int job_comms_njobs = -1;         // number of jobs job_comms was built for
  // memory plan of gp_mle_eval: (n, jobs) shapes whose trace jobs did not fit side by side; later
  // evaluations of such a shape run them in the serial order directly (no OOM-and-redo)
  std::vector<std::pair<long long, int>> serial_shapes;
  std::string last_error;
};

// ------------------------------------------------------------------ quadtree
// Points are sorted by 60-bit Morton key (30 bits per axis on the root [0,1]^2);
// every node owns a contiguous range [begin, end) of the sorted order ("tree
// index").  Children are in quadrant order SW, SE, NW, NE (q = bx + 2 by).
struct Tree {
  int n = 0, leaf = 0, L = 0;
  std::vector<int> perm;        // tree index -> original index
  std::vector<int> lev, parent, quad, begin, end;
  std::vector<std::array<int, 4>> child;    // by quadrant, -1 if absent
  std::vector<int> ix, iy;      // cell coordinates at the node's level
  std::vector<std::vector<int>> levels;     // node ids per level (Morton order)
  std::unordered_map<unsigned long long, int> cell;   // (level, ix, iy) -> node
  DBuf<double> xs, ys;          // coordinates in tree order (device)
  std::vector<double> hx, hy;   // same, host copy (near-list scheduling)
  DBuf<int> d_perm;             // tree index -> original index (device)
  bool is_leaf(int b) const { return child[b][0] < 0 && child[b][1] < 0 && child[b][2] < 0 && child[b][3] < 0; }
  double cx(int b) const { return (ix[b] + 0.5) / double(1u << lev[b]); }
  double cy(int b) const { return (iy[b] + 0.5) / double(1u << lev[b]); }
  double h(int b) const { return 0.5 / double(1u << lev[b]); }
  static unsigned long long cell_key(int l, int x, int y) {
    return ((unsigned long long)l << 58) | ((unsigned long long)x << 29) | (unsigned long long)y;
  }
  int find(int l, int x, int y) const {
    auto it = cell.find(cell_key(l, x, y));
    return it == cell.end() ? -1 : it->second;
  }
};

std::shared_ptr<Tree> build_tree(Ctx& ctx, const double* d_xy, int n, int leaf, int max_depth);

// ------------------------------------------------------------------ factor
struct Level {
  int lev = 0;
  int nbox = 0;
  std::vector<int> node;             // node ids
  std::vector<int> c, k, r;          // |I|, |S|, |R|
  std::vector<long long> soff, roff; // offsets into S/R index arrays
  DBuf<int> S, R;                    // tree indices
  // persistent blocks (offsets in doubles)
  std::vector<long long> toff, loff, eoff;
  DBuf<double> T;      // k x r (ld k)
  DBuf<double> L, Linv;  // r x r (Sigma) | XRR r x r (Sigma_i, in L)
  DBuf<double> E;      // k x r (Sigma: E; Sigma_i: X_SR)
  // Sigma_i levels swept by batched GEMMs: [X_SR; X_RR] stacked per box (c x r, ld c, the
  // columns R of the pivoted block), so that y_R = X_SR^T x_S + X_RR x_R is one GEMM over the
  // box's indices in [S; R] order (SR)
  bool stacked = false;
  DBuf<double> EL;
  std::vector<long long> eloff, sroff;
  DBuf<int> SR;
  long long rtot = 0;  // sum r (tmp columns)
  // sweep GEMM batches (M = number of RHS, per call)
  GemmBatch fs1, fs2, fs3;            // forward solve
  GemmBatch bs2, bs3, bs4;            // backward solve
  GemmBatch up1, up2, up3;            // apply, up
  GemmBatch dn1, dn2, dn4;            // apply, down
  GemmBatch ao1, ao2a, ao2b, ao3, ao4;  // apply-only (Sigma_i); ao2a alone when stacked
  // fused small-box sweeps (sweep.cuh): used when every box has |I_b| <= SWEEP_MAX_I
  bool fused = false;
  bool fused1 = false;                // ops built for the one-right-hand-side fused sweep (k = 1)
  int max_i = 0, nops = 0;
  bool sweep1(int k) const { return fused || (k == 1 && fused1); }
  DBuf<BoxOp> ops;
};

struct FactDiag {
  double flops_id = 0, flops_elim = 0, flops_top = 0;   // algorithmic (formulas of DESIGN.md)
  double bytes_factor = 0;                              // stored factor bytes
  // algorithmic bytes of one 1-RHS solve: the forward and the backward sweep
  // each read T, E and L^-1 of every box once and C^-1 once, and read + write every active
  // DOF of every level once: 2 (8 (2 sum k r + sum r^2) + 8 n0^2) + 2 * 16 sum |I|
  double bytes_solve = 0;
  double t_tree = 0, t_factor = 0;
  std::vector<int> level_boxes, level_I, level_S, level_maxI;
};

struct Fact {
  Ctx* ctx = nullptr;
  int which = W_SIGMA;
  bool solve_only = false;           // Sigma factor without L / C (Alg. 1: only solves are needed)
  KParams kp{};
  double eps = 0;
  Opts opts;
  std::shared_ptr<Tree> tree;
  std::vector<Level> levels;         // indexed by level number (0 unused)
  int n0 = 0;
  DBuf<int> I0;
  DBuf<double> C, Cinv;              // Sigma: top Cholesky and inverse; Sigma_i: C = B0
  double logdet = 0;
  long long tmp_cols = 0;            // max(sum r per level, n0)
  GemmBatch top_s1, top_s2, top_a1, top_a2, top_q1, top_ao;
  FactDiag diag;
  int n() const { return tree->n; }
};

std::unique_ptr<Fact> factor(Ctx& ctx, std::shared_ptr<Tree> tree, const KParams& kp, int which,
                             double eps, const Opts& opts, bool solve_only = false);

// Stream of the operators below: the factor's context stream unless a StreamScope on this
// thread redirects them (the peeling runs its G applies on a second stream).
cudaStream_t& stream_override();
inline cudaStream_t ctx_stream(const Ctx& c) { return stream_override() ? stream_override() : c.stream; }
inline cudaStream_t op_stream(const Fact& F) { return ctx_stream(*F.ctx); }
struct StreamScope {
  cudaStream_t prev;
  explicit StreamScope(cudaStream_t s) : prev(stream_override()) { stream_override() = s; }
  ~StreamScope() { stream_override() = prev; }
};

// operations on X' (k x n column-major, tree order, ld = k): in place
void solve_internal(const Fact& F, double* X, int k, double* tmp);
// halves of the solve for F = L L^T: X <- L^-1 X (fwd) and X <- L^-T X (bwd)
void solve_half_fwd(const Fact& F, double* X, int k, double* tmp);
void solve_half_bwd(const Fact& F, double* X, int k, double* tmp);
void apply_internal(const Fact& F, double* X, int k, double* tmp);
void sqrt_internal(const Fact& F, double* X, int k, double* tmp);
// apply-only Sigma_i: Y = F_i X (X is overwritten)
void apply_only_internal(const Fact& F, double* X, double* Y, int k);
// any operator: out = op(X) with X preserved? (helpers in rsf.cu)

// layout conversions between the caller's n x k (ld) original order and X'
void to_internal(cudaStream_t s, const Tree& t, const double* b, long long ld, int k, double* X);
void to_external(cudaStream_t s, const Tree& t, const double* X, int k, double* b, long long ld);

// kernel launch helpers (rsf_kernels.cu)
void colcopy(cudaStream_t s, double* dst, const double* src, int ldx, int M, const int* dmap,
             const int* smap, long long count, double alpha = 1.0, double beta = 0.0);

}  // namespace rsf

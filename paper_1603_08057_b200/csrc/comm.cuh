// Rank group of one sharded evaluation: the peeling probe
// columns of every probe block are split across the ranks (the independent peeling probe
// blocks of the north star; P:570-572 makes every column of Y = (G - sum G^(m)) W
// independent of the others), each rank applies G and the peeled levels to its own slice,
// and one all-gather per block gives every rank the whole sketch for the (replicated,
// deterministic) per-box basis work.  The extraction columns are split the same
// way and the leaf-trace partial sums are gathered and added in rank order.
//
// Transport: NCCL over NVLink / NVSwitch (loaded with dlopen at the first use, so librsf has
// no link-time dependency on it), one communicator per concurrent trace job (ncclCommSplit
// of the group's communicator: collectives of different host threads must not interleave on
// one communicator).  world == 1 issues no collective at all.  RSF_EMU_WORLD=P (P > 1) on a
// single-GPU context emulates P ranks in one process through the same slices and the same
// gather layout (each emulated rank's slice is computed in turn and copied into its slot of
// the gather buffer) -- the test of the partition and exchange layout on one GPU.
#pragma once
#include <algorithm>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace rsf {

struct Comm {
  int rank = 0, world = 1;
  void* nccl = nullptr;   // ncclComm_t
  int emu = 1;            // emulated ranks (world == 1 only)
  bool owned = false;     // nccl was created by the library (destroyed with the context)
  // a one-rank group that still issues its collectives through NCCL (RSF_NCCL_FORCE=1 at
  // rsf_ctx_create_group: the single-GPU test of the transport -- dlopen'd entry points,
  // communicator splits per trace job, in-place all-gathers, host staging)
  bool force = false;
  bool use_nccl() const { return world > 1 || (force && nccl != nullptr); }

  int parts() const { return world > 1 ? world : emu; }
  bool emulated() const { return world == 1 && emu > 1; }
  // this process computes parts [p0, p1) of every split block
  int p0() const { return world > 1 ? rank : 0; }
  int p1() const { return world > 1 ? rank + 1 : emu; }
  // column slice [lo, hi) of part r when k columns are split over P parts (contiguous,
  // sizes differ by at most one, larger slices first)
  static void slice(long long k, int P, int r, long long* lo, long long* hi) {
    const long long q = k / P, m = k % P;
    *lo = r * q + std::min<long long>(r, m);
    *hi = *lo + q + (r < m ? 1 : 0);
  }
  // every part's slice of k columns of an X' block (k_r x n, ld k_r) sits in slot r of the
  // gather buffer (slot size kmax * n doubles); after exchange() every slot holds its part
  long long kmax(long long k) const { return (k + parts() - 1) / parts(); }
  // NCCL all-gather of this rank's slot into every rank's gather buffer (no-op when emulated:
  // the emulated parts wrote their own slots)
  void exchange(cudaStream_t s, double* gath, long long slot) const;
  // merge the slots into the k x n X' block Y (ld k)
  void merge(cudaStream_t s, const double* gath, long long slot, long long k, int n, double* Y) const;
  // sum of cnt host doubles over the ranks, added in rank order (deterministic)
  void allsum(cudaStream_t s, double* v, int cnt) const;
  // every rank's cnt host doubles, rank-ordered into out (world * cnt)
  void allgather_host(cudaStream_t s, const double* in, int cnt, double* out) const;
  // trace jobs of one evaluation over the ranks: G = min(njobs, world) groups,
  // rank r in group r mod G, job j run by group j mod G (its ranks split the job's probe columns)
  static int job_groups(int njobs, int world) { return std::max(1, std::min(njobs, world)); }
  // group of `rank` when the G groups carry the estimated work gw[g] (the jobs dealt to them): ranks
  // 0..G-1 seed one group each, every further rank joins the group with the largest current work per
  // rank (ties: lowest group; this greedy minimises the largest work per rank) -- equal weights give
  // rank r -> group r mod G
  static int group_of_rank(const std::vector<double>& gw, int world, int rank) {
    const int G = (int)gw.size();
    if (G <= 1) return 0;
    if (rank < G) return rank;
    std::vector<int> cnt(G, 1);
    int g_of = 0;
    for (int r = G; r <= rank; ++r) {
      int best = 0;
      for (int g = 1; g < G; ++g)
        if (gw[g] / cnt[g] > gw[best] / cnt[best]) best = g;
      ++cnt[best];
      g_of = best;
    }
    return g_of;
  }
};

// NCCL entry points (dlopen'd): 128-byte unique id, communicator from (id, rank, world) or
// queried from an existing ncclComm_t, split for the trace jobs, destroy.
void nccl_unique_id(unsigned char out[128]);
void* nccl_init_rank(const unsigned char id[128], int rank, int world);
void nccl_query(void* comm, int* rank, int* world);
void* nccl_split(void* comm, int rank);
// split with a color (< 0: this rank joins no new communicator and gets nullptr)
void* nccl_split_color(void* comm, int color, int key);
void nccl_destroy(void* comm);
// NCCL collectives issued by this process so far (tests)
long long nccl_calls();

}  // namespace rsf

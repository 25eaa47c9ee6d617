// NCCL transport of the sharded evaluation (comm.cuh).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <string>

#include "comm.cuh"

namespace rsf {

namespace {

struct NcclApi {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclCommSplit) split = nullptr;
  decltype(&ncclCommCount) count = nullptr;
  decltype(&ncclCommUserRank) user_rank = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGetErrorString) err = nullptr;
};

const NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    // the copy torch already loaded (same soname) is reused by the dynamic loader
    for (const char* nm : {"libnccl.so.2", "libnccl.so"}) {
      a.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (!a.h) return;
    a.get_unique_id = (decltype(a.get_unique_id))dlsym(a.h, "ncclGetUniqueId");
    a.init_rank = (decltype(a.init_rank))dlsym(a.h, "ncclCommInitRank");
    a.destroy = (decltype(a.destroy))dlsym(a.h, "ncclCommDestroy");
    a.split = (decltype(a.split))dlsym(a.h, "ncclCommSplit");
    a.count = (decltype(a.count))dlsym(a.h, "ncclCommCount");
    a.user_rank = (decltype(a.user_rank))dlsym(a.h, "ncclCommUserRank");
    a.all_gather = (decltype(a.all_gather))dlsym(a.h, "ncclAllGather");
    a.err = (decltype(a.err))dlsym(a.h, "ncclGetErrorString");
  });
  RSF_REQUIRE(a.h && a.get_unique_id && a.init_rank && a.destroy && a.split && a.count && a.user_rank &&
                  a.all_gather && a.err,
              ST_ENCCL, "NCCL (libnccl.so.2) could not be loaded");
  return a;
}

std::atomic<long long> g_calls{0};

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(ST_ENCCL, std::string(what) + ": " + api().err(r));
}

constexpr int NT = 256;

// Y'(lo_r + j, t) = slot_r(j, t) for the k_r x n slice of part r (ld k_r)
__global__ void merge_kernel(const double* __restrict__ gath, long long slot, long long k, int P, int n,
                             double* __restrict__ Y) {
  const long long tot = (long long)n * k;
  const long long q = k / P, m = k % P;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < tot; e += (long long)gridDim.x * NT) {
    const long long t = e / k, j = e - t * k;
    // part of column j: the first m parts hold q + 1 columns
    const long long r = (j < m * (q + 1)) ? j / (q + 1) : m + (j - m * (q + 1)) / q;
    const long long lo = r * q + std::min<long long>(r, m);
    const long long kr = q + (r < m ? 1 : 0);
    Y[e] = gath[r * slot + t * kr + (j - lo)];
  }
}

}  // namespace

void Comm::exchange(cudaStream_t s, double* gath, long long slot) const {
  if (!use_nccl()) return;
  check(api().all_gather(gath + (long long)rank * slot, gath, (size_t)slot, ncclDouble, (ncclComm_t)nccl, s),
        "ncclAllGather");
  ++g_calls;
}

void Comm::merge(cudaStream_t s, const double* gath, long long slot, long long k, int n, double* Y) const {
  const long long tot = (long long)n * k;
  const int g = (int)std::max<long long>(1, std::min<long long>((tot + NT - 1) / NT, 4096));
  merge_kernel<<<g, NT, 0, s>>>(gath, slot, k, parts(), n, Y);
  count_launch();
  RSF_LAUNCH_CHECK();
}

void Comm::allsum(cudaStream_t s, double* v, int cnt) const {
  if (!use_nccl()) return;
  // gather every rank's values, then add them in rank order on the host (deterministic)
  DBuf<double> g((size_t)cnt * world, s);
  RSF_CUDA(cudaMemcpyAsync(g.p + (size_t)rank * cnt, v, cnt * sizeof(double), cudaMemcpyHostToDevice, s));
  check(api().all_gather(g.p + (size_t)rank * cnt, g.p, (size_t)cnt, ncclDouble, (ncclComm_t)nccl, s),
        "ncclAllGather");
  ++g_calls;
  const std::vector<double> h = g.to_host((size_t)cnt * world);
  for (int i = 0; i < cnt; ++i) {
    double a = 0.0;
    for (int r = 0; r < world; ++r) a += h[(size_t)r * cnt + i];
    v[i] = a;
  }
}

void Comm::allgather_host(cudaStream_t s, const double* in, int cnt, double* out) const {
  if (!use_nccl()) {
    std::copy(in, in + cnt, out);
    return;
  }
  DBuf<double> g((size_t)cnt * world, s);
  RSF_CUDA(cudaMemcpyAsync(g.p + (size_t)rank * cnt, in, cnt * sizeof(double), cudaMemcpyHostToDevice, s));
  check(api().all_gather(g.p + (size_t)rank * cnt, g.p, (size_t)cnt, ncclDouble, (ncclComm_t)nccl, s),
        "ncclAllGather");
  ++g_calls;
  const std::vector<double> h = g.to_host((size_t)cnt * world);
  std::copy(h.begin(), h.end(), out);
}

void nccl_unique_id(unsigned char out[128]) {
  ncclUniqueId id;
  check(api().get_unique_id(&id), "ncclGetUniqueId");
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out, &id, 128);
}

void* nccl_init_rank(const unsigned char idb[128], int rank, int world) {
  ncclUniqueId id;
  std::memcpy(&id, idb, 128);
  ncclComm_t c = nullptr;
  check(api().init_rank(&c, world, id, rank), "ncclCommInitRank");
  return c;
}

void nccl_query(void* comm, int* rank, int* world) {
  check(api().user_rank((ncclComm_t)comm, rank), "ncclCommUserRank");
  check(api().count((ncclComm_t)comm, world), "ncclCommCount");
}

void* nccl_split(void* comm, int rank) {
  ncclComm_t c = nullptr;
  check(api().split((ncclComm_t)comm, 0, rank, &c, nullptr), "ncclCommSplit");
  return c;
}

void* nccl_split_color(void* comm, int color, int key) {
  ncclComm_t c = nullptr;
  check(api().split((ncclComm_t)comm, color < 0 ? NCCL_SPLIT_NOCOLOR : color, key, &c, nullptr), "ncclCommSplit");
  return color < 0 ? nullptr : c;
}

long long nccl_calls() { return g_calls.load(); }

void nccl_destroy(void* comm) {
  if (comm) api().destroy((ncclComm_t)comm);
}

}  // namespace rsf

// Common runtime pieces of librsf: error type, stream-ordered device buffers,
// launch checks.  Internal header (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

namespace rsf {

// status codes mirror include/rsf.h
enum { ST_OK = 0, ST_EINVAL = 1, ST_ENUMERIC = 2, ST_ECUDA = 3, ST_ENOMEM = 4, ST_ENCCL = 5 };

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define RSF_CUDA(x)                                                                       \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess)                                                                \
      throw ::rsf::Error(e_ == cudaErrorMemoryAllocation ? ::rsf::ST_ENOMEM : ::rsf::ST_ECUDA, \
                         std::string(#x) + ": " + cudaGetErrorString(e_) + " (" __FILE__ ":" + \
                             std::to_string(__LINE__) + ")");                             \
  } while (0)

#define RSF_LAUNCH_CHECK() RSF_CUDA(cudaGetLastError())

#define RSF_REQUIRE(cond, code, msg) \
  do {                               \
    if (!(cond)) throw ::rsf::Error(code, msg); \
  } while (0)

// host seconds spent inside allocation / free / upload calls (diagnostics, RSF_KTRACE=1)
double host_clock();
extern double g_host_alloc, g_host_free, g_host_upload;
extern long long g_n_alloc;

// Size-class cache over cudaMallocAsync for buffers <= 64 MB (per stream: a block freed on a
// stream is reusable by later work on the same stream, exactly like the stream-ordered pool,
// without a driver call).  Larger buffers go to cudaMallocAsync directly.
void* dev_alloc(size_t bytes, cudaStream_t s);
void dev_free(void* p, size_t bytes, cudaStream_t s);
void dev_cache_trim(cudaStream_t s);   // release the cached blocks of a stream
void dev_cache_trim_bins(cudaStream_t s);   // release only the cached small (power-of-two bin) blocks
double dev_cache_bytes();
extern std::atomic<int> g_big_sync;          // > 0: large blocks via cudaMalloc/cudaFree (memory-saving mode)
void pool_trim();                            // return the stream-ordered pool's unused pages to the driver
struct BigSyncScope {                        // RAII: memory-saving mode for the scope when on
  bool on;
  explicit BigSyncScope(bool o) : on(o) { if (on && g_big_sync++ == 0) pool_trim(); }
  ~BigSyncScope() { if (on) --g_big_sync; }
};                    // bytes held in the bin caches of all streams (diagnostics)

// Stream-ordered device buffer (cudaMallocAsync on the context stream; the
// default memory pool keeps freed blocks cached for the next evaluation).
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = 0;
  DBuf() = default;
  DBuf(size_t count, cudaStream_t st) { alloc(count, st); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; s = o.s; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    if (count) {
      const double t0 = host_clock();
      p = static_cast<T*>(dev_alloc(count * sizeof(T), st));
      g_host_alloc += host_clock() - t0;
      ++g_n_alloc;
    }
  }
  void release() {
    if (p) {
      const double t0 = host_clock();
      dev_free(p, n * sizeof(T), s);
      g_host_free += host_clock() - t0;
    }
    p = nullptr;
    n = 0;
  }
  void zero() { if (n) RSF_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s)); }
  void upload(const T* h, size_t count) {
    if (count > n) alloc(count, s);
    const double t0 = host_clock();
    if (count) RSF_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
    g_host_upload += host_clock() - t0;
  }
  void upload(const std::vector<T>& v) { upload(v.data(), v.size()); }
  void download(T* h, size_t count) const {
    if (count) RSF_CUDA(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, s));
  }
  std::vector<T> to_host(size_t count) const {
    std::vector<T> v(count);
    download(v.data(), count);
    RSF_CUDA(cudaStreamSynchronize(s));
    return v;
  }
};

// Transient upload ring (per stream): small host arrays that live only until the kernels
// reading them have run (launch descriptors).  Data goes host -> pinned staging ring ->
// device ring with one truly asynchronous copy; when the ring wraps the stream is
// synchronised first, so every earlier reader has finished.  Replaces a cudaMallocAsync
// plus a pageable (host-blocking) copy per launch.
void* ring_upload(cudaStream_t s, const void* h, size_t bytes);
void ring_trim();   // free the retired (outgrown) rings; waits until their last readers ran
template <class T>
struct RPtr { T* p; };
template <class T>
RPtr<T> ring_up(const std::vector<T>& v, cudaStream_t s) {
  return RPtr<T>{static_cast<T*>(ring_upload(s, v.data(), v.size() * sizeof(T)))};
}

// kernel launch counter (diagnostics: the bench reports how many of our
// kernels ran inside the timed region)
extern thread_local long long g_launches;
// Launch trace (diagnostics, RSF_KTRACE=1): an event after every launch on the traced
// stream; the time between consecutive events is attributed to (current phase, launch site).
struct KTrace {
  static bool on();
  static void mark(const char* file, int line);
  static void set_stream(cudaStream_t s);
  static std::string dump();   // "phase|file:line=seconds,count;..." (synchronises)
  static void reset();
  static const char*& phase();   // current phase label (set by PhaseTimer / PhaseSeq)
};
inline void count_launch_at(const char* file, int line, long long k = 1) {
  g_launches += k;
  if (KTrace::on()) KTrace::mark(file, line);
}
#define count_launch(...) ::rsf::count_launch_at(__FILE__, __LINE__ __VA_OPT__(, ) __VA_ARGS__)

// Phase profiler (enabled by RSF_PROFILE=1): synchronises the stream at the
// scope boundaries and accumulates wall time per named phase.
struct Prof {
  static bool enabled();
  static void add(const char* name, double sec);
  static std::string dump();
  static void reset();
};
// per-level phase names wanted (profiling, GEMM log or NVTX ranges on)
bool phase_names_on();
struct PhaseTimer {
  const char* name;
  cudaStream_t s;
  double t0 = 0;
  bool on;
  const char* prev_phase;
  PhaseTimer(const char* n, cudaStream_t st);
  ~PhaseTimer();
};
// consecutive named phases inside one scope: next(name) closes the previous phase
struct PhaseSeq {
  cudaStream_t s;
  const char* name = nullptr;
  bool open_ = false;   // an NVTX range of this sequence is open
  double t0 = 0;
  bool on;
  const char* prev_phase;
  explicit PhaseSeq(cudaStream_t st);
  void next(const char* n);
  ~PhaseSeq() { next(nullptr); }
};
#define RSF_CAT2(a, b) a##b
#define RSF_CAT(a, b) RSF_CAT2(a, b)
#define RSF_PHASE(name, stream) ::rsf::PhaseTimer RSF_CAT(_rsf_pt_, __LINE__)(name, stream)

// Kernel statistics for the roofline (enabled by rsf_stats_enable): CUDA events
// around every batched-GEMM launch on its own stream, plus algorithmic flops.
struct KStats {
  static bool on;
  static void record(cudaStream_t s, cudaEvent_t* e0, cudaEvent_t* e1);
  static void push(cudaEvent_t e0, cudaEvent_t e1, double flops, double bytes);
  // returns {launches, seconds, flops, bytes}; synchronises pending events
  static void collect(double out[4]);
  static void reset();
};

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace rsf

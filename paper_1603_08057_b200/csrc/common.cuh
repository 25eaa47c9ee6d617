// Common runtime pieces of librsf: error type, stream-ordered device buffers,
// launch checks.  Internal header (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>

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
    if (count) RSF_CUDA(cudaMallocAsync((void**)&p, count * sizeof(T), st));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  void zero() { if (n) RSF_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s)); }
  void upload(const T* h, size_t count) {
    if (count > n) alloc(count, s);
    if (count) RSF_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
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

// kernel launch counter (diagnostics: the bench reports how many of our
// kernels ran inside the timed region)
extern thread_local long long g_launches;
inline void count_launch(long long k = 1) { g_launches += k; }

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace rsf

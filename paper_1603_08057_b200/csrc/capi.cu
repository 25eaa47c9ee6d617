// C ABI of librsf (include/rsf.h): argument checking, host/device staging,
// exception -> status translation.
#include <chrono>
#include <cmath>
#include <cstring>

#include "../../include/rsf.h"
#include "peel.cuh"
#include "rsf_impl.cuh"

struct rsf_ctx_s {
  rsf::Ctx ctx;
};
struct rsf_fact_s {
  std::unique_ptr<rsf::Fact> F;
  rsf_ctx_s* owner = nullptr;
};

namespace {

thread_local std::string g_err;

rsf_status fail(int code, const std::string& msg) {
  g_err = msg;
  return (rsf_status)code;
}

template <class Fn>
rsf_status guard(Fn&& fn) {
  try {
    g_err.clear();
    fn();
    return RSF_OK;
  } catch (const rsf::Error& e) {
    return fail(e.code, e.what());
  } catch (const std::bad_alloc&) {
    return fail(RSF_ENOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(RSF_ECUDA, e.what());
  }
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

rsf::Opts make_opts(const rsf_opts* o) {
  rsf::Opts r;
  if (!o) return r;
  if (o->eps_peel > 0) r.eps_peel = o->eps_peel;
  if (o->oversample > 0) r.oversample = o->oversample;
  if (o->probe_block > 0) r.probe_block = o->probe_block;
  if (o->peel_start > 0) r.peel_start = o->peel_start;
  if (o->max_depth > 0) r.max_depth = o->max_depth;
  if (o->r_near > 0) r.r_near = o->r_near;
  if (o->r_in > 0) r.r_in = o->r_in;
  if (o->r_out > 0) r.r_out = o->r_out;
  r.seed = o->seed;
  r.strong = o->strong != 0;
  r.peel_f32 = o->peel_f32 != 0;
  return r;
}

rsf::KParams check_kernel(const rsf_kernel* k) {
  RSF_REQUIRE(k != nullptr, rsf::ST_EINVAL, "kernel is NULL");
  RSF_REQUIRE(k->family >= 0 && k->family <= 4, rsf::ST_EINVAL, "unknown kernel family");
  RSF_REQUIRE(std::isfinite(k->rho) && k->rho > 0, rsf::ST_EINVAL, "rho must be > 0");
  RSF_REQUIRE(std::isfinite(k->sigma2) && k->sigma2 > 0, rsf::ST_EINVAL, "sigma2 must be > 0");
  RSF_REQUIRE(std::isfinite(k->nugget) && k->nugget >= 0, rsf::ST_EINVAL, "nugget must be >= 0");
  RSF_REQUIRE(std::isfinite(k->alpha) && (k->family != rsf::FAM_RQ || k->alpha > 0), rsf::ST_EINVAL,
              "alpha must be > 0");
  RSF_REQUIRE(std::isfinite(k->rho2) && k->rho2 >= 0, rsf::ST_EINVAL, "rho2 must be >= 0 (0: isotropic)");
  RSF_REQUIRE(k->p >= 0 && k->p <= 4, rsf::ST_EINVAL, "p out of range");
  for (int i = 0; i < k->p; ++i) {
    RSF_REQUIRE(k->theta[i] >= 0 && k->theta[i] <= 4, rsf::ST_EINVAL, "unknown theta component");
    RSF_REQUIRE(k->theta[i] != RSF_RHO2 || k->rho2 > 0, rsf::ST_EINVAL, "rho2 is a parameter of anisotropic kernels");
    RSF_REQUIRE(k->theta[i] != RSF_ALPHA || k->family == RSF_RQ, rsf::ST_EINVAL, "alpha is an RQ parameter");
    for (int j = 0; j < i; ++j) RSF_REQUIRE(k->theta[i] != k->theta[j], rsf::ST_EINVAL, "repeated theta component");
  }
  return rsf::KParams{k->family, k->rho, k->sigma2, k->nugget, k->alpha, k->rho2};
}

// device copy of a (possibly host) n x 2 point array
const double* stage_points(rsf::Ctx& c, const double* xy, int64_t n, rsf::DBuf<double>& keep) {
  if (is_device_ptr(xy)) return xy;
  keep.alloc(2 * n, c.stream);
  keep.upload(xy, 2 * n);
  return keep.p;
}

// run op on X' chunks of at most kmax columns; in/out in caller layout
template <class Op>
void blocked_op(const rsf::Fact& F, const double* in, double* out, int64_t nrhs, int64_t ld, Op op) {
  rsf::Ctx& c = *F.ctx;
  cudaStream_t s = c.stream;
  const int n = F.n();
  RSF_REQUIRE(in && out, rsf::ST_EINVAL, "null vector");
  RSF_REQUIRE(nrhs >= 0, rsf::ST_EINVAL, "nrhs < 0");
  RSF_REQUIRE(ld >= n, rsf::ST_EINVAL, "ld < n");
  if (nrhs == 0) return;
  const bool din = is_device_ptr(in), dout = is_device_ptr(out);
  const int kmax = 256;
  for (int64_t j0 = 0; j0 < nrhs; j0 += kmax) {
    const int k = (int)std::min<int64_t>(kmax, nrhs - j0);
    rsf::DBuf<double> stage;
    const double* src = in + j0 * ld;
    long long lds = ld;
    if (!din) {
      stage.alloc((size_t)n * k, s);
      for (int j = 0; j < k; ++j)
        RSF_CUDA(cudaMemcpyAsync(stage.p + (size_t)j * n, src + j * ld, n * sizeof(double), cudaMemcpyHostToDevice, s));
      src = stage.p;
      lds = n;
    }
    rsf::DBuf<double> X((size_t)n * k, s);
    rsf::to_internal(s, *F.tree, src, lds, k, X.p);
    op(X.p, k);
    if (dout) {
      rsf::to_external(s, *F.tree, X.p, k, out + j0 * ld, ld);
    } else {
      rsf::DBuf<double> o((size_t)n * k, s);
      rsf::to_external(s, *F.tree, X.p, k, o.p, n);
      for (int j = 0; j < k; ++j)
        RSF_CUDA(cudaMemcpyAsync(out + (j0 + j) * ld, o.p + (size_t)j * n, n * sizeof(double), cudaMemcpyDeviceToHost, s));
      RSF_CUDA(cudaStreamSynchronize(s));
    }
  }
  RSF_CUDA(cudaStreamSynchronize(s));
}

// conditional sampling helpers (gp_cond_sample): column-major blocks, k columns
__global__ void cs_diff_kernel(double* d, const double* z, const double* Y, int m, int n2, int N, int k) {
  // d(:, j) = z - Y(m:, j)   (d: n2 x k, Y: N x k)
  const long long tot = (long long)n2 * k;
  for (long long e = blockIdx.x * 256ll + threadIdx.x; e < tot; e += (long long)gridDim.x * 256) {
    const long long j = e / n2, i = e - j * n2;
    d[e] = z[i] - Y[j * N + m + i];
  }
}
__global__ void cs_pad_kernel(double* g, const double* e, int m, int n2, int N, int k) {
  // g(:, j) = [0_m; e(:, j)]
  const long long tot = (long long)N * k;
  for (long long x = blockIdx.x * 256ll + threadIdx.x; x < tot; x += (long long)gridDim.x * 256) {
    const long long j = x / N, i = x - j * N;
    g[x] = i < m ? 0.0 : e[j * n2 + (i - m)];
  }
}
__global__ void cs_out_kernel(double* out, long long ldo, const double* Y, const double* f, int m, int N, int k) {
  // out(:, j) = Y(0:m, j) + f(0:m, j)
  const long long tot = (long long)m * k;
  for (long long x = blockIdx.x * 256ll + threadIdx.x; x < tot; x += (long long)gridDim.x * 256) {
    const long long j = x / m, i = x - j * m;
    out[j * ldo + i] = Y[j * N + i] + f[j * N + i];
  }
}
int cs_grid(long long tot) { return (int)std::max<long long>(1, std::min<long long>((tot + 255) / 256, 4096)); }

// operators of a second handle (F_i) on the first handle's stream: order after F_i's context
// stream, then redirect (StreamScope) every operator of the call to F's stream
void join_stream(cudaStream_t s, rsf_fact other) {
  if (!other || other->owner->ctx.stream == s) return;
  cudaEvent_t ev;
  RSF_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  RSF_CUDA(cudaEventRecord(ev, other->owner->ctx.stream));
  RSF_CUDA(cudaStreamWaitEvent(s, ev, 0));
  cudaEventDestroy(ev);
}

}  // namespace

extern "C" {

void rsf_opts_default(rsf_opts* o) {
  if (!o) return;
  rsf::Opts d;
  o->eps_peel = d.eps_peel;
  o->oversample = d.oversample;
  o->probe_block = d.probe_block;
  o->peel_start = d.peel_start;
  o->max_depth = d.max_depth;
  o->r_near = d.r_near;
  o->r_in = d.r_in;
  o->r_out = d.r_out;
  o->seed = d.seed;
  o->strong = d.strong;
  o->peel_f32 = d.peel_f32;
}

rsf_status rsf_ctx_create(int device, void* cuda_stream, void* nccl_comm, rsf_ctx* out) {
  return guard([&] {
    RSF_REQUIRE(out != nullptr, rsf::ST_EINVAL, "out is NULL");
    int ndev = 0;
    RSF_CUDA(cudaGetDeviceCount(&ndev));
    RSF_REQUIRE(device >= 0 && device < ndev, rsf::ST_EINVAL, "no such CUDA device");
    RSF_CUDA(cudaSetDevice(device));
    auto* c = new rsf_ctx_s;
    c->ctx.device = device;
    if (nccl_comm) {   // the caller's communicator: this context is one rank of a sharded group
      try {
        c->ctx.comm.nccl = nccl_comm;
        rsf::nccl_query(nccl_comm, &c->ctx.comm.rank, &c->ctx.comm.world);
      } catch (...) {
        delete c;
        throw;
      }
    }
    if (cuda_stream) {
      c->ctx.stream = (cudaStream_t)cuda_stream;
    } else {
      RSF_CUDA(cudaStreamCreateWithFlags(&c->ctx.stream, cudaStreamNonBlocking));
      c->ctx.own_stream = true;
    }
    // keep freed device blocks cached in the stream-ordered pool across evaluations
    cudaMemPool_t pool;
    RSF_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    RSF_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    *out = c;
  });
}

void rsf_ctx_destroy(rsf_ctx ctx) {
  if (!ctx) return;
  for (cudaStream_t a : ctx->ctx.aux) {
    cudaStreamSynchronize(a);
    rsf::dev_cache_trim(a);
    cudaStreamSynchronize(a);
    cudaStreamDestroy(a);
  }
  cudaStreamSynchronize(ctx->ctx.stream);
  rsf::dev_cache_trim(ctx->ctx.stream);
  cudaStreamSynchronize(ctx->ctx.stream);
  if (ctx->ctx.own_stream) cudaStreamDestroy(ctx->ctx.stream);
  rsf::ring_trim();
  for (auto& jc : ctx->ctx.job_comms)
    if (jc.owned) rsf::nccl_destroy(jc.nccl);
  if (ctx->ctx.comm.owned) rsf::nccl_destroy(ctx->ctx.comm.nccl);
  delete ctx;
}

rsf_status rsf_nccl_unique_id(unsigned char* out) {
  return guard([&] {
    RSF_REQUIRE(out != nullptr, rsf::ST_EINVAL, "out is NULL");
    rsf::nccl_unique_id(out);
  });
}

rsf_status rsf_ctx_create_group(int device, void* cuda_stream, const unsigned char* id, int rank, int world,
                                rsf_ctx* out) {
  return guard([&] {
    RSF_REQUIRE(out != nullptr && id != nullptr, rsf::ST_EINVAL, "null argument");
    RSF_REQUIRE(world >= 1 && rank >= 0 && rank < world, rsf::ST_EINVAL, "rank / world out of range");
    rsf_ctx c = nullptr;
    const rsf_status st = rsf_ctx_create(device, cuda_stream, nullptr, &c);
    if (st != RSF_OK) throw rsf::Error(st, g_err);
    // (RSF_NCCL_FORCE=1: a one-rank group keeps its NCCL communicator and issues every collective
    // of the sharded path through it -- the transport test on one GPU, comm.cuh)
    const char* fe = getenv("RSF_NCCL_FORCE");
    const bool force = world == 1 && fe && fe[0] == '1';
    if (world > 1 || force) {
      try {
        RSF_CUDA(cudaSetDevice(device));
        c->ctx.comm.nccl = rsf::nccl_init_rank(id, rank, world);
        c->ctx.comm.owned = true;
        c->ctx.comm.rank = rank;
        c->ctx.comm.world = world;
        c->ctx.comm.force = force;
      } catch (...) {
        rsf_ctx_destroy(c);
        throw;
      }
    }
    *out = c;
  });
}

rsf_status rsf_ctx_group(rsf_ctx ctx, int* rank, int* world) {
  return guard([&] {
    RSF_REQUIRE(ctx && rank && world, rsf::ST_EINVAL, "null argument");
    *rank = ctx->ctx.comm.rank;
    *world = ctx->ctx.comm.world;
  });
}

int rsf_debug_job_runs(int njobs, int world, int rank, int job) {
  if (njobs < 1 || world < 1 || rank < 0 || rank >= world || job < 0 || job >= njobs) return -1;
  const int G = rsf::Comm::job_groups(njobs, world);
  return (world == 1 || job % G == rank % G) ? 1 : 0;   // (equal job weights: rank r in group r mod G)
}

int64_t rsf_debug_nccl_calls(void) { return (int64_t)rsf::nccl_calls(); }

int rsf_debug_job_group(int ngroups, const double* gw, int world, int rank) {
  if (ngroups < 1 || !gw || world < ngroups || rank < 0 || rank >= world) return -1;
  return rsf::Comm::group_of_rank(std::vector<double>(gw, gw + ngroups), world, rank);
}

void rsf_debug_col_slice(int64_t k, int parts, int part, int64_t* lo, int64_t* hi) {
  long long a = 0, b = 0;
  if (parts >= 1 && part >= 0 && part < parts && k >= 0) rsf::Comm::slice(k, parts, part, &a, &b);
  *lo = a;
  *hi = b;
}

rsf_status rsf_ctx_wait_stream(rsf_ctx ctx, void* stream) {
  return guard([&] {
    RSF_REQUIRE(ctx != nullptr, rsf::ST_EINVAL, "null context");
    RSF_CUDA(cudaSetDevice(ctx->ctx.device));
    cudaStream_t cs = (cudaStream_t)stream;
    if (cs == ctx->ctx.stream) return;
    cudaEvent_t ev;
    RSF_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    RSF_CUDA(cudaEventRecord(ev, cs));
    const cudaError_t e = cudaStreamWaitEvent(ctx->ctx.stream, ev, 0);
    cudaEventDestroy(ev);   // destruction is deferred by the runtime until the wait resolved
    RSF_CUDA(e);
  });
}

rsf_status rsf_factor(rsf_ctx ctx, const double* xy, int64_t n, const rsf_kernel* kernel, int32_t which,
                      double eps, int32_t leaf, const rsf_opts* opts, rsf_fact* out) {
  return guard([&] {
    RSF_REQUIRE(ctx && xy && out, rsf::ST_EINVAL, "null argument");
    RSF_REQUIRE(n >= 1 && n < (1ll << 31), rsf::ST_EINVAL, "n out of range");
    RSF_REQUIRE(eps > 0 && std::isfinite(eps), rsf::ST_EINVAL, "eps must be > 0");
    RSF_REQUIRE(leaf >= 1, rsf::ST_EINVAL, "leaf must be >= 1");
    rsf::KParams kp = check_kernel(kernel);
    int w = rsf::W_SIGMA;
    if (which >= 0) {
      RSF_REQUIRE(which < kernel->p, rsf::ST_EINVAL, "which out of range");
      w = kernel->theta[which];
    } else {
      RSF_REQUIRE(which == -1, rsf::ST_EINVAL, "which must be -1 or a theta index");
    }
    RSF_CUDA(cudaSetDevice(ctx->ctx.device));
    rsf::Opts o = make_opts(opts);
    rsf::DBuf<double> keep;
    const double* dxy = stage_points(ctx->ctx, xy, n, keep);
    auto tree = rsf::build_tree(ctx->ctx, dxy, (int)n, leaf, o.max_depth);
    auto F = rsf::factor(ctx->ctx, tree, kp, w, eps, o);
    auto* h = new rsf_fact_s;
    h->F = std::move(F);
    h->owner = ctx;
    *out = h;
  });
}

void rsf_fact_destroy(rsf_fact f) {
  if (!f) return;
  cudaStreamSynchronize(f->owner->ctx.stream);
  delete f;
}

rsf_status rsf_fact_info(rsf_fact f, rsf_fact_diag* out) {
  return guard([&] {
    RSF_REQUIRE(f && out, rsf::ST_EINVAL, "null argument");
    std::memset(out, 0, sizeof(*out));
    const rsf::Fact& F = *f->F;
    out->levels = F.tree->L;
    out->top_size = F.n0;
    const auto& d = F.diag;
    for (size_t i = 0; i < d.level_boxes.size() && i < 32; ++i) {
      int lev = F.tree->L - (int)i;   // recorded from L down to 1
      if (lev < 0 || lev >= 32) continue;
      out->level_boxes[lev] = d.level_boxes[i];
      out->level_active[lev] = d.level_I[i];
      out->level_skel[lev] = d.level_S[i];
      out->level_maxI[lev] = d.level_maxI[i];
    }
    out->flops_id = d.flops_id;
    out->flops_elim = d.flops_elim;
    out->flops_top = d.flops_top;
    out->factor_bytes = d.bytes_factor;
    out->seconds = d.t_factor;
  });
}

rsf_status rsf_logdet(rsf_fact f, double* out) {
  return guard([&] {
    RSF_REQUIRE(f && out, rsf::ST_EINVAL, "null argument");
    RSF_REQUIRE(f->F->which == rsf::W_SIGMA, rsf::ST_EINVAL, "logdet of a Sigma_i handle");
    *out = f->F->logdet;
  });
}

rsf_status rsf_solve(rsf_fact f, const double* b, double* x, int64_t nrhs, int64_t ld) {
  return guard([&] {
    RSF_REQUIRE(f, rsf::ST_EINVAL, "null handle");
    RSF_REQUIRE(f->F->which == rsf::W_SIGMA, rsf::ST_EINVAL, "solve with a Sigma_i handle");
    RSF_CUDA(cudaSetDevice(f->owner->ctx.device));
    const rsf::Fact& F = *f->F;
    blocked_op(F, b, x, nrhs, ld, [&](double* X, int k) {
      rsf::DBuf<double> tmp((size_t)std::max<long long>(F.tmp_cols, 1) * k, F.ctx->stream);
      rsf::solve_internal(F, X, k, tmp.p);
    });
  });
}

rsf_status rsf_apply(rsf_fact f, const double* x, double* y, int64_t nrhs, int64_t ld) {
  return guard([&] {
    RSF_REQUIRE(f, rsf::ST_EINVAL, "null handle");
    RSF_CUDA(cudaSetDevice(f->owner->ctx.device));
    const rsf::Fact& F = *f->F;
    blocked_op(F, x, y, nrhs, ld, [&](double* X, int k) {
      cudaStream_t s = F.ctx->stream;
      if (F.which == rsf::W_SIGMA) {
        rsf::DBuf<double> tmp((size_t)std::max<long long>(F.tmp_cols, 1) * k, s);
        rsf::apply_internal(F, X, k, tmp.p);
      } else {
        rsf::DBuf<double> Y((size_t)F.n() * k, s);
        rsf::apply_only_internal(F, X, Y.p, k);
        RSF_CUDA(cudaMemcpyAsync(X, Y.p, (size_t)F.n() * k * sizeof(double), cudaMemcpyDeviceToDevice, s));
      }
    });
  });
}

rsf_status rsf_sample(rsf_fact f, const double* w, double* z, int64_t nrhs, int64_t ld) {
  return guard([&] {
    RSF_REQUIRE(f, rsf::ST_EINVAL, "null handle");
    RSF_REQUIRE(f->F->which == rsf::W_SIGMA, rsf::ST_EINVAL, "sample with a Sigma_i handle");
    RSF_CUDA(cudaSetDevice(f->owner->ctx.device));
    const rsf::Fact& F = *f->F;
    blocked_op(F, w, z, nrhs, ld, [&](double* X, int k) {
      rsf::DBuf<double> tmp((size_t)std::max<long long>(F.tmp_cols, 1) * k, F.ctx->stream);
      rsf::sqrt_internal(F, X, k, tmp.p);
    });
  });
}

rsf_status hutch_trace(rsf_fact F, rsf_fact Fi, int64_t nprobe, uint64_t seed, double* trace, double* std_err) {
  return guard([&] {
    RSF_REQUIRE(F && trace && std_err, rsf::ST_EINVAL, "null argument");
    RSF_REQUIRE(F->F->which == rsf::W_SIGMA, rsf::ST_EINVAL, "F must be a Sigma factor");
    RSF_REQUIRE(!Fi || Fi->F->which != rsf::W_SIGMA, rsf::ST_EINVAL, "Fi must be a Sigma_i compression");
    RSF_REQUIRE(!Fi || Fi->F->n() == F->F->n(), rsf::ST_EINVAL, "dimension mismatch");
    RSF_REQUIRE(nprobe >= 1, rsf::ST_EINVAL, "nprobe must be >= 1");
    RSF_CUDA(cudaSetDevice(F->owner->ctx.device));
    join_stream(F->owner->ctx.stream, Fi);
    rsf::StreamScope scope(F->owner->ctx.stream);
    rsf::hutch(*F->F, Fi ? Fi->F.get() : nullptr, nprobe, seed, trace, std_err);
  });
}

rsf_status peel_trace(rsf_fact F, rsf_fact Fi, double eps_peel, const rsf_opts* opts, int32_t trace_id,
                      double* trace, rsf_peel_diag* diag) {
  return guard([&] {
    RSF_REQUIRE(F && trace, rsf::ST_EINVAL, "null argument");
    RSF_REQUIRE(F->F->which == rsf::W_SIGMA, rsf::ST_EINVAL, "F must be a Sigma factor");
    RSF_REQUIRE(!Fi || Fi->F->which != rsf::W_SIGMA, rsf::ST_EINVAL, "Fi must be a Sigma_i compression");
    RSF_REQUIRE(!Fi || Fi->F->n() == F->F->n(), rsf::ST_EINVAL, "dimension mismatch");
    RSF_REQUIRE(eps_peel > 0, rsf::ST_EINVAL, "eps_peel must be > 0");
    RSF_CUDA(cudaSetDevice(F->owner->ctx.device));
    join_stream(F->owner->ctx.stream, Fi);
    rsf::StreamScope scope(F->owner->ctx.stream);
    rsf::Opts o = opts ? make_opts(opts) : F->F->opts;
    o.eps_peel = eps_peel;
    rsf::PeelDiag pd;
    *trace = rsf::peel(*F->F, Fi ? Fi->F.get() : nullptr, o, trace_id, &pd);
    if (diag) rsf::fill_peel_diag(pd, diag);
  });
}

rsf_status gp_mle_eval(rsf_ctx ctx, const double* xy, const double* z, int64_t n, const rsf_kernel* kernel,
                       double eps, int32_t leaf, const rsf_opts* opts, double* ell, double* grad,
                       rsf_eval_diag* diag) {
  return guard([&] {
    RSF_REQUIRE(ctx && xy && z && ell, rsf::ST_EINVAL, "null argument");
    RSF_REQUIRE(n >= 1 && n < (1ll << 31), rsf::ST_EINVAL, "n out of range");
    RSF_REQUIRE(eps > 0 && std::isfinite(eps), rsf::ST_EINVAL, "eps must be > 0");
    RSF_REQUIRE(leaf >= 1, rsf::ST_EINVAL, "leaf must be >= 1");
    rsf::KParams kp = check_kernel(kernel);
    RSF_REQUIRE(kernel->p == 0 || grad != nullptr, rsf::ST_EINVAL, "grad is NULL");
    RSF_CUDA(cudaSetDevice(ctx->ctx.device));
    rsf::Opts o = make_opts(opts);
    rsf::EvalResult r = rsf::mle_eval(ctx->ctx, xy, z, (int)n, kp, kernel->p, kernel->theta, eps, leaf, o);
    *ell = r.ell;
    for (int i = 0; i < kernel->p; ++i) grad[i] = r.grad[i];
    if (diag) rsf::fill_eval_diag(r, diag);
  });
}

rsf_status gp_profile_eval(rsf_ctx ctx, const double* xy, const double* z, int64_t n, const rsf_kernel* kernel,
                           double eps, int32_t leaf, const rsf_opts* opts, double* ell, double* grad,
                           rsf_eval_diag* diag) {
  return guard([&] {
    RSF_REQUIRE(ctx && xy && z && ell, rsf::ST_EINVAL, "null argument");
    RSF_REQUIRE(n >= 2 && n < (1ll << 31), rsf::ST_EINVAL, "n out of range");
    RSF_REQUIRE(eps > 0 && std::isfinite(eps), rsf::ST_EINVAL, "eps must be > 0");
    RSF_REQUIRE(leaf >= 1, rsf::ST_EINVAL, "leaf must be >= 1");
    rsf::KParams kp = check_kernel(kernel);
    RSF_REQUIRE(kernel->p == 0 || grad != nullptr, rsf::ST_EINVAL, "grad is NULL");
    for (int i = 0; i < kernel->p; ++i)
      RSF_REQUIRE(kernel->theta[i] != RSF_SIGMA2, rsf::ST_EINVAL, "sigma2 is profiled out (not a theta component)");
    RSF_CUDA(cudaSetDevice(ctx->ctx.device));
    rsf::Opts o = make_opts(opts);
    rsf::EvalResult r = rsf::mle_eval(ctx->ctx, xy, z, (int)n, kp, kernel->p, kernel->theta, eps, leaf, o, true);
    *ell = r.ell;
    for (int i = 0; i < kernel->p; ++i) grad[i] = r.grad[i];
    if (diag) rsf::fill_eval_diag(r, diag);
  });
}

rsf_status gp_cond_mean(rsf_fact F, const double* z, const double* xy_new, int64_t m, double* out) {
  return guard([&] {
    RSF_REQUIRE(F && z && (m == 0 || (xy_new && out)), rsf::ST_EINVAL, "null argument");
    RSF_REQUIRE(F->F->which == rsf::W_SIGMA, rsf::ST_EINVAL, "F must be a Sigma factor");
    RSF_REQUIRE(m >= 0, rsf::ST_EINVAL, "m < 0");
    RSF_CUDA(cudaSetDevice(F->owner->ctx.device));
    const rsf::Fact& f = *F->F;
    cudaStream_t s = f.ctx->stream;
    const int n = f.n();
    rsf::DBuf<double> zd, xd, od;
    const double* dz = z;
    const double* dx = xy_new;
    double* dout = out;
    if (!is_device_ptr(z)) { zd.alloc(n, s); zd.upload(z, n); dz = zd.p; }
    if (m > 0 && !is_device_ptr(xy_new)) { xd.alloc(2 * (size_t)m, s); xd.upload(xy_new, 2 * (size_t)m); dx = xd.p; }
    const bool host_out = m > 0 && !is_device_ptr(out);
    if (host_out) { od.alloc((size_t)m, s); dout = od.p; }
    rsf::cond_mean(f, dz, dx, m, dout);
    if (host_out) RSF_CUDA(cudaMemcpyAsync(out, od.p, (size_t)m * sizeof(double), cudaMemcpyDeviceToHost, s));
    RSF_CUDA(cudaStreamSynchronize(s));
  });
}

rsf_status gp_cond_sample(rsf_fact F, rsf_fact F22, int64_t m, const double* z, const double* w, double* out,
                          int64_t nrhs) {
  return guard([&] {
    RSF_REQUIRE(F && F22 && z && w && out, rsf::ST_EINVAL, "null argument");
    RSF_REQUIRE(F->F->which == rsf::W_SIGMA && F22->F->which == rsf::W_SIGMA, rsf::ST_EINVAL,
                "F and F22 must be Sigma factors");
    RSF_REQUIRE(!F->F->solve_only, rsf::ST_EINVAL, "F must be a full factor (rsf_factor)");
    RSF_REQUIRE(m >= 1 && F->F->n() == m + F22->F->n(), rsf::ST_EINVAL,
                "F must factor the m new points followed by the n2 data points of F22");
    RSF_REQUIRE(nrhs >= 0, rsf::ST_EINVAL, "nrhs < 0");
    RSF_REQUIRE(F->owner->ctx.device == F22->owner->ctx.device, rsf::ST_EINVAL, "F and F22 on different devices");
    RSF_CUDA(cudaSetDevice(F->owner->ctx.device));
    const rsf::Fact& fj = *F->F;
    const rsf::Fact& fd = *F22->F;
    cudaStream_t s = fj.ctx->stream;
    // every operator below runs on F's stream (F22 may belong to another context / stream)
    if (F22->owner->ctx.stream != s) {
      cudaEvent_t ev;
      RSF_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      RSF_CUDA(cudaEventRecord(ev, F22->owner->ctx.stream));
      RSF_CUDA(cudaStreamWaitEvent(s, ev, 0));
      cudaEventDestroy(ev);
    }
    rsf::StreamScope scope(s);
    const int N = fj.n(), n2 = fd.n();
    if (nrhs == 0) return;
    rsf::DBuf<double> zd;
    const double* dz = z;
    if (!is_device_ptr(z)) { zd.alloc(n2, s); zd.upload(z, n2); dz = zd.p; }
    const bool dw = is_device_ptr(w), dout = is_device_ptr(out);
    const int kmax = 256;
    for (int64_t j0 = 0; j0 < nrhs; j0 += kmax) {
      const int k = (int)std::min<int64_t>(kmax, nrhs - j0);
      // y = F^{1/2} w (joint order: new points first)
      rsf::DBuf<double> wst, Y((size_t)N * k, s), X((size_t)N * k, s),
          tmpj((size_t)std::max<long long>(fj.tmp_cols, 1) * k, s), tmpd((size_t)std::max<long long>(fd.tmp_cols, 1) * k, s);
      const double* src = w + j0 * (int64_t)N;
      if (!dw) { wst.alloc((size_t)N * k, s); wst.upload(src, (size_t)N * k); src = wst.p; }
      rsf::to_internal(s, *fj.tree, src, N, k, X.p);
      rsf::sqrt_internal(fj, X.p, k, tmpj.p);
      rsf::to_external(s, *fj.tree, X.p, k, Y.p, N);
      // e = F22^-1 (z - y_2)
      rsf::DBuf<double> D((size_t)n2 * k, s), Xd((size_t)n2 * k, s);
      cs_diff_kernel<<<cs_grid((long long)n2 * k), 256, 0, s>>>(D.p, dz, Y.p, (int)m, n2, N, k);
      count_launch();
      rsf::to_internal(s, *fd.tree, D.p, n2, k, Xd.p);
      rsf::solve_internal(fd, Xd.p, k, tmpd.p);
      rsf::to_external(s, *fd.tree, Xd.p, k, D.p, n2);
      // f = F [0; e]  (its first m rows apply Sigma_12 e, "through appropriate padding")
      rsf::DBuf<double> G((size_t)N * k, s);
      cs_pad_kernel<<<cs_grid((long long)N * k), 256, 0, s>>>(G.p, D.p, (int)m, n2, N, k);
      count_launch();
      rsf::to_internal(s, *fj.tree, G.p, N, k, X.p);
      rsf::apply_internal(fj, X.p, k, tmpj.p);
      rsf::to_external(s, *fj.tree, X.p, k, G.p, N);
      // out = y_1 + f_1 = mu + [I, -Sigma_12 F22^-1] F^{1/2} w
      if (dout) {
        cs_out_kernel<<<cs_grid((long long)m * k), 256, 0, s>>>(out + j0 * m, m, Y.p, G.p, (int)m, N, k);
        count_launch();
      } else {
        rsf::DBuf<double> O((size_t)m * k, s);
        cs_out_kernel<<<cs_grid((long long)m * k), 256, 0, s>>>(O.p, m, Y.p, G.p, (int)m, N, k);
        count_launch();
        RSF_CUDA(cudaMemcpyAsync(out + j0 * m, O.p, (size_t)m * k * sizeof(double), cudaMemcpyDeviceToHost, s));
        RSF_CUDA(cudaStreamSynchronize(s));
      }
      RSF_LAUNCH_CHECK();
    }
    RSF_CUDA(cudaStreamSynchronize(s));
  });
}

const char* rsf_last_error(void) { return g_err.c_str(); }

int64_t rsf_kernel_launches(void) { return rsf::g_launches; }

const char* rsf_profile_dump(void) {
  static thread_local std::string s;
  s = rsf::Prof::dump();
  return s.c_str();
}
void rsf_profile_reset(void) { rsf::Prof::reset(); rsf::KTrace::reset(); rsf::GemmLog::reset(); }

const char* rsf_trace_dump(void) {
  static thread_local std::string s;
  s = rsf::KTrace::dump();
  return s.c_str();
}

const char* rsf_debug_gemm_log(void) {
  static thread_local std::string s;
  s = rsf::GemmLog::dump();
  return s.c_str();
}

int rsf_debug_gemm(int ta, int tb, int M, int N, int K, int batch, double alpha, const double* A,
                   const double* B, double beta, double* C, int splitk) {
  // diagnostics / tests: C_i = alpha op(A_i) op(B_i) + beta C_i on `batch` contiguous problems (device
  // pointers, column-major, packed leading dimensions) through the batched pipelined GEMM
  try {
    if (M < 0 || N < 0 || K < 0 || batch < 0 || !A || !B || !C) return RSF_EINVAL;
    cudaStream_t s = 0;
    const size_t sa = (size_t)M * K, sb = (size_t)K * N, sc = (size_t)M * N;
    rsf::GemmBatch g(ta != 0, tb != 0);
    for (int i = 0; i < batch; ++i) {
      rsf::GemmDesc d = rsf::gdesc(M, N, K);
      d.A = A + sa * i; d.lda = std::max(1, ta ? K : M);
      d.B = B + sb * i; d.ldb = std::max(1, tb ? N : K);
      d.C = C + sc * i; d.ldc = std::max(1, M);
      d.alpha = alpha; d.beta = beta;
      g.add(d);
    }
    rsf::gemm_force_splitk() = splitk;
    g.run(s);
    rsf::gemm_force_splitk() = 0;
    RSF_CUDA(cudaStreamSynchronize(s));
    return RSF_OK;
  } catch (...) {
    rsf::gemm_force_splitk() = 0;
    return RSF_ECUDA;
  }
}

double rsf_debug_gemm_bench(int M, int N, int K, int batch, int ta, int tb, int reps) {
  // diagnostics: TFLOP/s of the batched FP64 GEMM on `batch` independent M x N x K problems
  try {
    cudaStream_t s = 0;   // legacy default stream (buffers are released before return)
    const size_t sa = (size_t)M * K, sb = (size_t)K * N, sc = (size_t)M * N;
    rsf::DBuf<double> A(sa * batch, s), B(sb * batch, s), C(sc * batch, s);
    A.zero(); B.zero(); C.zero();
    rsf::GemmBatch g(ta != 0, tb != 0);
    for (int i = 0; i < batch; ++i) {
      rsf::GemmDesc d = rsf::gdesc(M, N, K);
      d.A = A.p + sa * i; d.lda = ta ? K : M;
      d.B = B.p + sb * i; d.ldb = tb ? N : K;
      d.C = C.p + sc * i; d.ldc = M;
      g.add(d);
    }
    g.finalize(s);
    g.run(s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int r = 0; r < reps; ++r) g.run(s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaStreamSynchronize(s);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return 2.0 * M * N * (double)K * batch * reps / (ms * 1e-3) / 1e12;
  } catch (...) {
    return -1.0;
  }
}

namespace {
// FP64 peak probes (roofline denominator, measured live by bench.py): independent
// DMMA.8x8x4 (mma.sync m8n8k4 f64) or DFMA chains, no memory traffic.
__global__ void peak_dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-7;
  double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int q = 0; q < 4; ++q) s += c[q][0] + c[q][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void peak_dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
}  // namespace

double rsf_debug_fp64_peak(int dmma, int reps) {
  try {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = sms * 4, threads = 512, iters = 4000;
    rsf::DBuf<double> out((size_t)blocks * threads, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0.0;
    for (int r = 0; r < std::max(reps, 1) + 1; ++r) {
      cudaEventRecord(e0, 0);
      if (dmma) peak_dmma_kernel<<<blocks, threads>>>(out.p, iters);
      else peak_dfma_kernel<<<blocks, threads>>>(out.p, iters);
      cudaEventRecord(e1, 0);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fl = dmma ? 2.0 * 8 * 8 * 4 * 16 * (double)iters * blocks * (threads / 32)
                             : 2.0 * 8 * 16 * (double)iters * blocks * threads;
      if (r > 0) best = std::max(best, fl / (ms * 1e-3) / 1e12);   // first launch = warm-up
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaDeviceSynchronize();
    return best;
  } catch (...) {
    return -1.0;
  }
}

double rsf_debug_solve_bench(rsf_fact f, int nrhs, int reps, double* bytes) {
  // diagnostics (bench.py "solve" roofline): device time of one F^-1 X sweep pair
  // on nrhs internal-layout columns (CUDA events on the op stream, after one warm-up), and
  // its algorithmic bytes for nrhs = 1 (FactDiag::bytes_solve)
  try {
    if (!f || f->F->which != rsf::W_SIGMA || nrhs < 1 || reps < 1) return -1.0;
    const rsf::Fact& F = *f->F;
    RSF_CUDA(cudaSetDevice(f->owner->ctx.device));
    cudaStream_t s = rsf::op_stream(F);
    rsf::KTrace::set_stream(s);   // (RSF_KTRACE=1: time per launch site, rsf_trace_dump)
    rsf::DBuf<double> X((size_t)F.n() * nrhs, s), tmp((size_t)std::max<long long>(F.tmp_cols, 1) * nrhs, s);
    RSF_CUDA(cudaMemsetAsync(X.p, 0, (size_t)F.n() * nrhs * sizeof(double), s));
    rsf::solve_internal(F, X.p, nrhs, tmp.p);
    cudaEvent_t e0, e1;
    RSF_CUDA(cudaEventCreate(&e0));
    RSF_CUDA(cudaEventCreate(&e1));
    RSF_CUDA(cudaEventRecord(e0, s));
    for (int r = 0; r < reps; ++r) rsf::solve_internal(F, X.p, nrhs, tmp.p);
    RSF_CUDA(cudaEventRecord(e1, s));
    RSF_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    RSF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (bytes) *bytes = F.diag.bytes_solve;
    return ms * 1e-3 / reps;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

void rsf_stats_enable(int on) { rsf::KStats::on = on != 0; }
void rsf_stats_get(double* out4) { rsf::KStats::collect(out4); }
void rsf_stats_reset(void) { rsf::KStats::reset(); }

}  // extern "C"

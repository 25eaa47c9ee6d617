// Quadtree on the GPU-sorted Morton order.
//   a1: 60-bit Morton keys on the root [0,1]^2 (kernel) + stable radix sort
//       (CUB) of (key, original index) -> permutation.
//   a2: adaptive split while a box holds more than `leaf` points (PAPER P:202,
//       P:192): boxes are contiguous key ranges; the split of a range is a
//       binary search on its next 2-bit key digit (host scheduler; the tree is
//       the metadata the per-level launches are built from).
#include <cub/cub.cuh>

#include <algorithm>
#include <functional>

#include "rsf_impl.cuh"

namespace rsf {

namespace {

__device__ __forceinline__ unsigned long long spread(unsigned int v) {
  unsigned long long x = v & 0x3fffffffu;
  x = (x | (x << 16)) & 0x0000ffff0000ffffull;
  x = (x | (x << 8)) & 0x00ff00ff00ff00ffull;
  x = (x | (x << 4)) & 0x0f0f0f0f0f0f0f0full;
  x = (x | (x << 2)) & 0x3333333333333333ull;
  x = (x | (x << 1)) & 0x5555555555555555ull;
  return x;
}

__global__ void morton_kernel(const double* __restrict__ xy, int n, unsigned long long* keys,
                              int* idx, int* bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = xy[2 * i], y = xy[2 * i + 1];
  if (!(x >= 0.0 && x <= 1.0 && y >= 0.0 && y <= 1.0)) {   // also catches NaN
    atomicExch(bad, 1);
    x = 0.0; y = 0.0;
  }
  const double S = 1073741824.0;   // 2^30 (exact scaling: split lines are dyadic)
  unsigned int xi = (unsigned int)fmin(floor(x * S), S - 1.0);
  unsigned int yi = (unsigned int)fmin(floor(y * S), S - 1.0);
  keys[i] = spread(xi) | (spread(yi) << 1);
  idx[i] = i;
}

__global__ void gather_xy_kernel(const double* __restrict__ xy, const int* __restrict__ perm, int n,
                                 double* xs, double* ys) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  int o = perm[t];
  xs[t] = xy[2 * o];
  ys[t] = xy[2 * o + 1];
}

inline unsigned int compact1(unsigned long long x) {
  x &= 0x5555555555555555ull;
  x = (x | (x >> 1)) & 0x3333333333333333ull;
  x = (x | (x >> 2)) & 0x0f0f0f0f0f0f0f0full;
  x = (x | (x >> 4)) & 0x00ff00ff00ff00ffull;
  x = (x | (x >> 8)) & 0x0000ffff0000ffffull;
  x = (x | (x >> 16)) & 0x00000000ffffffffull;
  return (unsigned int)x;
}

}  // namespace

std::shared_ptr<Tree> build_tree(Ctx& ctx, const double* d_xy, int n, int leaf, int max_depth) {
  RSF_REQUIRE(n >= 1, ST_EINVAL, "n must be >= 1");
  RSF_REQUIRE(leaf >= 1, ST_EINVAL, "leaf must be >= 1");
  max_depth = std::max(0, std::min(max_depth, 30));
  cudaStream_t s = ctx.stream;
  auto t = std::make_shared<Tree>();
  t->n = n;
  t->leaf = leaf;
  DBuf<unsigned long long> keys(n, s), keys2(n, s);
  DBuf<int> idx(n, s), idx2(n, s), bad(1, s);
  bad.zero();
  morton_kernel<<<ceil_div(n, 256), 256, 0, s>>>(d_xy, n, keys.p, idx.p, bad.p);
  count_launch();
  RSF_LAUNCH_CHECK();
  size_t tmp_bytes = 0;
  RSF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.p, keys2.p, idx.p, idx2.p, n, 0, 60, s));
  DBuf<char> tmp(tmp_bytes, s);
  RSF_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys.p, keys2.p, idx.p, idx2.p, n, 0, 60, s));
  count_launch();
  std::vector<unsigned long long> hk(n);
  keys2.download(hk.data(), n);
  t->perm.resize(n);
  idx2.download(t->perm.data(), n);
  int hbad = 0;
  bad.download(&hbad, 1);
  RSF_CUDA(cudaStreamSynchronize(s));
  RSF_REQUIRE(!hbad, ST_EINVAL, "coordinates must be finite and lie in the unit square [0,1]^2");
  t->d_perm = std::move(idx2);
  t->xs.alloc(n, s);
  t->ys.alloc(n, s);
  gather_xy_kernel<<<ceil_div(n, 256), 256, 0, s>>>(d_xy, t->d_perm.p, n, t->xs.p, t->ys.p);
  count_launch();
  RSF_LAUNCH_CHECK();
  t->hx.resize(n);
  t->hy.resize(n);
  t->xs.download(t->hx.data(), n);
  t->ys.download(t->hy.data(), n);
  RSF_CUDA(cudaStreamSynchronize(s));

  // host: recursive split of key ranges (DFS in quadrant order = Morton order)
  auto digit = [&](int i, int l) { return (int)((hk[i] >> (2 * (30 - l))) & 3ull); };
  std::function<int(int, int, int, int, int, int)> rec = [&](int l, int x, int y, int b, int e, int par) -> int {
    const int id = (int)t->lev.size();
    t->lev.push_back(l);
    t->parent.push_back(par);
    t->quad.push_back(par < 0 ? 0 : ((x & 1) + 2 * (y & 1)));
    t->begin.push_back(b);
    t->end.push_back(e);
    t->child.push_back({-1, -1, -1, -1});
    t->ix.push_back(x);
    t->iy.push_back(y);
    t->cell[Tree::cell_key(l, x, y)] = id;
    if (e - b > leaf && l < max_depth) {
      int lo = b;
      for (int q = 0; q < 4; ++q) {
        // first index in [lo, e) whose digit at level l+1 exceeds q
        int a = lo, z = e;
        while (a < z) {
          int m = (a + z) >> 1;
          if (digit(m, l + 1) <= q) a = m + 1; else z = m;
        }
        if (a > lo) {
          int c = rec(l + 1, 2 * x + (q & 1), 2 * y + (q >> 1), lo, a, id);
          t->child[id][q] = c;
        }
        lo = a;
      }
    }
    return id;
  };
  rec(0, 0, 0, 0, n, -1);
  int L = 0;
  for (int l : t->lev) L = std::max(L, l);
  t->L = L;
  t->levels.assign(L + 1, {});
  for (int i = 0; i < (int)t->lev.size(); ++i) t->levels[t->lev[i]].push_back(i);
  (void)compact1;
  return t;
}

}  // namespace rsf

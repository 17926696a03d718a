// Quadtree build on the GPU: root box, depth choice, box keys, stable key
// sort, leaf run-length encoding, interpolation weights and M2L operators.
// Restates FmmTree._build (fmm.py:106-135) and its helpers; integer results
// are bit-exact with the reference (checked by tests/test_gpu_parity.py).
#include <cub/cub.cuh>

#include <algorithm>
#include <cfloat>
#include <cmath>

#include "fmm_device.cuh"
#include "tree.h"

namespace hikf {

namespace {

constexpr int kThreads = 256;

// per-block min/max of x and y -> part[4 * block]
__global__ void minmax_partial(const double* __restrict__ xy, int64_t m, double* __restrict__ part) {
  double mn0 = DBL_MAX, mn1 = DBL_MAX, mx0 = -DBL_MAX, mx1 = -DBL_MAX;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    double x = xy[2 * i], y = xy[2 * i + 1];
    mn0 = fmin(mn0, x);
    mx0 = fmax(mx0, x);
    mn1 = fmin(mn1, y);
    mx1 = fmax(mx1, y);
  }
  typedef cub::BlockReduce<double, kThreads> BR;
  __shared__ typename BR::TempStorage tmp;
  double r0 = BR(tmp).Reduce(mn0, cub::Min());
  __syncthreads();
  double r1 = BR(tmp).Reduce(mn1, cub::Min());
  __syncthreads();
  double r2 = BR(tmp).Reduce(mx0, cub::Max());
  __syncthreads();
  double r3 = BR(tmp).Reduce(mx1, cub::Max());
  if (threadIdx.x == 0) {
    part[4 * blockIdx.x + 0] = r0;
    part[4 * blockIdx.x + 1] = r1;
    part[4 * blockIdx.x + 2] = r2;
    part[4 * blockIdx.x + 3] = r3;
  }
}

// box coordinate with the split-line rule of fmm.py:152-164
__device__ __forceinline__ int64_t box_coord(double x, double lo, double h, int64_t G) {
  double u = __ddiv_rn(__dsub_rn(x, lo), h);
  double f = floor(u);
  int64_t b = (int64_t)f;
  if (u == f && b > 0) b -= 1;
  return b < 0 ? 0 : (b > G - 1 ? G - 1 : b);
}

__global__ void box_keys(const double* __restrict__ xy, int64_t m, double lo0, double lo1, double h, int64_t G,
                         int64_t* __restrict__ keys, int32_t* __restrict__ hist) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t key = box_coord(xy[2 * i], lo0, h, G) * G + box_coord(xy[2 * i + 1], lo1, h, G);
    if (keys) keys[i] = key;
    if (hist) atomicAdd(hist + key, 1);
  }
}

__global__ void iota64(int64_t* v, int64_t m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = i;
}

__global__ void inverse_perm(const int64_t* __restrict__ order, int64_t m, int32_t* __restrict__ inv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    inv[order[i]] = (int32_t)i;
}

__global__ void leaf_ranks(const int32_t* __restrict__ start, const int32_t* __restrict__ count, int64_t nl,
                           int32_t* __restrict__ leaf_of) {
  for (int64_t r = blockIdx.x; r < nl; r += gridDim.x)
    for (int32_t i = threadIdx.x; i < count[r]; i += blockDim.x) leaf_of[start[r] + i] = (int32_t)r;
}

__global__ void gather_xy(const double* __restrict__ xy, const int64_t* __restrict__ order, int64_t m,
                          double* __restrict__ xy_s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = order[i];
    xy_s[2 * i] = xy[2 * o];
    xy_s[2 * i + 1] = xy[2 * o + 1];
  }
}

// Leaf interpolation weights (fmm.py:246-262): for each point (sorted order)
// xi = 2((x - lo)/h - bx) - 1; S_k(xi) = (1 + 2 sum_{j>=1} T_j(x_k) T_j(xi)) / n.
__global__ void interp_weights(const double* __restrict__ xy_s, int64_t m, double lo0, double lo1, double h, int64_t G,
                               int n, const double* __restrict__ Tn, double* __restrict__ W2) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
    double w[2][kMaxLeafOrder];
    for (int d = 0; d < 2; ++d) {
      double x = xy_s[2 * p + d], lo = d == 0 ? lo0 : lo1;
      int64_t b = box_coord(x, lo, h, G);
      double xi = __dsub_rn(__dmul_rn(2.0, __dsub_rn(__ddiv_rn(__dsub_rn(x, lo), h), (double)b)), 1.0);
      double T[kMaxLeafOrder];
      T[0] = 1.0;
      if (n > 1) T[1] = xi;
      double two_x = __dmul_rn(2.0, xi);
      for (int j = 2; j < n; ++j) T[j] = __dsub_rn(__dmul_rn(two_x, T[j - 1]), T[j - 2]);
      for (int k = 0; k < n; ++k) {
        double dot = 0.0;
        for (int j = 1; j < n; ++j) dot = __dadd_rn(dot, __dmul_rn(T[j], Tn[k * n + j]));
        w[d][k] = __ddiv_rn(__dadd_rn(1.0, __dmul_rn(2.0, dot)), (double)n);
      }
    }
    double* out = W2 + p * (int64_t)(n * n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) out[i * n + j] = __dmul_rn(w[0][i], w[1][j]);
  }
}

// M2L operators of one level (fmm.py:286-312): for offset slot s,
// M[a][b] = K(|tn_a - (d h + tn_b)|), tn = nodes2d * (h / 2), a = ix * n + iy.
__global__ void m2l_operators(KParams kp, int n, double h, const double* __restrict__ nodes, uint64_t present,
                              M2LOffsets offs, double* __restrict__ ops) {
  int q = n * n;
  int64_t total = 40LL * q * q;
  double half = h / 2.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int s = (int)(e / ((int64_t)q * q));
    int ab = (int)(e % ((int64_t)q * q));
    int a = ab / q, b = ab % q;
    if (!((present >> s) & 1)) {
      ops[e] = 0.0;
      continue;
    }
    double tx = __dmul_rn(nodes[a / n], half), ty = __dmul_rn(nodes[a % n], half);
    double sx = __dadd_rn(__dmul_rn((double)offs.dx[s], h), __dmul_rn(nodes[b / n], half));
    double sy = __dadd_rn(__dmul_rn((double)offs.dy[s], h), __dmul_rn(nodes[b % n], half));
    ops[e] = kernel_of_r(kp, dist2d(tx, ty, sx, sy));
  }
}

// Full-lattice M2L pair enumeration for one (level, offset), using the same
// rule the M2L kernel uses; flags[t] = 1 if target t has a source.
__global__ void m2l_pair_flags(int64_t G, int dx, int dy, uint8_t* flags) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < G * G; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t s;
    flags[t] = m2l_source(t / G, t % G, dx, dy, G, s) ? 1 : 0;
  }
}

int grid_for(int64_t n) {
  int64_t b = (n + kThreads - 1) / kThreads;
  int64_t cap = (int64_t)num_sms() * 16;
  return (int)std::max<int64_t>(1, std::min(b, cap));
}

template <class T>
int dalloc(T** p, size_t count) {
  HIKF_CHECK_CUDA(cudaMalloc((void**)p, std::max<size_t>(1, count) * sizeof(T)));
  return HIKF_OK;
}

}  // namespace

void tree_free(hikf_tree* t) {
  if (!t) return;
  cudaFree(t->xy);
  cudaFree(t->xy_s);
  cudaFree(t->order);
  cudaFree(t->inv_order);
  cudaFree(t->leaf_of);
  cudaFree(t->leaf_box);
  cudaFree(t->leaf_start);
  cudaFree(t->leaf_count);
  cudaFree(t->box2leaf);
  cudaFree(t->W2s);
  if (t->near) {  // stream-ordered pool allocation (kept reserved across trees)
    cudaDeviceSynchronize();
    cudaFreeAsync(t->near, 0);
  }
  for (int l = 0; l <= kMaxDepth; ++l) {
    cudaFree(t->occ[l]);
    cudaFree(t->occ_flag[l]);
    cudaFree(t->m2l[l]);
    cudaFree(t->shift[l]);
  }
  delete t;
}

static // near[((T * 9 + s) * 64 + c) * 64 + t] = K(x_t, x_c) (kernels.py evaluation, as P2P does it)
__global__ void near_blocks(KParams kp, int64_t G, const int32_t* __restrict__ leaf_box,
                            const int32_t* __restrict__ leaf_start, const int32_t* __restrict__ leaf_count,
                            const int32_t* __restrict__ box2leaf, const double* __restrict__ xy_s,
                            double* __restrict__ near) {
  const int64_t T = blockIdx.x;
  const int s = blockIdx.y;
  const int64_t box = leaf_box[T], bx = box / G, by = box % G;
  const int64_t nx = bx + (s / 3 - 1), ny = by + (s % 3 - 1);
  if (nx < 0 || nx >= G || ny < 0 || ny >= G) return;
  const int32_t S = box2leaf[nx * G + ny];
  if (S < 0) return;
  const int32_t t0 = leaf_start[T], ct = leaf_count[T], s0 = leaf_start[S], cs = leaf_count[S];
  double* blk = near + ((T * 9 + s) * 64) * 64;
  for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) {
    const int t = e & 63, c = e >> 6;
    double v = 0.0;
    if (t < ct && c < cs)
      v = kernel_of_r_near(kp, dist2d(xy_s[2 * (int64_t)(t0 + t)], xy_s[2 * (int64_t)(t0 + t) + 1],
                                      xy_s[2 * (int64_t)(s0 + c)], xy_s[2 * (int64_t)(s0 + c) + 1]));
    blk[e] = v;
  }
}

int build_impl(hikf_tree* t, const double* xy_host, cudaStream_t st) {
  const int64_t m = t->m;
  HIKF_TRY(dalloc(&t->xy, 2 * m));
  HIKF_CHECK_CUDA(cudaMemcpyAsync(t->xy, xy_host, sizeof(double) * 2 * m, cudaMemcpyHostToDevice, st));

  // ---- root box (fmm.py:107-114) ----
  int nb = std::min(grid_for(m), 1024);
  double* part = nullptr;
  HIKF_TRY(dalloc(&part, 4 * (size_t)nb));
  minmax_partial<<<nb, kThreads, 0, st>>>(t->xy, m, part);
  HIKF_CHECK_LAUNCH();
  std::vector<double> hp(4 * (size_t)nb);
  HIKF_CHECK_CUDA(cudaMemcpyAsync(hp.data(), part, sizeof(double) * 4 * nb, cudaMemcpyDeviceToHost, st));
  HIKF_CHECK_CUDA(cudaStreamSynchronize(st));
  cudaFree(part);
  double lo0 = DBL_MAX, lo1 = DBL_MAX, hi0 = -DBL_MAX, hi1 = -DBL_MAX;
  for (int b = 0; b < nb; ++b) {
    lo0 = std::min(lo0, hp[4 * b]);
    lo1 = std::min(lo1, hp[4 * b + 1]);
    hi0 = std::max(hi0, hp[4 * b + 2]);
    hi1 = std::max(hi1, hp[4 * b + 3]);
  }
  double size = std::max(hi0 - lo0, hi1 - lo1);
  if (size == 0.0) size = 1.0;
  size *= 1.0 + 1e-12;
  t->lo[0] = lo0;
  t->lo[1] = lo1;
  t->size = size;

  // ---- depth: smallest uniform depth with max leaf count <= max_leaf (fmm.py:137-150) ----
  int64_t cap_bins = std::max<int64_t>(4096, 8 * m);
  int32_t* hist = nullptr;
  int32_t* dmax = nullptr;
  HIKF_TRY(dalloc(&hist, (size_t)cap_bins));
  HIKF_TRY(dalloc(&dmax, 1));
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
  cub::DeviceReduce::Max(nullptr, cub_bytes, hist, dmax, (int)cap_bins, st);
  HIKF_CHECK_CUDA(cudaMalloc(&cub_tmp, cub_bytes));
  // Depths below d0 fail both tests of the reference loop, so the search starts there
  // (exact): some box holds >= ceil(m / 4^d) points (pigeonhole), and the cap test
  // 4^(d+1) > cap_bins first fires at d_cap.  At cfg4 this is one box-key pass, not eight
  // (the coarse passes serialise on histogram atomics).
  int d_lb = 0, d_cap = 0;
  while (d_lb < kMaxDepth && (m + (1LL << (2 * d_lb)) - 1) / (1LL << (2 * d_lb)) > t->max_leaf) ++d_lb;
  while (d_cap < kMaxDepth && !((4LL << (2 * d_cap)) > cap_bins)) ++d_cap;
  int depth = std::min(d_lb, d_cap);
  for (;;) {
    if (depth >= kMaxDepth) break;
    int64_t G = 1LL << depth;
    int64_t bins = G * G;  // <= cap_bins: deeper depths stop below
    HIKF_CHECK_CUDA(cudaMemsetAsync(hist, 0, sizeof(int32_t) * bins, st));
    box_keys<<<grid_for(m), kThreads, 0, st>>>(t->xy, m, lo0, lo1, size / (double)G, G, nullptr, hist);
    HIKF_CHECK_LAUNCH();
    size_t bytes = cub_bytes;
    cub::DeviceReduce::Max(cub_tmp, bytes, hist, dmax, (int)bins, st);
    int32_t mx = 0;
    HIKF_CHECK_CUDA(cudaMemcpyAsync(&mx, dmax, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    HIKF_CHECK_CUDA(cudaStreamSynchronize(st));
    if (mx <= t->max_leaf) break;
    // 4^(depth+1) > max(4096, 8m): deeper levels would cost more than they save
    if ((4LL << (2 * depth)) > cap_bins) break;
    ++depth;
  }
  cudaFree(cub_tmp);
  cudaFree(dmax);
  cudaFree(hist);
  if (depth > 15) {
    set_error("tree depth %d exceeds the supported 15 levels", depth);
    return HIKF_BAD_ARGUMENT;
  }
  t->depth = depth;
  const int64_t G = 1LL << depth;
  t->G = G;
  const double h = size / (double)G;

  // ---- box keys + stable sort + unique (fmm.py:117-128) ----
  int64_t *keys = nullptr, *keys_sorted = nullptr, *iota = nullptr, *uniq = nullptr;
  int32_t *counts = nullptr, *n_runs = nullptr;
  HIKF_TRY(dalloc(&keys, m));
  HIKF_TRY(dalloc(&keys_sorted, m));
  HIKF_TRY(dalloc(&iota, m));
  HIKF_TRY(dalloc(&t->order, m));
  HIKF_TRY(dalloc(&uniq, m));
  HIKF_TRY(dalloc(&counts, m));
  HIKF_TRY(dalloc(&n_runs, 1));
  box_keys<<<grid_for(m), kThreads, 0, st>>>(t->xy, m, lo0, lo1, h, G, keys, nullptr);
  HIKF_CHECK_LAUNCH();
  iota64<<<grid_for(m), kThreads, 0, st>>>(iota, m);
  HIKF_CHECK_LAUNCH();
  int end_bit = std::max(1, 2 * depth);
  size_t sort_bytes = 0, rle_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, keys, keys_sorted, iota, t->order, (int)m, 0, end_bit, st);
  cub::DeviceRunLengthEncode::Encode(nullptr, rle_bytes, keys_sorted, uniq, counts, n_runs, (int)m, st);
  void* tmp = nullptr;
  HIKF_CHECK_CUDA(cudaMalloc(&tmp, std::max(sort_bytes, rle_bytes)));
  cub::DeviceRadixSort::SortPairs(tmp, sort_bytes, keys, keys_sorted, iota, t->order, (int)m, 0, end_bit, st);
  cub::DeviceRunLengthEncode::Encode(tmp, rle_bytes, keys_sorted, uniq, counts, n_runs, (int)m, st);
  HIKF_CHECK_LAUNCH();
  int32_t nl = 0;
  HIKF_CHECK_CUDA(cudaMemcpyAsync(&nl, n_runs, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  HIKF_CHECK_CUDA(cudaStreamSynchronize(st));
  t->n_leaves = nl;
  std::vector<int64_t> hu(nl);
  std::vector<int32_t> hc(nl);
  HIKF_CHECK_CUDA(cudaMemcpyAsync(hu.data(), uniq, sizeof(int64_t) * nl, cudaMemcpyDeviceToHost, st));
  HIKF_CHECK_CUDA(cudaMemcpyAsync(hc.data(), counts, sizeof(int32_t) * nl, cudaMemcpyDeviceToHost, st));
  HIKF_CHECK_CUDA(cudaStreamSynchronize(st));
  cudaFree(tmp);
  cudaFree(keys);
  cudaFree(keys_sorted);
  cudaFree(iota);
  cudaFree(uniq);
  cudaFree(counts);
  cudaFree(n_runs);

  // leaf tables (host: O(#leaves)), box -> leaf map, per-level occupancy
  t->h_leaf_box.resize(nl);
  t->h_leaf_start.resize(nl);
  t->h_leaf_count.resize(nl);
  std::vector<int32_t> lb(nl), ls(nl), lc(nl), b2l(G * G, -1);
  int64_t run = 0;
  t->max_count = 0;
  for (int32_t r = 0; r < nl; ++r) {
    t->h_leaf_box[r] = hu[r];
    t->h_leaf_start[r] = run;
    t->h_leaf_count[r] = hc[r];
    lb[r] = (int32_t)hu[r];
    ls[r] = (int32_t)run;
    lc[r] = hc[r];
    b2l[hu[r]] = r;
    run += hc[r];
    t->max_count = std::max<int64_t>(t->max_count, hc[r]);
  }
  HIKF_TRY(dalloc(&t->leaf_box, nl));
  HIKF_TRY(dalloc(&t->leaf_start, nl));
  HIKF_TRY(dalloc(&t->leaf_count, nl));
  HIKF_TRY(dalloc(&t->box2leaf, G * G));
  HIKF_CHECK_CUDA(cudaMemcpyAsync(t->leaf_box, lb.data(), sizeof(int32_t) * nl, cudaMemcpyHostToDevice, st));
  HIKF_CHECK_CUDA(cudaMemcpyAsync(t->leaf_start, ls.data(), sizeof(int32_t) * nl, cudaMemcpyHostToDevice, st));
  HIKF_CHECK_CUDA(cudaMemcpyAsync(t->leaf_count, lc.data(), sizeof(int32_t) * nl, cudaMemcpyHostToDevice, st));
  HIKF_CHECK_CUDA(cudaMemcpyAsync(t->box2leaf, b2l.data(), sizeof(int32_t) * G * G, cudaMemcpyHostToDevice, st));

  HIKF_TRY(dalloc(&t->inv_order, m));
  HIKF_TRY(dalloc(&t->leaf_of, m));
  inverse_perm<<<grid_for(m), kThreads, 0, st>>>(t->order, m, t->inv_order);
  HIKF_CHECK_LAUNCH();
  leaf_ranks<<<(unsigned)std::min<int64_t>(nl, 65535), kThreads, 0, st>>>(t->leaf_start, t->leaf_count, nl,
                                                                          t->leaf_of);
  HIKF_CHECK_LAUNCH();
  HIKF_TRY(dalloc(&t->xy_s, 2 * m));
  gather_xy<<<grid_for(m), kThreads, 0, st>>>(t->xy, t->order, m, t->xy_s);
  HIKF_CHECK_LAUNCH();

  // ---- near-field kernel blocks of every (target leaf, neighbour leaf) pair ----
  if (t->max_count <= 64) {
    const size_t bytes = sizeof(double) * (size_t)nl * 9 * 64 * 64;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && bytes <= free_b / 4) {
      // from the stream-ordered pool: a cudaMalloc of the 4.8 GB cfg4 blocks costs ~30 ms of mapping
      // per tree, the pool (release threshold kept at max) maps it once per process
      HIKF_CHECK_CUDA(cudaMallocAsync((void**)&t->near, bytes, st));
      near_blocks<<<dim3((unsigned)nl, 9), kThreads, 0, st>>>(t->kp, G, t->leaf_box, t->leaf_start, t->leaf_count,
                                                               t->box2leaf, t->xy_s, t->near);
      HIKF_CHECK_LAUNCH();
    }
  }

  if (depth < 2) return HIKF_OK;  // near field only (fmm.py:131)

  // ---- per-level occupancy: boxes with >= 1 point below them ----
  std::vector<std::vector<uint8_t>> flags(depth + 1);
  for (int l = 2; l <= depth; ++l) flags[l].assign((size_t)1 << (2 * l), 0);
  for (int32_t r = 0; r < nl; ++r) {
    int64_t bx = hu[r] / G, by = hu[r] % G;
    for (int l = depth; l >= 2; --l) {
      int sh = depth - l;
      flags[l][((bx >> sh) << l) + (by >> sh)] = 1;
    }
  }
  for (int l = 2; l <= depth; ++l) {
    std::vector<int32_t> ids;
    for (size_t b = 0; b < flags[l].size(); ++b)
      if (flags[l][b]) ids.push_back((int32_t)b);
    t->n_occ[l] = (int64_t)ids.size();
    HIKF_TRY(dalloc(&t->occ[l], ids.size()));
    HIKF_TRY(dalloc(&t->occ_flag[l], flags[l].size()));
    HIKF_CHECK_CUDA(cudaMemcpyAsync(t->occ[l], ids.data(), sizeof(int32_t) * ids.size(), cudaMemcpyHostToDevice, st));
    HIKF_CHECK_CUDA(cudaMemcpyAsync(t->occ_flag[l], flags[l].data(), flags[l].size(), cudaMemcpyHostToDevice, st));
    HIKF_CHECK_CUDA(cudaStreamSynchronize(st));  // host vectors go out of scope
  }

  // ---- per-level Chebyshev orders (fmm.py:227-244) ----
  select_orders(t->kp, t->n_cheb, depth, size, t->orders);

  // ---- leaf interpolation weights (fmm.py:246-262) ----
  const int nleaf = t->orders[depth];
  {
    std::vector<double> tn = cheb_node_table(nleaf);
    double* dTn = nullptr;
    HIKF_TRY(dalloc(&dTn, tn.size()));
    HIKF_CHECK_CUDA(cudaMemcpyAsync(dTn, tn.data(), sizeof(double) * tn.size(), cudaMemcpyHostToDevice, st));
    HIKF_TRY(dalloc(&t->W2s, (size_t)m * nleaf * nleaf));
    interp_weights<<<grid_for(m), kThreads, 0, st>>>(t->xy_s, m, lo0, lo1, h, G, nleaf, dTn, t->W2s);
    HIKF_CHECK_LAUNCH();
    HIKF_CHECK_CUDA(cudaStreamSynchronize(st));
    cudaFree(dTn);
  }

  // ---- shift operators (fmm.py:264-278) ----
  for (int l = 2; l < depth; ++l) {
    int np_ = t->orders[l], nc = t->orders[l + 1];
    size_t one = (size_t)nc * nc * np_ * np_;
    std::vector<double> all(4 * one);
    for (int c = 0; c < 4; ++c) {
      std::vector<double> op = shift_operator(np_, nc, c >> 1, c & 1);
      std::copy(op.begin(), op.end(), all.begin() + c * one);
    }
    HIKF_TRY(dalloc(&t->shift[l], all.size()));
    HIKF_CHECK_CUDA(cudaMemcpyAsync(t->shift[l], all.data(), sizeof(double) * all.size(), cudaMemcpyHostToDevice, st));
    HIKF_CHECK_CUDA(cudaStreamSynchronize(st));
  }

  // ---- M2L operators (fmm.py:286-312) ----
  M2LOffsets offs;
  for (int l = 2; l <= depth; ++l) {
    int n = t->orders[l];
    int64_t Gl = 1LL << l;
    uint64_t present = 0;
    for (int s = 0; s < 40; ++s) {
      bool any_x = false, any_y = false;
      for (int64_t i = 0; i < Gl; ++i) {
        int64_t jx = i + offs.dx[s], jy = i + offs.dy[s];
        any_x |= jx >= 0 && jx < Gl && std::llabs((jx >> 1) - (i >> 1)) <= 1;
        any_y |= jy >= 0 && jy < Gl && std::llabs((jy >> 1) - (i >> 1)) <= 1;
      }
      if (any_x && any_y) present |= 1ULL << s;
    }
    t->m2l_present[l] = present;
    std::vector<double> nodes = cheb_nodes(n);
    double* dn = nullptr;
    HIKF_TRY(dalloc(&dn, nodes.size()));
    HIKF_CHECK_CUDA(cudaMemcpyAsync(dn, nodes.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
    size_t total = 40 * (size_t)n * n * n * n;
    HIKF_TRY(dalloc(&t->m2l[l], total));
    m2l_operators<<<grid_for((int64_t)total), kThreads, 0, st>>>(t->kp, n, size / (double)Gl, dn, present, offs,
                                                                   t->m2l[l]);
    HIKF_CHECK_LAUNCH();
    HIKF_CHECK_CUDA(cudaStreamSynchronize(st));
    cudaFree(dn);
  }
  return HIKF_OK;
}

int tree_build(const double* xy_host, int64_t m, const hikf_kernel& k, int n_cheb, int64_t max_leaf,
               cudaStream_t stream, hikf_tree** out) {
  if (!xy_host || m < 1 || !out) {
    set_error("need at least one point");
    return HIKF_BAD_ARGUMENT;
  }
  if (n_cheb < 2 || n_cheb > 12) {
    set_error("n_cheb must lie in [2, 12]");
    return HIKF_BAD_ARGUMENT;
  }
  if (max_leaf < 1) {
    set_error("max_leaf_points must be >= 1");
    return HIKF_BAD_ARGUMENT;
  }
  if (m > (int64_t)INT32_MAX) {
    set_error("at most 2^31-1 points are supported");
    return HIKF_BAD_ARGUMENT;
  }
  for (int64_t i = 0; i < 2 * m; ++i)
    if (!std::isfinite(xy_host[i])) {
      set_error("coordinates must be finite");
      return HIKF_BAD_ARGUMENT;
    }
  hikf_tree* t = new hikf_tree();
  t->m = m;
  t->spec = k;
  t->kp = make_kparams(k);
  t->n_cheb = n_cheb;
  t->max_leaf = max_leaf;
  int s = build_impl(t, xy_host, stream);
  if (s != HIKF_OK) {
    cudaStreamSynchronize(stream);
    tree_free(t);
    return s;
  }
  HIKF_CHECK_CUDA(cudaStreamSynchronize(stream));
  *out = t;
  return HIKF_OK;
}

int tree_export_m2l_pairs(const hikf_tree* t, int lev, int dx, int dy, std::vector<int64_t>& tgt,
                          std::vector<int64_t>& src) {
  tgt.clear();
  src.clear();
  if (lev < 2 || lev > t->depth) return HIKF_OK;
  int64_t G = 1LL << lev;
  uint8_t* d = nullptr;
  HIKF_TRY(dalloc(&d, G * G));
  m2l_pair_flags<<<grid_for(G * G), kThreads>>>(G, dx, dy, d);
  HIKF_CHECK_LAUNCH();
  std::vector<uint8_t> f(G * G);
  HIKF_CHECK_CUDA(cudaMemcpy(f.data(), d, G * G, cudaMemcpyDeviceToHost));
  cudaFree(d);
  for (int64_t i = 0; i < G * G; ++i)
    if (f[i]) {
      tgt.push_back(i);
      src.push_back(i + dx * G + dy);
    }
  return HIKF_OK;
}

}  // namespace hikf

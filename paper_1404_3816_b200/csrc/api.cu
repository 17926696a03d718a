// C-ABI entry points of libhikf_b200.so (declared in include/hikf_b200.h).
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "dense.h"
#include "fmm3d.h"
#include "kf.h"
#include "host_ops.h"
#include "dgemm.cuh"
#include "prof.h"
#include "rays.h"
#include "tree.h"
#include "update.h"

namespace hikf {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

const std::string& last_error() { return g_last_error; }

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

KParams make_kparams(const hikf_kernel& k) {
  KParams p;
  p.family = k.family;
  p.variance = k.variance;
  p.length = k.length_scale;
  p.inv_length = 1.0 / k.length_scale;
  p.power = k.power;
  p.log_amp = k.log_amplitude;
  p.pmode = 0;
  if (k.power == 1.0) p.pmode = 1;
  if (k.power == 2.0) p.pmode = 2;
  if (k.power == 0.5) p.pmode = 3;
  return p;
}

namespace {

constexpr int kT = 256;

// dense H^T (m x n) from CSR H (n x m); Ht must be zeroed first
__global__ void scatter_transpose(int64_t n, const int32_t* __restrict__ ip, const int32_t* __restrict__ ix,
                                  const double* __restrict__ val, double* __restrict__ Ht) {
  int64_t r = blockIdx.x;
  if (r >= n) return;
  for (int64_t e = ip[r] + threadIdx.x; e < ip[r + 1]; e += blockDim.x) Ht[(int64_t)ix[e] * n + r] = val[e];
}

// X = H C (n x n), one CTA per row of H.  Each thread owns 4 adjacent columns
// (one 32-byte load per nonzero) and accumulates them in CSR order, so 4
// independent FMA chains and the row's gathers stay in flight.
__global__ void spmm_rows(int64_t n, const int32_t* __restrict__ ip, const int32_t* __restrict__ ix,
                          const double* __restrict__ val, const double* __restrict__ C, double* __restrict__ X) {
  const int64_t r = blockIdx.x;
  const int32_t b = ip[r], e1 = ip[r + 1];
  const bool vec = (n % 4) == 0 && (((uintptr_t)C) & 31) == 0;
  for (int64_t j0 = 4 * (int64_t)threadIdx.x; j0 < n; j0 += 4 * (int64_t)blockDim.x) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    if (vec) {
      // 8 rows of C_Q in flight per thread (loads first, then the sums in entry order)
      int32_t e = b;
      for (; e + 8 <= e1; e += 8) {
        double v[8];
        double2 a[8], c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          v[u] = val[e + u];
          const double* row = C + (int64_t)ix[e + u] * n + j0;
          a[u] = __ldg(reinterpret_cast<const double2*>(row));
          c[u] = __ldg(reinterpret_cast<const double2*>(row + 2));
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          s0 += v[u] * a[u].x;
          s1 += v[u] * a[u].y;
          s2 += v[u] * c[u].x;
          s3 += v[u] * c[u].y;
        }
      }
      for (; e < e1; ++e) {
        const double v = val[e];
        const double* row = C + (int64_t)ix[e] * n + j0;
        const double2 a = __ldg(reinterpret_cast<const double2*>(row));
        const double2 c = __ldg(reinterpret_cast<const double2*>(row + 2));
        s0 += v * a.x;
        s1 += v * a.y;
        s2 += v * c.x;
        s3 += v * c.y;
      }
    } else {
      for (int32_t e = b; e < e1; ++e) {
        const double v = val[e];
        const double* row = C + (int64_t)ix[e] * n;
        s0 += v * row[j0];
        if (j0 + 1 < n) s1 += v * row[j0 + 1];
        if (j0 + 2 < n) s2 += v * row[j0 + 2];
        if (j0 + 3 < n) s3 += v * row[j0 + 3];
      }
    }
    X[r * n + j0] = s0;
    if (j0 + 1 < n) X[r * n + j0 + 1] = s1;
    if (j0 + 2 < n) X[r * n + j0 + 2] = s2;
    if (j0 + 3 < n) X[r * n + j0 + 3] = s3;
  }
}

__global__ void symmetrize(const double* __restrict__ X, int64_t n, double* __restrict__ Y) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e / n, j = e % n;
    Y[e] = 0.5 * (X[e] + X[j * n + i]);
  }
}

__global__ void fill(double* x, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) x[i] = v;
}

__global__ void scale_copy(const double* __restrict__ x, int64_t n, double a, double* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = a * x[i];
}

int grid_for(int64_t n) {
  int64_t b = (n + kT - 1) / kT;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)num_sms() * 32));
}

int matmat_csrT(hikf_tree* t, int64_t n, const int32_t* ip, const int32_t* ix, const double* val, double* U,
                cudaStream_t st) {
  return fmm_matmat_csrT(t, n, ip, ix, val, U, st);
}

}  // namespace
}  // namespace hikf

using namespace hikf;

static cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Keep stream-ordered allocations cached in the device's default pool between
// calls (the default release threshold of 0 would unmap and remap the FMM
// workspace at every synchronisation).
static void keep_pool() {
  static bool done = false;
  if (done) return;
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done = true;
}

extern "C" {

int hikf_abi_version(void) { return 1; }

int hikf_last_error(char* buf, size_t len) {
  if (!buf || len == 0) return HIKF_BAD_ARGUMENT;
  std::strncpy(buf, g_last_error.c_str(), len - 1);
  buf[len - 1] = '\0';
  return HIKF_OK;
}

int hikf_tree_create(const double* xy_host, int64_t m, const hikf_kernel* kernel, int32_t n_cheb, int64_t max_leaf,
                     void* stream, hikf_tree** out) {
  if (!kernel || !out) {
    set_error("null argument");
    return HIKF_BAD_ARGUMENT;
  }
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0) {
    set_error("no CUDA device: the HiKF B200 path has no CPU fallback");
    return HIKF_NO_DEVICE;
  }
  keep_pool();
  return tree_build(xy_host, m, *kernel, n_cheb, max_leaf, as_stream(stream), out);
}

int hikf_tree_destroy(hikf_tree* tree) {
  tree_free(tree);
  return HIKF_OK;
}

int hikf_release_cached_memory(void) {
  int dev = 0;
  cudaMemPool_t pool;
  HIKF_CHECK_CUDA(cudaGetDevice(&dev));
  HIKF_CHECK_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  HIKF_CHECK_CUDA(cudaDeviceSynchronize());
  HIKF_CHECK_CUDA(cudaMemPoolTrimTo(pool, 0));
  return HIKF_OK;
}

int hikf_tree_info(const hikf_tree* t, int64_t* m, int32_t* depth, int32_t* orders21, double* root_lo2,
                   double* root_size, int64_t* n_leaves, int64_t* n_near_pairs) {
  if (!t) return HIKF_BAD_ARGUMENT;
  if (m) *m = t->m;
  if (depth) *depth = t->depth;
  if (orders21)
    for (int l = 0; l <= kMaxDepth; ++l) orders21[l] = t->orders[l];
  if (root_lo2) {
    root_lo2[0] = t->lo[0];
    root_lo2[1] = t->lo[1];
  }
  if (root_size) *root_size = t->size;
  if (n_leaves) *n_leaves = t->n_leaves;
  if (n_near_pairs) {
    int64_t G = t->G, cnt = 0;
    std::vector<int32_t> b2l(G * G, -1);
    for (int64_t r = 0; r < t->n_leaves; ++r) b2l[t->h_leaf_box[r]] = (int32_t)r;
    for (int64_t r = 0; r < t->n_leaves; ++r) {
      int64_t bx = t->h_leaf_box[r] / G, by = t->h_leaf_box[r] % G;
      for (int ox = -1; ox <= 1; ++ox)
        for (int oy = -1; oy <= 1; ++oy) {
          int64_t nx = bx + ox, ny = by + oy;
          if (nx >= 0 && nx < G && ny >= 0 && ny < G && b2l[nx * G + ny] >= 0) ++cnt;
        }
    }
    *n_near_pairs = cnt;
  }
  return HIKF_OK;
}

int hikf_tree_export(const hikf_tree* t, int64_t* order, int64_t* leaf_ids, int64_t* leaf_starts, int64_t* leaf_counts,
                     int64_t* near_t, int64_t* near_s) {
  if (!t) return HIKF_BAD_ARGUMENT;
  if (order) HIKF_CHECK_CUDA(cudaMemcpy(order, t->order, sizeof(int64_t) * t->m, cudaMemcpyDeviceToHost));
  for (int64_t r = 0; r < t->n_leaves; ++r) {
    if (leaf_ids) leaf_ids[r] = t->h_leaf_box[r];
    if (leaf_starts) leaf_starts[r] = t->h_leaf_start[r];
    if (leaf_counts) leaf_counts[r] = t->h_leaf_count[r];
  }
  if (near_t || near_s) {
    // fmm.py:170-179: for each offset (ox outer, oy inner), every occupied leaf in
    // rank order whose neighbour box is occupied -- the same rule P2P uses
    int64_t G = t->G, p = 0;
    std::vector<int32_t> b2l(G * G, -1);
    HIKF_CHECK_CUDA(cudaMemcpy(b2l.data(), t->box2leaf, sizeof(int32_t) * G * G, cudaMemcpyDeviceToHost));
    for (int ox = -1; ox <= 1; ++ox)
      for (int oy = -1; oy <= 1; ++oy)
        for (int64_t r = 0; r < t->n_leaves; ++r) {
          int64_t bx = t->h_leaf_box[r] / G + ox, by = t->h_leaf_box[r] % G + oy;
          if (bx < 0 || bx >= G || by < 0 || by >= G) continue;
          int32_t s = b2l[bx * G + by];
          if (s < 0) continue;
          if (near_t) near_t[p] = r;
          if (near_s) near_s[p] = s;
          ++p;
        }
  }
  return HIKF_OK;
}

int hikf_tree_export_op(const hikf_tree* t, int32_t which, int32_t lev, int32_t dx, int32_t dy, double* out) {
  if (!t || !out) return HIKF_BAD_ARGUMENT;
  if (t->depth < 2) {
    set_error("tree has no far field (depth < 2)");
    return HIKF_BAD_ARGUMENT;
  }
  if (which == 0) {
    if (lev < 2 || lev > t->depth) return HIKF_BAD_ARGUMENT;
    M2LOffsets offs;
    int s = -1;
    for (int i = 0; i < 40; ++i)
      if (offs.dx[i] == dx && offs.dy[i] == dy) s = i;
    if (s < 0 || !((t->m2l_present[lev] >> s) & 1)) {
      set_error("no M2L operator for offset (%d, %d) at level %d", dx, dy, lev);
      return HIKF_BAD_ARGUMENT;
    }
    int64_t q = (int64_t)t->orders[lev] * t->orders[lev];
    HIKF_CHECK_CUDA(cudaMemcpy(out, t->m2l[lev] + s * q * q, sizeof(double) * q * q, cudaMemcpyDeviceToHost));
    return HIKF_OK;
  }
  if (which == 1) {
    if (lev < 2 || lev >= t->depth || dx < 0 || dx > 1 || dy < 0 || dy > 1) return HIKF_BAD_ARGUMENT;
    int64_t qp = (int64_t)t->orders[lev] * t->orders[lev], qc = (int64_t)t->orders[lev + 1] * t->orders[lev + 1];
    HIKF_CHECK_CUDA(cudaMemcpy(out, t->shift[lev] + (dx * 2 + dy) * qp * qc, sizeof(double) * qp * qc,
                               cudaMemcpyDeviceToHost));
    return HIKF_OK;
  }
  if (which == 2) {
    int64_t q = (int64_t)t->orders[t->depth] * t->orders[t->depth];
    std::vector<double> w(t->m * q);
    std::vector<int64_t> ord(t->m);
    HIKF_CHECK_CUDA(cudaMemcpy(w.data(), t->W2s, sizeof(double) * w.size(), cudaMemcpyDeviceToHost));
    HIKF_CHECK_CUDA(cudaMemcpy(ord.data(), t->order, sizeof(int64_t) * t->m, cudaMemcpyDeviceToHost));
    for (int64_t p = 0; p < t->m; ++p) std::memcpy(out + ord[p] * q, &w[p * q], sizeof(double) * q);
    return HIKF_OK;
  }
  return HIKF_BAD_ARGUMENT;
}

int hikf_tree_m2l_pairs(const hikf_tree* t, int32_t lev, int32_t dx, int32_t dy, int64_t* tgt, int64_t* src,
                        int64_t* count) {
  if (!t || !count) return HIKF_BAD_ARGUMENT;
  std::vector<int64_t> a, b;
  HIKF_TRY(tree_export_m2l_pairs(t, lev, dx, dy, a, b));
  if (tgt && src) {
    if (*count < (int64_t)a.size()) return HIKF_BAD_ARGUMENT;
    std::memcpy(tgt, a.data(), sizeof(int64_t) * a.size());
    std::memcpy(src, b.data(), sizeof(int64_t) * b.size());
  }
  *count = (int64_t)a.size();
  return HIKF_OK;
}

int hikf_tree_matmat(hikf_tree* t, const double* V, int64_t ldv, int64_t k, double* U, int64_t ldu, void* stream) {
  if (!t || (k > 0 && (!V || !U)) || k < 0 || ldv < k || ldu < k) {
    set_error("bad matmat arguments");
    return HIKF_BAD_ARGUMENT;
  }
  return fmm_matmat(t, V, ldv, k, U, ldu, as_stream(stream));
}

int hikf_tree_matmat_csrT(hikf_tree* t, int64_t n, const int32_t* ip, const int32_t* ix, const double* val, double* U,
                          void* stream) {
  if (!t || n < 0 || (n > 0 && (!ip || !U))) {
    set_error("bad matmat_csrT arguments");
    return HIKF_BAD_ARGUMENT;
  }
  return matmat_csrT(t, n, ip, ix, val, U, as_stream(stream));
}

int hikf_precompute(hikf_tree* t, int64_t n, const int32_t* ip, const int32_t* ix, const double* val, double* CQ,
                    double* HCQ, double* dQ, void* stream) {
  if (!t || n < 0) {
    set_error("bad precompute arguments");
    return HIKF_BAD_ARGUMENT;
  }
  cudaStream_t st = as_stream(stream);
  HIKF_TRY(matmat_csrT(t, n, ip, ix, val, CQ, st));
  if (n > 0) {
    double* X = nullptr;
    HIKF_CHECK_CUDA(cudaMallocAsync((void**)&X, sizeof(double) * n * n, st));
    spmm_rows<<<(unsigned)n, kT, 0, st>>>(n, ip, ix, val, CQ, X);
    HIKF_CHECK_LAUNCH();
    symmetrize<<<grid_for(n * n), kT, 0, st>>>(X, n, HCQ);
    HIKF_CHECK_LAUNCH();
    cudaFreeAsync(X, st);
  }
  double k0 = t->spec.family == HIKF_LOGARITHM ? 0.0 : t->spec.variance;  // value_at_zero (kernels.py:91-95)
  fill<<<grid_for(t->m), kT, 0, st>>>(dQ, t->m, k0);
  HIKF_CHECK_LAUNCH();
  return HIKF_OK;
}

// H[:, r0:r1] C_Q_local (n x n), C_Q_local = rows r0..r1 of C_Q
__global__ void spmm_cols_window(int64_t n, int64_t r0, int64_t r1, const int32_t* __restrict__ ip,
                                 const int32_t* __restrict__ ix, const double* __restrict__ val,
                                 const double* __restrict__ C, double* __restrict__ X) {
  const int64_t r = blockIdx.x;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    double s = 0.0;
    for (int64_t e = ip[r]; e < ip[r + 1]; ++e) {
      const int64_t c = ix[e];
      if (c >= r0 && c < r1) s += val[e] * C[(c - r0) * n + j];
    }
    X[r * n + j] = s;
  }
}

int hikf_precompute_rows(hikf_tree* t, int64_t n, const int32_t* ip, const int32_t* ix, const double* val, int64_t r0,
                         int64_t r1, double* CQ_rows, double* HCQ_partial, double* dQ_rows, void* stream) {
  if (!t || n < 0 || r0 < 0 || r1 < r0 || r1 > t->m) {
    set_error("bad precompute_rows arguments (need 0 <= r0 <= r1 <= m)");
    return HIKF_BAD_ARGUMENT;
  }
  cudaStream_t st = as_stream(stream);
  if (r1 > r0) HIKF_TRY(fmm_matmat_csrT(t, n, ip, ix, val, CQ_rows, st, r0, r1));
  if (n > 0) {
    spmm_cols_window<<<(unsigned)n, kT, 0, st>>>(n, r0, r1, ip, ix, val, CQ_rows, HCQ_partial);
    HIKF_CHECK_LAUNCH();
  }
  double k0 = t->spec.family == HIKF_LOGARITHM ? 0.0 : t->spec.variance;
  if (r1 > r0) {
    fill<<<grid_for(r1 - r0), kT, 0, st>>>(dQ_rows, r1 - r0, k0);
    HIKF_CHECK_LAUNCH();
  }
  return HIKF_OK;
}

int hikf_leaf_partition(const hikf_tree* t, int32_t world, int32_t rank, int64_t* out4) {
  if (!t || !out4 || world < 1 || rank < 0 || rank >= world) {
    set_error("bad leaf_partition arguments (need 0 <= rank < world)");
    return HIKF_BAD_ARGUMENT;
  }
  // contiguous leaves, cut where the running point count passes rank * m / world
  auto cut = [&](int64_t r) -> int64_t {
    if (r <= 0) return 0;
    if (r >= world) return t->n_leaves;
    const int64_t target = (t->m * r + world / 2) / world;
    int64_t lo = 0, hi = t->n_leaves;  // first leaf whose start >= target
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (t->h_leaf_start[mid] < target) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  LeafWindow w;
  HIKF_TRY(leaf_window(t, cut(rank), cut(rank + 1), &w));
  out4[0] = w.leaf0;
  out4[1] = w.leaf1;
  out4[2] = w.s0;
  out4[3] = w.s1;
  return HIKF_OK;
}

// HC_Q partial over a leaf shard: X[r][j] = sum_{e in row r, sorted position p of
// column ix[e] in [s0, s1)} val[e] C[p - s0][j]
__global__ void spmm_cols_sorted(int64_t n, int64_t s0, int64_t s1, const int32_t* __restrict__ ip,
                                 const int32_t* __restrict__ ix, const double* __restrict__ val,
                                 const int32_t* __restrict__ inv_order, const double* __restrict__ C,
                                 double* __restrict__ X) {
  const int64_t r = blockIdx.x;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    double s = 0.0;
    for (int64_t e = ip[r]; e < ip[r + 1]; ++e) {
      const int64_t p = inv_order[ix[e]];
      if (p >= s0 && p < s1) s += val[e] * C[(p - s0) * n + j];
    }
    X[r * n + j] = s;
  }
}

int hikf_precompute_leaves(hikf_tree* t, int64_t n, const int32_t* ip, const int32_t* ix, const double* val,
                           int64_t leaf0, int64_t leaf1, double* CQ_rows, double* HCQ_partial, double* dQ_rows,
                           void* stream) {
  if (!t || n < 0) {
    set_error("bad precompute_leaves arguments");
    return HIKF_BAD_ARGUMENT;
  }
  LeafWindow w;
  HIKF_TRY(leaf_window(t, leaf0, leaf1, &w));
  cudaStream_t st = as_stream(stream);
  if (w.s1 > w.s0) HIKF_TRY(fmm_matmat_csrT(t, n, ip, ix, val, CQ_rows, st, 0, -1, &w));
  if (n > 0) {
    spmm_cols_sorted<<<(unsigned)n, kT, 0, st>>>(n, w.s0, w.s1, ip, ix, val, t->inv_order, CQ_rows, HCQ_partial);
    HIKF_CHECK_LAUNCH();
  }
  double k0 = t->spec.family == HIKF_LOGARITHM ? 0.0 : t->spec.variance;
  if (w.s1 > w.s0) {
    fill<<<grid_for(w.s1 - w.s0), kT, 0, st>>>(dQ_rows, w.s1 - w.s0, k0);
    HIKF_CHECK_LAUNCH();
  }
  return HIKF_OK;
}

int hikf_precompute_dense(const double* xy_host, int64_t m, const hikf_kernel* kernel, int64_t n, const int32_t* ip,
                          const int32_t* ix, const double* val, double* CQ, double* HCQ, double* dQ, void* stream) {
  if (!xy_host || !kernel || m < 1 || n < 0) {
    set_error("bad dense precompute arguments");
    return HIKF_BAD_ARGUMENT;
  }
  if (kernel->family != HIKF_GAUSSIAN && kernel->family != HIKF_EXPONENTIAL && kernel->family != HIKF_LOGARITHM) {
    set_error("unknown kernel family %d", kernel->family);
    return HIKF_BAD_ARGUMENT;
  }
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0) {
    set_error("no CUDA device: the HiKF B200 path has no CPU fallback");
    return HIKF_NO_DEVICE;
  }
  keep_pool();
  cudaStream_t st = as_stream(stream);
  double* xy = nullptr;
  HIKF_CHECK_CUDA(cudaMallocAsync((void**)&xy, sizeof(double) * 2 * m, st));
  HIKF_CHECK_CUDA(cudaMemcpyAsync(xy, xy_host, sizeof(double) * 2 * m, cudaMemcpyHostToDevice, st));
  const KParams kp = make_kparams(*kernel);
  int s = dense_cq(m, n, xy, ip, ix, val, kp, CQ, st);
  if (s == HIKF_OK && n > 0) {
    double* X = nullptr;
    HIKF_CHECK_CUDA(cudaMallocAsync((void**)&X, sizeof(double) * n * n, st));
    spmm_rows<<<(unsigned)n, kT, 0, st>>>(n, ip, ix, val, CQ, X);
    HIKF_CHECK_LAUNCH();
    symmetrize<<<grid_for(n * n), kT, 0, st>>>(X, n, HCQ);
    HIKF_CHECK_LAUNCH();
    cudaFreeAsync(X, st);
  }
  // diag(Q) = K(0) = value_at_zero (kernels.py:91-95): the dense Gram's diagonal
  fill<<<grid_for(m), kT, 0, st>>>(dQ, m, kernel->family == HIKF_LOGARITHM ? 0.0 : kernel->variance);
  HIKF_CHECK_LAUNCH();
  cudaFreeAsync(xy, st);
  return s;
}

int hikf_init_state(int64_t m, int64_t n, const int32_t* ip, const int32_t* ix, const double* val, double alpha,
                    double* C_out, double* var_out, double* HC_out, void* stream) {
  if (m < 1 || n < 0) return HIKF_BAD_ARGUMENT;
  cudaStream_t st = as_stream(stream);
  fill<<<grid_for(m), kT, 0, st>>>(var_out, m, alpha);
  HIKF_CHECK_LAUNCH();
  if (n == 0) return HIKF_OK;
  // C = alpha H^T (dense), HC = alpha (H H^T)  (filters.py:118-126)
  if (alpha == 0.0) {  // the BASELINE configs: 0 * H^T and 0 * H H^T are zeros (H >= 0)
    HIKF_CHECK_CUDA(cudaMemsetAsync(C_out, 0, sizeof(double) * m * n, st));
    HIKF_CHECK_CUDA(cudaMemsetAsync(HC_out, 0, sizeof(double) * n * n, st));
    return HIKF_OK;
  }
  double* Ht = nullptr;
  double* X = nullptr;
  HIKF_CHECK_CUDA(cudaMallocAsync((void**)&Ht, sizeof(double) * m * n, st));
  HIKF_CHECK_CUDA(cudaMallocAsync((void**)&X, sizeof(double) * n * n, st));
  HIKF_CHECK_CUDA(cudaMemsetAsync(Ht, 0, sizeof(double) * m * n, st));
  scatter_transpose<<<(unsigned)n, kT, 0, st>>>(n, ip, ix, val, Ht);
  HIKF_CHECK_LAUNCH();
  spmm_rows<<<(unsigned)n, kT, 0, st>>>(n, ip, ix, val, Ht, X);
  HIKF_CHECK_LAUNCH();
  scale_copy<<<grid_for(m * n), kT, 0, st>>>(Ht, m * n, alpha, C_out);
  HIKF_CHECK_LAUNCH();
  scale_copy<<<grid_for(n * n), kT, 0, st>>>(X, n * n, alpha, HC_out);
  HIKF_CHECK_LAUNCH();
  cudaFreeAsync(Ht, st);
  cudaFreeAsync(X, st);
  return HIKF_OK;
}

int hikf_predict(int64_t m, int64_t n, const double* C, const double* var, const double* HC, const double* CQ,
                 const double* dQ, const double* HCQ, double* Co, double* varo, double* HCo, void* stream) {
  if (m < 0 || n < 0) return HIKF_BAD_ARGUMENT;
  return predict(m, n, C, var, HC, CQ, dQ, HCQ, Co, varo, HCo, as_stream(stream));
}

size_t hikf_update_workspace_bytes(int64_t m, int64_t n) { return update_workspace_bytes(m, n); }

int hikf_update(int64_t m, int64_t n, const double* mean, const double* C, const double* var, const double* HC,
                const double* CQ, const double* dQ, const double* HCQ, const int32_t* ip, const int32_t* ix,
                const double* val, double r, const double* z, double* mean_out, double* C_out, double* var_out,
                double* HC_out, void* workspace, size_t workspace_bytes, double* min_var_out, void* stream) {
  return hikf_update_chained(m, n, mean, C, var, HC, CQ, dQ, HCQ, ip, ix, val, r, z, mean_out, C_out, var_out, HC_out,
                             workspace, workspace_bytes, min_var_out, 0, nullptr, stream);
}

int hikf_update_chained(int64_t m, int64_t n, const double* mean, const double* C, const double* var,
                        const double* HC, const double* CQ, const double* dQ, const double* HCQ, const int32_t* ip,
                        const int32_t* ix, const double* val, double r, const double* z, double* mean_out,
                        double* C_out, double* var_out, double* HC_out, void* workspace, size_t workspace_bytes,
                        double* min_var_out, int32_t chain, double* mean_host, void* stream) {
  if (m < 1 || n < 1 || !mean || !C || !var || !HC || !ip || !z || !mean_out || !C_out || !var_out || !HC_out) {
    set_error("bad update arguments");
    return HIKF_BAD_ARGUMENT;
  }
  if (CQ && (!dQ || !HCQ)) {
    set_error("fused predict needs C_Q, diag_Q and HC_Q");
    return HIKF_BAD_ARGUMENT;
  }
  UpdateArgs a;
  a.m = m;
  a.n = n;
  a.mean = mean;
  a.C = C;
  a.var = var;
  a.HC = HC;
  a.CQ = CQ;
  a.dQ = dQ;
  a.HCQ = HCQ;
  a.ip = ip;
  a.ix = ix;
  a.val = val;
  a.r = r;
  a.z = z;
  a.mean_out = mean_out;
  a.C_out = C_out;
  a.var_out = var_out;
  a.HC_out = HC_out;
  a.workspace = workspace;
  a.workspace_bytes = workspace_bytes;
  a.chain = (chain & 1) != 0;
  a.chain_in = (chain & 2) != 0;
  a.mean_host = mean_host;
  if (chain & 4) {  // deferred: min_var_out = pinned host status[4], filled on the stream
    if (!min_var_out) {
      set_error("deferred update (chain bit 2) needs a pinned host status[4] in min_var_out");
      return HIKF_BAD_ARGUMENT;
    }
    a.status_host = min_var_out;
  }
  UpdateResult res;
  int s = update(a, as_stream(stream), &res);
  if (min_var_out && !(chain & 4)) *min_var_out = res.min_var;
  return s;
}

size_t hikf_update_factored_workspace_bytes(int64_t m, int64_t n) { return update_factored_workspace_bytes(m, n); }

int hikf_update_factored(int64_t m, int64_t n, const double* mean, const double* N, const double* var,
                         const double* HC, const double* CQ, const double* dQ, const double* HCQ, int32_t predict,
                         const int32_t* ip, const int32_t* ix, const double* val, double r, const double* z,
                         double* mean_out, double* N_out, double* var_out, double* HC_out, void* workspace,
                         size_t workspace_bytes, double* min_var_out, double* mean_host, double alpha0,
                         const double* A, double* A_out, const int32_t* ht_indptr, const int32_t* ht_indices,
                         const double* ht_data, void* stream) {
  if (m < 1 || n < 1 || !mean || !N || !var || !HC || !CQ || !ip || !z || !mean_out || !N_out || !var_out ||
      !HC_out || N == N_out) {
    set_error("bad factored update arguments");
    return HIKF_BAD_ARGUMENT;
  }
  if (predict && (!dQ || !HCQ)) {
    set_error("fused predict needs diag_Q and HC_Q");
    return HIKF_BAD_ARGUMENT;
  }
  UpdateArgs a;
  a.m = m;
  a.n = n;
  a.mean = mean;
  a.var = var;
  a.HC = HC;
  a.CQ = CQ;
  a.dQ = predict ? dQ : nullptr;
  a.HCQ = predict ? HCQ : nullptr;
  a.ip = ip;
  a.ix = ix;
  a.val = val;
  a.r = r;
  a.z = z;
  a.mean_out = mean_out;
  a.var_out = var_out;
  a.HC_out = HC_out;
  a.workspace = workspace;
  a.workspace_bytes = workspace_bytes;
  a.mean_host = mean_host;
  a.factored = true;
  a.predict_in = predict != 0;
  a.Nin = N;
  a.Nout = N_out;
  if (alpha0 != 0.0) {
    if (!A || !A_out || !ht_indptr || !ht_indices || !ht_data) {
      set_error("factored update with alpha0 != 0 needs A (in / out) and H^T (CSR)");
      return HIKF_BAD_ARGUMENT;
    }
    a.alpha0 = alpha0;
    a.Ain = A;
    a.Aout = A_out;
    a.ht_ip = ht_indptr;
    a.ht_ix = ht_indices;
    a.ht_val = ht_data;
  }
  UpdateResult res;
  int s = update(a, as_stream(stream), &res);
  if (min_var_out) *min_var_out = res.min_var;
  return s;
}

int hikf_csr_spmm_add(int64_t rows, int64_t k, const int32_t* indptr, const int32_t* indices, const double* data,
                      const double* X, double alpha, double* Y, void* stream) {
  if (rows < 0 || k < 0 || (rows > 0 && (!indptr || !X || !Y))) {
    set_error("bad csr_spmm_add arguments");
    return HIKF_BAD_ARGUMENT;
  }
  return csr_spmm_add(rows, k, indptr, indices, data, X, alpha, Y, as_stream(stream));
}

int hikf_update_rows(int64_t m_local, int64_t n, const double* mean, const double* C, const double* var,
                     const double* HC, const double* CQ, const double* dQ, const double* HCQ, const double* Hmean,
                     double r, const double* z, double* mean_out, double* C_out, double* var_out, double* HC_out,
                     void* workspace, size_t workspace_bytes, double* minmax_out, int32_t chain, void* stream) {
  if (m_local < 1 || n < 1 || !mean || !C || !var || !HC || !Hmean || !z || !mean_out || !C_out || !var_out ||
      !HC_out) {
    set_error("bad update_rows arguments");
    return HIKF_BAD_ARGUMENT;
  }
  if (CQ && (!dQ || !HCQ)) {
    set_error("fused predict needs C_Q, diag_Q and HC_Q");
    return HIKF_BAD_ARGUMENT;
  }
  UpdateArgs a;
  a.m = m_local;
  a.n = n;
  a.mean = mean;
  a.C = C;
  a.var = var;
  a.HC = HC;
  a.CQ = CQ;
  a.dQ = dQ;
  a.HCQ = HCQ;
  a.Hmean = Hmean;
  a.no_check = true;
  a.chain = (chain & 1) != 0;
  a.chain_in = (chain & 2) != 0;
  if (chain & 4) {  // deferred: minmax_out is a device array of 3 doubles
    if (!minmax_out) {
      set_error("deferred update_rows (chain bit 4) needs a device minmax_out[3]");
      return HIKF_BAD_ARGUMENT;
    }
    a.mm_dev = minmax_out;
  }
  a.r = r;
  a.z = z;
  a.mean_out = mean_out;
  a.C_out = C_out;
  a.var_out = var_out;
  a.HC_out = HC_out;
  a.workspace = workspace;
  a.workspace_bytes = workspace_bytes;
  UpdateResult res;
  int s = update(a, as_stream(stream), &res);
  if (minmax_out && !(chain & 4)) {
    minmax_out[0] = res.min_var;
    minmax_out[1] = res.max_prior_var;
  }
  return s;
}

int hikf_csr_spmv(int64_t n, const int32_t* ip, const int32_t* ix, const double* val, const double* x, double* y,
                  void* stream) {
  if (n < 0) return HIKF_BAD_ARGUMENT;
  return spmv(n, ip, ix, val, x, y, as_stream(stream));
}

size_t hikf_spd_solve_workspace_bytes(int64_t n, int64_t k) { return spd_workspace_bytes(n, k); }

int hikf_spd_solve(int64_t n, int64_t k, const double* A, const double* B, double* X, void* ws, size_t ws_bytes,
                   int64_t* info, void* stream) {
  if (n < 0 || k < 0) return HIKF_BAD_ARGUMENT;
  return spd_solve(n, k, A, B, X, ws, ws_bytes, info, as_stream(stream));
}

int hikf_dgemm(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B, int64_t ldb,
               double* C, int64_t ldc, double alpha, double beta, int32_t kmode, int32_t variant, void* stream) {
  if (M < 0 || N < 0 || K < 0 || kmode < 0 || kmode > 2) return HIKF_BAD_ARGUMENT;
  int prev = dgemm_variant();
  if (variant >= 0) set_dgemm_variant(variant);
  GemmArgs g;
  g.M = M; g.N = N; g.K = K;
  g.A = A; g.sa_r = lda;
  g.B = B; g.sb_r = ldb;
  g.C = C; g.ldc = ldc;
  if (beta != 0.0) {
    g.Cin = C;
    g.ldcin = ldc;
  }
  g.alpha = alpha;
  g.beta = beta;
  g.kmode = kmode;
  int s = dgemm(g, 1, as_stream(stream));
  set_dgemm_variant(prev);
  return s;
}

int hikf_ray_operator_device(int64_t nx, int64_t ny, double dx, double dy, double x0, double y0, int64_t n,
                             const double* src, const double* rcv, int32_t* indptr_dev, int32_t* indices_dev,
                             double* data_dev, int64_t capacity, int64_t* nnz_out, void* stream) {
  if (!src || !rcv || !indptr_dev || !nnz_out) {
    set_error("hikf_ray_operator_device: null argument");
    return HIKF_BAD_ARGUMENT;
  }
  return ray_operator_device(nx, ny, dx, dy, x0, y0, n, src, rcv, indptr_dev, indices_dev, data_dev, capacity,
                             nnz_out, as_stream(stream));
}

int hikf_ray_operator(int64_t nx, int64_t ny, double dx, double dy, double x0, double y0, int64_t n, const double* src,
                      const double* rcv, int32_t* indptr, int32_t* indices, double* data, int64_t* nnz_out) {
  std::vector<int32_t> ip, ix;
  std::vector<double> v;
  HIKF_TRY(ray_operator(nx, ny, dx, dy, x0, y0, n, src, rcv, ip, ix, v));
  if (nnz_out) *nnz_out = (int64_t)ix.size();
  if (indices) {
    std::memcpy(indptr, ip.data(), sizeof(int32_t) * ip.size());
    std::memcpy(indices, ix.data(), sizeof(int32_t) * ix.size());
    std::memcpy(data, v.data(), sizeof(double) * v.size());
  }
  return HIKF_OK;
}

// ---- 3D path (parity unpinned; oracle/hikf_oracle3d.py) ----
int hikf_ray_operator_3d(const int64_t* n3, const double* d3, const double* o3, int64_t n, const double* src,
                         const double* rcv, int32_t* indptr, int32_t* indices, double* data, int64_t* nnz_out) {
  if (!n3 || !d3 || !o3 || (n > 0 && (!src || !rcv))) {
    set_error("hikf_ray_operator_3d: null argument");
    return HIKF_BAD_ARGUMENT;
  }
  std::vector<int32_t> ip, ix;
  std::vector<double> v;
  HIKF_TRY(ray_operator_3d(n3, d3, o3, n, src, rcv, ip, ix, v));
  if (nnz_out) *nnz_out = (int64_t)ix.size();
  if (indices) {
    std::memcpy(indptr, ip.data(), sizeof(int32_t) * ip.size());
    std::memcpy(indices, ix.data(), sizeof(int32_t) * ix.size());
    std::memcpy(data, v.data(), sizeof(double) * v.size());
  }
  return HIKF_OK;
}

int hikf_ray_operator_3d_device(const int64_t* n3, const double* d3, const double* o3, int64_t n,
                                const double* src, const double* rcv, int32_t* indptr_dev, int32_t* indices_dev,
                                double* data_dev, int64_t capacity, int64_t* nnz_out, void* stream) {
  if (!n3 || !d3 || !o3 || !indptr_dev || !nnz_out || (n > 0 && (!src || !rcv))) {
    set_error("hikf_ray_operator_3d_device: null argument");
    return HIKF_BAD_ARGUMENT;
  }
  return ray_operator_3d_device(n3, d3, o3, n, src, rcv, indptr_dev, indices_dev, data_dev, capacity, nnz_out,
                                as_stream(stream));
}

int hikf_tree3_create(const double* xyz_host, int64_t m, const hikf_kernel3* kernel, int32_t n_cheb,
                      int64_t max_leaf, void* stream, hikf_tree3** out) {
  if (!kernel || !out) {
    set_error("null argument");
    return HIKF_BAD_ARGUMENT;
  }
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0) {
    set_error("no CUDA device: the HiKF B200 path has no CPU fallback");
    return HIKF_NO_DEVICE;
  }
  keep_pool();
  return tree3_build(xyz_host, m, *kernel, n_cheb, max_leaf, as_stream(stream), out);
}

int hikf_tree3_destroy(hikf_tree3* tree) {
  tree3_free(tree);
  return HIKF_OK;
}

int hikf_tree3_info(const hikf_tree3* tree, int64_t* m, int32_t* depth, int32_t* n_cheb, int64_t* n_leaves,
                    double* lo3, double* size) {
  return tree3_info(tree, m, depth, n_cheb, n_leaves, lo3, size);
}

int hikf_tree3_export(const hikf_tree3* tree, int64_t* order, int64_t* leaf_keys, int64_t* leaf_starts,
                      int64_t* leaf_counts) {
  return tree3_export(tree, order, leaf_keys, leaf_starts, leaf_counts);
}

int hikf_tree3_matmat(const hikf_tree3* tree, const double* V, int64_t k, double* U, void* stream) {
  if (!tree || k < 0 || (k > 0 && (!V || !U))) {
    set_error("bad tree3 matmat arguments");
    return HIKF_BAD_ARGUMENT;
  }
  int64_t m = 0;
  tree3_info(tree, &m, nullptr, nullptr, nullptr, nullptr, nullptr);
  return tree3_matmat(tree, V, k, k, U, k, as_stream(stream));
}

int hikf_precompute3(hikf_tree3* t, int64_t n, const int32_t* ip, const int32_t* ix, const double* val, double* CQ,
                     double* HCQ, double* dQ, void* stream) {
  if (!t || n < 0) {
    set_error("bad precompute3 arguments");
    return HIKF_BAD_ARGUMENT;
  }
  cudaStream_t st = as_stream(stream);
  int64_t m = 0;
  tree3_info(t, &m, nullptr, nullptr, nullptr, nullptr, nullptr);
  HIKF_TRY(tree3_matmat_csrT(t, n, ip, ix, val, CQ, st));
  if (n > 0) {
    double* X = nullptr;
    HIKF_CHECK_CUDA(cudaMallocAsync((void**)&X, sizeof(double) * n * n, st));
    spmm_rows<<<(unsigned)n, kT, 0, st>>>(n, ip, ix, val, CQ, X);
    HIKF_CHECK_LAUNCH();
    symmetrize<<<grid_for(n * n), kT, 0, st>>>(X, n, HCQ);
    HIKF_CHECK_LAUNCH();
    cudaFreeAsync(X, st);
  }
  hikf_kernel3 k{};
  tree3_kernel(t, &k);
  fill<<<grid_for(m), kT, 0, st>>>(dQ, m, k.variance);  // K(0) = variance
  HIKF_CHECK_LAUNCH();
  return HIKF_OK;
}

// ---- dense Kalman filter + dense Gram (filters.py:45-74, kernels.py:97-117) ----
int hikf_dense_gram(const double* xy_host, int64_t m, const hikf_kernel* kernel, double* G_dev, void* stream) {
  if (!xy_host || !kernel || !G_dev || m < 1) {
    set_error("bad dense_gram arguments");
    return HIKF_BAD_ARGUMENT;
  }
  cudaStream_t st = as_stream(stream);
  double* xy = nullptr;
  HIKF_CHECK_CUDA(cudaMallocAsync((void**)&xy, sizeof(double) * 2 * m, st));
  HIKF_CHECK_CUDA(cudaMemcpyAsync(xy, xy_host, sizeof(double) * 2 * m, cudaMemcpyHostToDevice, st));
  int s = dense_gram(xy, m, make_kparams(*kernel), G_dev, st);
  cudaFreeAsync(xy, st);
  return s;
}

int hikf_kf_predict(int64_t m, const double* P, const double* Q, double* P_out, void* stream) {
  if (m < 1 || !P || !Q || !P_out) {
    set_error("bad kf_predict arguments");
    return HIKF_BAD_ARGUMENT;
  }
  return kf_predict(m, P, Q, P_out, as_stream(stream));
}

size_t hikf_kf_workspace_bytes(int64_t m, int64_t n) { return kf_workspace_bytes(m, n); }

int hikf_kf_update(int64_t m, int64_t n, const double* mean, const double* P, const int32_t* ip, const int32_t* ix,
                   const double* val, double r, const double* z, double* mean_out, double* P_out, void* workspace,
                   size_t workspace_bytes, void* stream) {
  if (m < 1 || n < 0 || !mean || !P || !mean_out || !P_out || (n > 0 && (!ip || !z))) {
    set_error("bad kf_update arguments");
    return HIKF_BAD_ARGUMENT;
  }
  return kf_update(m, n, mean, P, ip, ix, val, r, z, mean_out, P_out, workspace, workspace_bytes,
                   as_stream(stream));
}

}  // extern "C"

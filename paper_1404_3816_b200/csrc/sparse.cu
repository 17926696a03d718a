// Q H^T with the charges V = H^T kept sparse (filters.py:101-102 densifies
// H^T on the host; here it never exists densely anywhere).
//
// H (CSR, n rays x m cells) is regrouped on the device into "entries"
// (sorted position of the cell, ray j, length) ordered by (leaf, j, cell):
// for the crosswell operator a leaf holds ~10 rays x ~8 cells, so
//   * P2M becomes a tiny per-(leaf, ray) sum (W_leaf[a][j] = sum S_a(x_p) h_jp),
//   * P2P becomes, per active (target leaf, ray) item, a direct sum over the
//     ray's cells in the 3x3 neighbourhood (the reference's near @ V restricted
//     to its nonzeros -- the skipped terms are exact zeros),
//   * every multipole carries an 8-column activity mask that lets the DMMA
//     M2M/M2L stages skip exact-zero column groups.
#include <cub/cub.cuh>

#include <algorithm>

#include "fmm_device.cuh"
#include "prof.h"
#include "sparse.h"
#include "tree.h"

namespace hikf {

namespace {

constexpr int kT = 256;

int grid_for(int64_t n) {
  int64_t b = (n + kT - 1) / kT;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)num_sms() * 32));
}

// one CTA per ray: key = leaf * n + j, value = CSR position
__global__ void entry_keys(int64_t n, const int32_t* __restrict__ ip, const int32_t* __restrict__ ix,
                           const int32_t* __restrict__ inv_order, const int32_t* __restrict__ leaf_of,
                           int64_t* __restrict__ key, int32_t* __restrict__ pos) {
  int64_t j = blockIdx.x;
  for (int64_t e = ip[j] + threadIdx.x; e < ip[j + 1]; e += blockDim.x) {
    int32_t sp = inv_order[ix[e]];
    key[e] = (int64_t)leaf_of[sp] * n + j;
    pos[e] = (int32_t)e;
  }
}

__global__ void entry_gather(int64_t nnz, int64_t n, const int64_t* __restrict__ key, const int32_t* __restrict__ pos,
                             const int32_t* __restrict__ ix, const double* __restrict__ val,
                             const int32_t* __restrict__ inv_order, int32_t* __restrict__ e_sp,
                             int32_t* __restrict__ e_j, double* __restrict__ e_v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t p = pos[i];
    e_sp[i] = inv_order[ix[p]];
    e_j[i] = (int32_t)(key[i] % n);
    e_v[i] = val[p];
  }
}

// groups: run starts of equal (leaf, j) keys
__global__ void group_tables(int64_t ng, int64_t n, const int64_t* __restrict__ gkey, const int32_t* __restrict__ gcnt,
                             const int32_t* __restrict__ gstart_excl, int32_t* __restrict__ g_j,
                             int32_t* __restrict__ g_leaf, int32_t* __restrict__ g_start) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ng; i += (int64_t)gridDim.x * blockDim.x) {
    g_j[i] = (int32_t)(gkey[i] % n);
    g_leaf[i] = (int32_t)(gkey[i] / n);
    g_start[i] = gstart_excl[i];
    if (i == ng - 1) g_start[ng] = gstart_excl[i] + gcnt[i];
  }
}

// leaf_g[L] = first group with leaf >= L (binary search), L in [0, nleaves]
__global__ void leaf_group_offsets(int64_t nleaves, int64_t ng, const int32_t* __restrict__ g_leaf,
                                   int32_t* __restrict__ leaf_g) {
  for (int64_t L = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; L <= nleaves; L += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = ng;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (g_leaf[mid] < L) lo = mid + 1; else hi = mid;
    }
    leaf_g[L] = (int32_t)lo;
  }
}

// leaf-level mask: a leaf box is active for group j/8 if it holds a nonzero of ray j
__global__ void leaf_mask(int64_t ng, const int32_t* __restrict__ g_leaf, const int32_t* __restrict__ g_j,
                          const int32_t* __restrict__ leaf_box, int64_t ngr, uint8_t* __restrict__ mask) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ng; i += (int64_t)gridDim.x * blockDim.x)
    mask[(int64_t)leaf_box[g_leaf[i]] * ngr + g_j[i] / 8] = 1;
}

// parent mask = OR of the four children (exact: a parent multipole is a sum of children's)
__global__ void parent_mask(int64_t Gp, int64_t ngr, const uint8_t* __restrict__ child, uint8_t* __restrict__ parent) {
  int64_t total = Gp * Gp * ngr;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t box = e / ngr, gg = e % ngr, X = box / Gp, Y = box % Gp;
    uint8_t v = 0;
    for (int c = 0; c < 4; ++c) {
      int64_t ch = (2 * X + (c >> 1)) * (2 * Gp) + (2 * Y + (c & 1));
      v |= child[ch * ngr + gg];
    }
    parent[e] = v;
  }
}

// a sorted unique key list ends with the sentinel when some inputs carried it: drop it from the count
__global__ void drop_sentinel(int32_t* __restrict__ num, const int64_t* __restrict__ keys, int64_t sentinel) {
  if (*num > 0 && keys[*num - 1] == sentinel) --*num;
}

// candidate P2P items: for every (source leaf, j) group, the <= 9 adjacent
// occupied target leaves; key = target * n + j (sentinel = none; it sorts last)
__global__ void item_candidates(int64_t ng, int64_t n, int64_t G, const int32_t* __restrict__ g_leaf,
                                const int32_t* __restrict__ g_j, const int32_t* __restrict__ leaf_box,
                                const int32_t* __restrict__ box2leaf, int64_t sentinel, int64_t* __restrict__ cand) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ng; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t box = leaf_box[g_leaf[i]], bx = box / G, by = box % G;
    for (int s = 0; s < 9; ++s) {
      int64_t nx = bx + (s / 3 - 1), ny = by + (s % 3 - 1);
      int64_t k = sentinel;
      if (nx >= 0 && nx < G && ny >= 0 && ny < G) {
        int32_t T = box2leaf[nx * G + ny];
        if (T >= 0) k = (int64_t)T * n + g_j[i];
      }
      cand[i * 9 + s] = k;
    }
  }
}

// Sparse P2M: W_leaf[a][j] = sum_{entries (p, j, v) of the leaf} W2[p][a] v, and
// zeros for the inactive columns of every active 8-column group.
__global__ void p2m_sparse(int q, int64_t kcols, int64_t c0, int64_t ngr, const int32_t* __restrict__ leaf_box,
                           const int32_t* __restrict__ leaf_g, const int32_t* __restrict__ g_j,
                           const int32_t* __restrict__ g_start, const int32_t* __restrict__ e_sp,
                           const double* __restrict__ e_v, const double* __restrict__ W2s,
                           const uint8_t* __restrict__ mask, double* __restrict__ W) {
  const int64_t L = blockIdx.x;
  const int64_t box = leaf_box[L];
  const int32_t gb = leaf_g[L], ge = leaf_g[L + 1];
  if (gb == ge) return;
  double* Wb = W + box * q * kcols;
  const uint8_t* mrow = mask + box * ngr;
  // zero the active groups of this column pass [c0, c0 + kcols)
  for (int64_t e = threadIdx.x; e < (int64_t)q * kcols; e += blockDim.x) {
    int64_t a = e / kcols, c = e % kcols;
    if (mrow[(c0 + c) >> 3]) Wb[a * kcols + c] = 0.0;
  }
  __syncthreads();
  for (int64_t e = threadIdx.x; e < (int64_t)(ge - gb) * q; e += blockDim.x) {
    int32_t gi = gb + (int32_t)(e / q);
    int a = (int)(e % q);
    int64_t c = (int64_t)g_j[gi] - c0;
    if (c < 0 || c >= kcols) continue;
    double s = 0.0;
    for (int32_t k = g_start[gi]; k < g_start[gi + 1]; ++k) s += W2s[(int64_t)e_sp[k] * q + a] * e_v[k];
    Wb[(int64_t)a * kcols + c] = s;
  }
}

// Sparse P2P, one warp per active (target leaf T, ray j):
// U[t][j] += sum_{adjacent leaves s (ox outer, oy inner)} sum_{entries (p, j, v) in s} K(x_t, x_p) v
__global__ void __launch_bounds__(256, 8) p2p_sparse(int64_t nitems, const int64_t* __restrict__ items, int64_t n, int64_t G, KParams kp,
                           const int32_t* __restrict__ leaf_box, const int32_t* __restrict__ leaf_start,
                           const int32_t* __restrict__ leaf_count, const int32_t* __restrict__ box2leaf,
                           const int32_t* __restrict__ leaf_g, const int32_t* __restrict__ g_j,
                           const int32_t* __restrict__ g_start, const int32_t* __restrict__ e_sp,
                           const double* __restrict__ e_v, const double* __restrict__ xy_s,
                           const int64_t* __restrict__ order, double* __restrict__ U, int64_t ldu,
                           double* __restrict__ Pnear, int32_t maxc, int64_t r0, int64_t r1,
                           unsigned long long* __restrict__ flops, int64_t leaf0, int64_t leaf1, int64_t s0,
                           const double* __restrict__ near) {
  const int64_t item = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (item >= nitems) return;
  const int64_t key = items[item];
  const int32_t T = (int32_t)(key / n);
  const int32_t j = (int32_t)(key % n);
  if (T < leaf0 || T >= leaf1) return;  // another shard's target leaf
  const int64_t box = leaf_box[T], bx = box / G, by = box % G;
  // the <= 9 entry ranges of ray j in the adjacent leaves (and their first sorted positions):
  // lane s looks up neighbour s, the ranges are then exchanged by shuffles
  int32_t my_rb = 0, my_re = 0, my_sb = 0;
  if (lane < 9) {
    const int s = lane;
    int64_t nx = bx + (s / 3 - 1), ny = by + (s % 3 - 1);
    if (nx >= 0 && nx < G && ny >= 0 && ny < G) {
      int32_t S = box2leaf[nx * G + ny];
      if (S >= 0) {
        my_sb = leaf_start[S];
        const int32_t end = leaf_g[S + 1];
        int32_t lo = leaf_g[S], hi = end;
        while (lo < hi) {
          int32_t mid = (lo + hi) >> 1;
          if (g_j[mid] < j) lo = mid + 1; else hi = mid;
        }
        if (lo < end && g_j[lo] == j) {
          my_rb = g_start[lo];
          my_re = g_start[lo + 1];
        }
      }
    }
  }
  const int32_t t0 = leaf_start[T], cnt = leaf_count[T];
  // inclusive prefix of the ranges' lengths over the neighbours (lanes 0..8)
  int32_t incl = my_re - my_rb;
#pragma unroll
  for (int d = 1; d < 16; d <<= 1) {
    const int32_t up = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += up;
  }
  const int32_t total = __shfl_sync(0xffffffffu, incl, 8);
  if (flops && lane == 0) atomicAdd(flops, 2ull * (unsigned long long)total * cnt);
  if (near) {
    // kernel values from the tree's near blocks (the same values, evaluated at build).  The
    // ray's entries in the neighbourhood, in (neighbour, entry) order, are fetched 32 at a time
    // (one per lane, coalesced) and handed round by shuffles; the block loads of several
    // entries are in flight together, the sums keep the entry order.
    const double* blkT = near + (int64_t)T * 9 * 64 * 64;
    const bool ok0 = lane < cnt, ok1 = lane + 32 < cnt;
    double acc0 = 0.0, acc1 = 0.0;
    for (int32_t base = 0; base < total; base += 32) {
      const int32_t e = base + lane;
      int s_of = 0;
      int32_t excl = 0;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int32_t inc_s = __shfl_sync(0xffffffffu, incl, s);
        if (e >= inc_s) {
          s_of = s + 1;
          excl = inc_s;
        }
      }
      const int32_t rb_s = __shfl_sync(0xffffffffu, my_rb, s_of), sb_s = __shfl_sync(0xffffffffu, my_sb, s_of);
      int32_t off = 0;
      double v = 0.0;
      if (e < total) {
        const int32_t k = rb_s + (e - excl);
        off = (s_of * 64 + (e_sp[k] - sb_s)) * 64;
        v = e_v[k];
      }
      const int nch = total - base < 32 ? total - base : 32;
#pragma unroll 8
      for (int i = 0; i < nch; ++i) {
        const int32_t off_i = __shfl_sync(0xffffffffu, off, i);
        const double v_i = __shfl_sync(0xffffffffu, v, i);
        if (ok0) acc0 += blkT[off_i + lane] * v_i;
        if (ok1) acc1 += blkT[off_i + lane + 32] * v_i;
      }
    }
#pragma unroll
    for (int hb = 0; hb < 2; ++hb) {
      const int t = hb * 32 + lane;
      if (t >= cnt) continue;
      const double acc = hb ? acc1 : acc0;
      if (Pnear)
        Pnear[item * maxc + t] = acc;  // added into U later (leaf_down / p2p_scatter): U = far + near either way
      else if (s0 >= 0) {
        U[(t0 + t - s0) * ldu + j] += acc;
      } else {
        const int64_t row = order[t0 + t];
        if (row >= r0 && row < r1) U[(row - r0) * ldu + j] += acc;
      }
    }
    return;
  }
  int32_t rb[9], re[9];
#pragma unroll
  for (int s = 0; s < 9; ++s) {
    rb[s] = __shfl_sync(0xffffffffu, my_rb, s);
    re[s] = __shfl_sync(0xffffffffu, my_re, s);
  }
  for (int tb = 0; tb < cnt; tb += 32) {
    const int t = tb + lane;
    const bool ok = t < cnt;
    double tx = 0.0, ty = 0.0;
    if (ok) {
      tx = xy_s[2 * (int64_t)(t0 + t)];
      ty = xy_s[2 * (int64_t)(t0 + t) + 1];
    }
    double acc = 0.0;
#pragma unroll 1
    for (int s = 0; s < 9; ++s)
      for (int32_t k = rb[s]; k < re[s]; ++k) {
        const int32_t p = e_sp[k];
        const double v = e_v[k];
        acc += kernel_of_r_near(kp, dist2d(tx, ty, xy_s[2 * (int64_t)p], xy_s[2 * (int64_t)p + 1])) * v;
      }
    if (!ok) continue;
    if (Pnear)
      Pnear[item * maxc + t] = acc;  // added into U later (leaf_down / p2p_scatter): U = far + near either way
    else if (s0 >= 0) {
      U[(t0 + t - s0) * ldu + j] += acc;
    } else {
      const int64_t row = order[t0 + t];
      if (row >= r0 && row < r1) U[(row - r0) * ldu + j] += acc;
    }
  }
}

// U[target, ray] += near sum (the deferred add of p2p_sparse, for the paths that do not
// add it inside the fused leaf step).  One warp per item, lanes over the leaf's points;
// Pnear is item-major (item * maxc + t).
__global__ void p2p_scatter(int64_t nitems, const int64_t* __restrict__ items, int64_t n,
                            const int32_t* __restrict__ leaf_start, const int32_t* __restrict__ leaf_count,
                            const int64_t* __restrict__ order, const double* __restrict__ Pnear, int32_t maxc,
                            double* __restrict__ U, int64_t ldu, int64_t r0, int64_t r1, int64_t leaf0,
                            int64_t leaf1, int64_t s0) {
  const int64_t item = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (item >= nitems) return;
  const int64_t key = items[item];
  const int32_t T = (int32_t)(key / n);
  const int32_t j = (int32_t)(key % n);
  if (T < leaf0 || T >= leaf1) return;
  const int32_t t0 = leaf_start[T], cnt = leaf_count[T];
  for (int t = lane; t < cnt; t += 32) {
    if (s0 >= 0) {
      U[(t0 + t - s0) * ldu + j] += Pnear[item * maxc + t];
      continue;
    }
    const int64_t row = order[t0 + t];
    if (row >= r0 && row < r1) U[(row - r0) * ldu + j] += Pnear[item * maxc + t];
  }
}

// item_start[L] = first item of target leaf L (items ascend in leaf * n + ray), L in [0, nleaves]
__global__ void item_offsets(int64_t nleaves, int64_t nitems, int64_t n, const int64_t* __restrict__ items,
                             int32_t* __restrict__ item_start) {
  const int64_t L = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (L > nleaves) return;
  int64_t lo = 0, hi = nitems;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (items[mid] < L * n) lo = mid + 1; else hi = mid;
  }
  item_start[L] = (int32_t)lo;
}
}  // namespace

void sparse_free(SparseHt* s, cudaStream_t st) {
  cudaFreeAsync(s->e_sp, st);
  cudaFreeAsync(s->e_j, st);
  cudaFreeAsync(s->e_v, st);
  cudaFreeAsync(s->g_j, st);
  cudaFreeAsync(s->g_start, st);
  cudaFreeAsync(s->leaf_g, st);
  cudaFreeAsync(s->g_leaf, st);
  cudaFreeAsync(s->items, st);
  cudaFreeAsync(s->item_start, st);
  for (int l = 0; l <= kMaxDepth; ++l) cudaFreeAsync(s->mask[l], st);
  *s = SparseHt();
}

template <class T>
static int aalloc(T** p, size_t count, cudaStream_t st) {
  HIKF_CHECK_CUDA(cudaMallocAsync((void**)p, std::max<size_t>(1, count) * sizeof(T), st));
  return HIKF_OK;
}

int sparse_build(const hikf_tree* t, int64_t n, const int32_t* ip, const int32_t* ix, const double* val, SparseHt* s,
                 cudaStream_t st) {
  const bool masks = s->build_masks;
  *s = SparseHt();
  s->build_masks = masks;
  s->n = n;
  s->ngr = (n + 7) / 8;
  int32_t nnz32 = 0;
  HIKF_CHECK_CUDA(cudaMemcpyAsync(&nnz32, ip + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  HIKF_CHECK_CUDA(cudaStreamSynchronize(st));
  const int64_t nnz = nnz32;
  s->nnz = nnz;
  const int64_t L = t->n_leaves;

  // ---- entries sorted by (leaf, j); CSR order (j, cell) makes the sort keep cell order ----
  int64_t *key = nullptr, *key_s = nullptr;
  int32_t *pos = nullptr, *pos_s = nullptr;
  HIKF_TRY(aalloc(&key, nnz, st));
  HIKF_TRY(aalloc(&key_s, nnz, st));
  HIKF_TRY(aalloc(&pos, nnz, st));
  HIKF_TRY(aalloc(&pos_s, nnz, st));
  if (n > 0) {
    entry_keys<<<(unsigned)n, kT, 0, st>>>(n, ip, ix, t->inv_order, t->leaf_of, key, pos);
    HIKF_CHECK_LAUNCH();
  }
  int end_bit = 1;
  while (end_bit < 63 && ((int64_t)1 << end_bit) < L * n) ++end_bit;
  size_t b1 = 0, b2 = 0, b3 = 0, b4 = 0;
  int32_t* d_num = nullptr;
  HIKF_TRY(aalloc(&d_num, 2, st));
  int64_t* gkey = nullptr;
  int32_t *gcnt = nullptr, *gexcl = nullptr;
  HIKF_TRY(aalloc(&gkey, nnz, st));
  HIKF_TRY(aalloc(&gcnt, nnz, st));
  HIKF_TRY(aalloc(&gexcl, nnz, st));
  cub::DeviceRadixSort::SortPairs(nullptr, b1, key, key_s, pos, pos_s, (int)nnz, 0, end_bit, st);
  cub::DeviceRunLengthEncode::Encode(nullptr, b2, key_s, gkey, gcnt, d_num, (int)nnz, st);
  cub::DeviceScan::ExclusiveSum(nullptr, b3, gcnt, gexcl, (int)nnz, st);
  void* tmp = nullptr;
  size_t tb = std::max(std::max(b1, b2), b3);
  HIKF_CHECK_CUDA(cudaMallocAsync(&tmp, std::max<size_t>(tb, 1), st));
  cub::DeviceRadixSort::SortPairs(tmp, b1, key, key_s, pos, pos_s, (int)nnz, 0, end_bit, st);
  HIKF_TRY(aalloc(&s->e_sp, nnz, st));
  HIKF_TRY(aalloc(&s->e_j, nnz, st));
  HIKF_TRY(aalloc(&s->e_v, nnz, st));
  entry_gather<<<grid_for(nnz), kT, 0, st>>>(nnz, n, key_s, pos_s, ix, val, t->inv_order, s->e_sp, s->e_j, s->e_v);
  HIKF_CHECK_LAUNCH();
  cub::DeviceRunLengthEncode::Encode(tmp, b2, key_s, gkey, gcnt, d_num, (int)nnz, st);
  int32_t ngroups = 0;
  HIKF_CHECK_CUDA(cudaMemcpyAsync(&ngroups, d_num, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  HIKF_CHECK_CUDA(cudaStreamSynchronize(st));
  s->ngroups = ngroups;
  cub::DeviceScan::ExclusiveSum(tmp, b3, gcnt, gexcl, (int)ngroups, st);
  HIKF_TRY(aalloc(&s->g_j, ngroups, st));
  HIKF_TRY(aalloc(&s->g_leaf, ngroups, st));
  int32_t* g_leaf = s->g_leaf;
  HIKF_TRY(aalloc(&s->g_start, ngroups + 1, st));
  HIKF_TRY(aalloc(&s->leaf_g, L + 1, st));
  if (ngroups > 0) {
    group_tables<<<grid_for(ngroups), kT, 0, st>>>(ngroups, n, gkey, gcnt, gexcl, s->g_j, g_leaf, s->g_start);
    HIKF_CHECK_LAUNCH();
  } else {
    HIKF_CHECK_CUDA(cudaMemsetAsync(s->g_start, 0, sizeof(int32_t), st));
  }
  leaf_group_offsets<<<grid_for(L + 1), kT, 0, st>>>(L, ngroups, g_leaf, s->leaf_g);
  HIKF_CHECK_LAUNCH();

  // ---- activity masks per level (only for the masked dense path) ----
  const int D = t->depth;
  if (D >= 2 && s->build_masks) {
    int64_t G = t->G;
    HIKF_TRY(aalloc(&s->mask[D], G * G * s->ngr, st));
    HIKF_CHECK_CUDA(cudaMemsetAsync(s->mask[D], 0, G * G * s->ngr, st));
    if (ngroups > 0) {
      leaf_mask<<<grid_for(ngroups), kT, 0, st>>>(ngroups, g_leaf, s->g_j, t->leaf_box, s->ngr, s->mask[D]);
      HIKF_CHECK_LAUNCH();
    }
    for (int l = D - 1; l >= 2; --l) {
      int64_t Gp = (int64_t)1 << l;
      HIKF_TRY(aalloc(&s->mask[l], Gp * Gp * s->ngr, st));
      parent_mask<<<grid_for(Gp * Gp * s->ngr), kT, 0, st>>>(Gp, s->ngr, s->mask[l + 1], s->mask[l]);
      HIKF_CHECK_LAUNCH();
    }
  }

  // ---- P2P work items: unique (target leaf, j) over all groups' neighbourhoods ----
  int64_t ncand = 9 * (int64_t)ngroups;
  int64_t *cand = nullptr, *cand_s = nullptr;
  HIKF_TRY(aalloc(&cand, ncand, st));
  HIKF_TRY(aalloc(&cand_s, ncand, st));
  HIKF_TRY(aalloc(&s->items, ncand, st));
  if (ngroups > 0) {
    // keys < L n; the sentinel L n sorts last; only the bits that can be set are sorted
    const int64_t sentinel = L * n;
    int item_bits = 1;
    while (item_bits < 62 && ((int64_t)1 << item_bits) <= sentinel) ++item_bits;
    item_candidates<<<grid_for(ngroups), kT, 0, st>>>(ngroups, n, t->G, g_leaf, s->g_j, t->leaf_box, t->box2leaf,
                                                      sentinel, cand);
    HIKF_CHECK_LAUNCH();
    size_t b5 = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, b4, cand, cand_s, (int)ncand, 0, item_bits, st);
    cub::DeviceSelect::Unique(nullptr, b5, cand_s, s->items, d_num + 1, (int)ncand, st);
    void* tmp2 = nullptr;
    HIKF_CHECK_CUDA(cudaMallocAsync(&tmp2, std::max(b4, b5), st));
    cub::DeviceRadixSort::SortKeys(tmp2, b4, cand, cand_s, (int)ncand, 0, item_bits, st);
    cub::DeviceSelect::Unique(tmp2, b5, cand_s, s->items, d_num + 1, (int)ncand, st);
    drop_sentinel<<<1, 1, 0, st>>>(d_num + 1, s->items, sentinel);
    HIKF_CHECK_LAUNCH();
    int32_t nu = 0;
    HIKF_CHECK_CUDA(cudaMemcpyAsync(&nu, d_num + 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    HIKF_CHECK_CUDA(cudaStreamSynchronize(st));
    s->nitems = nu;
    cudaFreeAsync(tmp2, st);
  }
  HIKF_TRY(aalloc(&s->item_start, L + 1, st));
  item_offsets<<<grid_for(L + 1), kT, 0, st>>>(L, s->nitems, n, s->items, s->item_start);
  HIKF_CHECK_LAUNCH();
  cudaFreeAsync(tmp, st);
  cudaFreeAsync(key, st);
  cudaFreeAsync(key_s, st);
  cudaFreeAsync(pos, st);
  cudaFreeAsync(pos_s, st);
  cudaFreeAsync(gkey, st);
  cudaFreeAsync(gcnt, st);
  cudaFreeAsync(gexcl, st);
  cudaFreeAsync(cand, st);
  cudaFreeAsync(cand_s, st);
  cudaFreeAsync(d_num, st);
  return HIKF_OK;
}

int sparse_p2m(const hikf_tree* t, const SparseHt& s, double* W, int64_t kcols, int64_t c0, cudaStream_t st) {
  const int q = t->orders[t->depth] * t->orders[t->depth];
  if (t->n_leaves > 0) {
    p2m_sparse<<<(unsigned)t->n_leaves, 128, 0, st>>>(q, kcols, c0, s.ngr, t->leaf_box, s.leaf_g, s.g_j, s.g_start,
                                                       s.e_sp, s.e_v, t->W2s, s.mask[t->depth], W);
    HIKF_CHECK_LAUNCH();
  }
  return HIKF_OK;
}

static int g_near_blocks = 1;

int p2p_set_near_blocks(int on) {
  const int prev = g_near_blocks;
  g_near_blocks = on ? 1 : 0;
  return prev;
}

int sparse_p2p(const hikf_tree* t, const SparseHt& s, double* U, int64_t ldu, cudaStream_t st, double* Pnear,
               int64_t r0, int64_t r1, const LeafWindow* lw) {
  if (s.nitems <= 0) return HIKF_OK;
  const int64_t threads = s.nitems * 32;
  p2p_sparse<<<(unsigned)((threads + kT - 1) / kT), kT, 0, st>>>(
      s.nitems, s.items, s.n, t->G, t->kp, t->leaf_box, t->leaf_start, t->leaf_count, t->box2leaf, s.leaf_g, s.g_j,
      s.g_start, s.e_sp, s.e_v, t->xy_s, t->order, U, ldu, Pnear, (int32_t)t->max_count, r0,
      r1 < 0 ? INT64_MAX : r1, prof_flops_ptr(ST_P2P), lw ? lw->leaf0 : 0, lw ? lw->leaf1 : INT64_MAX,
      lw ? lw->s0 : -1, g_near_blocks ? t->near : nullptr);
  HIKF_CHECK_LAUNCH();
  return HIKF_OK;
}

int sparse_p2p_scatter(const hikf_tree* t, const SparseHt& s, const double* Pnear, double* U, int64_t ldu,
                       cudaStream_t st, int64_t r0, int64_t r1, const LeafWindow* lw) {
  if (s.nitems <= 0) return HIKF_OK;
  p2p_scatter<<<(unsigned)((s.nitems * 32 + kT - 1) / kT), kT, 0, st>>>(s.nitems, s.items, s.n, t->leaf_start,
                                                                 t->leaf_count, t->order, Pnear,
                                                                 (int32_t)t->max_count, U, ldu, r0,
                                                                 r1 < 0 ? INT64_MAX : r1, lw ? lw->leaf0 : 0,
                                                                 lw ? lw->leaf1 : INT64_MAX, lw ? lw->s0 : -1);
  HIKF_CHECK_LAUNCH();
  return HIKF_OK;
}


namespace {

__global__ void leaf_pair_keys(int64_t ng, int64_t n, const int32_t* __restrict__ g_leaf,
                               const int32_t* __restrict__ g_j, const int32_t* __restrict__ leaf_box,
                               int64_t* __restrict__ key) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ng; i += (int64_t)gridDim.x * blockDim.x)
    key[i] = (int64_t)leaf_box[g_leaf[i]] * n + g_j[i];
}

// Wc[g][a] = sum_{entries (p, v) of group g} W2[p][a] v   (fmm.py:338 restricted to nonzeros)
__device__ __forceinline__ void count_flops(unsigned long long* flops, unsigned v) {
  if (!flops) return;
  unsigned tot = __reduce_add_sync(__activemask(), v);
  if ((threadIdx.x & 31) == __ffs(__activemask()) - 1 && tot) atomicAdd(flops, (unsigned long long)tot);
}

__global__ void p2m_pairs(int64_t ng, int q, const int32_t* __restrict__ g_start, const int32_t* __restrict__ e_sp,
                          const double* __restrict__ e_v, const double* __restrict__ W2s, double* __restrict__ Wc,
                          unsigned long long* __restrict__ flops) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ng * q; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t gi = e / q;
    int a = (int)(e % q);
    double s = 0.0;
    for (int32_t k = g_start[gi]; k < g_start[gi + 1]; ++k) s += W2s[(int64_t)e_sp[k] * q + a] * e_v[k];
    Wc[e] = s;
    count_flops(flops, 2u * (unsigned)(g_start[gi + 1] - g_start[gi]));
  }
}

// keys of the ancestors sh levels above the pairs' boxes (Gc: the pairs' grid)
// (np: allocated child pairs; np_dev: their actual number on the device, or null when np is
// exact -- the slots past it get the sentinel key, which sorts last)
__global__ void parent_keys(int64_t np, const int32_t* __restrict__ np_dev, const int64_t* __restrict__ ckey,
                            int64_t n, int64_t Gc, int sh, int64_t sentinel, int64_t* __restrict__ pkey) {
  const int64_t nv = np_dev ? *np_dev : np;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np; i += (int64_t)gridDim.x * blockDim.x) {
    if (i >= nv) {
      pkey[i] = sentinel;
      continue;
    }
    int64_t box = ckey[i] / n, j = ckey[i] % n;
    int64_t cx = box / Gc, cy = box % Gc;
    pkey[i] = ((cx >> sh) * (Gc >> sh) + (cy >> sh)) * n + j;
  }
}

__device__ __forceinline__ int64_t find_key(const int64_t* __restrict__ keys, int64_t np, int64_t k) {
  int64_t lo = 0, hi = np;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < k) lo = mid + 1; else hi = mid;
  }
  return (lo < np && keys[lo] == k) ? lo : -1;
}

// cidx[parent pair][c] = the child pair (2X + (c >> 1), 2Y + (c & 1), j) of a parent pair, or -1:
// one thread per child pair finds its parent by binary search (all searches in parallel,
// instead of four per parent warp in front of the M2M sums)
__global__ void child_index(int64_t npc, const int32_t* __restrict__ npc_dev, const int64_t* __restrict__ ckey,
                            int64_t n, int64_t Gc, int64_t npp, const int32_t* __restrict__ npp_dev,
                            const int64_t* __restrict__ pkey, int32_t* __restrict__ cidx) {
  if (npc_dev) npc = *npc_dev;
  if (npp_dev) npp = *npp_dev;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npc; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t box = ckey[i] / n, j = ckey[i] % n, cx = box / Gc, cy = box % Gc;
    const int64_t p = find_key(pkey, npp, ((cx >> 1) * (Gc >> 1) + (cy >> 1)) * n + j);
    if (p >= 0) cidx[p * 4 + (((cx & 1) << 1) | (cy & 1))] = (int32_t)i;
  }
}

// W_P[b][j] = sum_{children c (cx, cy order)} sum_a C_c[a][b] W_c[a][j]  (fmm.py:339-345)
// One warp per parent pair, the lanes stride over b; each output keeps the
// children-then-a summation order.
__global__ void m2m_pairs(int64_t npp, const int32_t* __restrict__ npp_dev, int qp, int qc,
                          const double* __restrict__ shift, const int32_t* __restrict__ cidx,
                          const double* __restrict__ Wcc, double* __restrict__ Wp, unsigned long long* __restrict__ flops) {
  if (npp_dev) npp = *npp_dev;  // the pair count on the device (deferred mode: npp is the allocated size)
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t pi = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; pi < npp; pi += nwarps) {
    const int4 ci4 = *reinterpret_cast<const int4*>(cidx + pi * 4);
    const int32_t ci[4] = {ci4.x, ci4.y, ci4.z, ci4.w};
    unsigned found = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) found += ci[c] >= 0;
    // two outputs per lane (b, b + 32) share each broadcast child coefficient
    for (int bb = 0; bb < qp; bb += 64) {
      const int b0 = bb + lane, b1 = bb + lane + 32;
      const bool ok0 = b0 < qp, ok1 = b1 < qp;
      const int c0 = ok0 ? b0 : 0, c1 = ok1 ? b1 : 0;  // in-range columns for the idle lanes
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (ci[c] < 0) continue;
        const double* C = shift + (int64_t)c * qc * qp;
        const double* w = Wcc + (int64_t)ci[c] * qc;
#pragma unroll 4
        for (int a = 0; a < qc; ++a) {
          const double wa = w[a];
          s0 += C[(int64_t)a * qp + c0] * wa;
          s1 += C[(int64_t)a * qp + c1] * wa;
        }
      }
      if (ok0) Wp[pi * qp + b0] = s0;
      if (ok1) Wp[pi * qp + b1] = s1;
    }
    if (flops && lane == 0) atomicAdd(flops, 2ull * found * (unsigned long long)qc * qp);
  }
}

__host__ __device__ inline int m2l_ld(int q) { return q + ((4 - q % 16) + 16) % 16; }  // == 4 mod 16

// All M2L terms of a level in one launch: Pr[i][:] = M_d W_p for every entry i = (p, slot)
// of every offset d.  The products do not depend on one another, so the 40 offsets need no
// ordering (and no read-modify-write of the targets); m2l_reduce then adds each target's
// products in the reference's offset order.  A CTA stages M_d once and its warps walk gpw
// groups of 8 entries (the 8 columns of the DMMA tiles); the product of an entry is formed
// in two accumulator chains (even / odd k-steps) that are then summed, so the rounding is that of
// l_lev[t] += M @ w (fmm.py:349-360) term by term.
struct M2LProd {
  const int2* ent;
  const double *W, *M;  // source coefficients (q per pair), the level's 40 operators
  double* Pr;           // q per entry
  int32_t* tab;         // tab[slot][d] = the entry of offset d that targets the slot (preset to -1)
  int64_t off[41];      // first entry of every offset
  int64_t blk[41];      // first CTA of every offset
};

template <int NK4, int NRT>
__global__ void __launch_bounds__(256, (NK4 <= 13) ? 3 : 2) m2l_prod_kernel(M2LProd a, int q, int gpw,
                                                                         unsigned long long* __restrict__ flops) {
  __shared__ int s_d;
  if (threadIdx.x < 40) {
    const int d = threadIdx.x;
    if ((int64_t)blockIdx.x >= a.blk[d] && (int64_t)blockIdx.x < a.blk[d + 1]) s_d = d;
  }
  __syncthreads();
  const int d = s_d;
  extern __shared__ double Ms[];
  const int ld = m2l_ld(q);
  const double* __restrict__ M = a.M + (int64_t)d * q * q;
  // M_d: asynchronous copies, all in flight at once
  for (int e = threadIdx.x; e < q * q; e += blockDim.x) cp_async8(Ms + (e / q) * ld + e % q, M + e, true);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t4 = lane & 3;
  const int64_t e_end = a.off[d + 1];
  const int64_t chunk0 = a.off[d] + ((int64_t)blockIdx.x - a.blk[d]) * (64 * (int64_t)gpw);
  int64_t i0 = chunk0 + warp * 8;
  int2 pe_next = make_int2(-1, -1);
  if (i0 + g < e_end) pe_next = a.ent[i0 + g];
  unsigned long long useful = 0;  // profiling: one global atomic per CTA
  for (int gi = 0; gi < gpw; ++gi, i0 += 64) {
    if (i0 >= e_end) break;
    const int2 pe = pe_next;
    pe_next = make_int2(-1, -1);
    if (gi + 1 < gpw && i0 + 64 + g < e_end) pe_next = a.ent[i0 + 64 + g];
    useful += 2ull * (unsigned long long)(e_end - i0 < 8 ? e_end - i0 : 8) * q * q;
    double b[NK4];
#pragma unroll
    for (int k4 = 0; k4 < NK4; ++k4) {
      const int k = k4 * 4 + t4;
      b[k4] = (pe.x >= 0 && k < q) ? a.W[(int64_t)pe.x * q + k] : 0.0;
    }
    if (t4 == 0 && pe.x >= 0) a.tab[(int64_t)pe.y * 40 + d] = (int32_t)(i0 + g);  // a target has one source per offset
    double* out[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t i = i0 + 2 * t4 + h;
      out[h] = i < e_end ? a.Pr + i * q : nullptr;
    }
#pragma unroll 2
    for (int i = 0; i < NRT; ++i) {
      const int r = i * 8 + g;
      double acc0[2] = {0.0, 0.0}, acc1[2] = {0.0, 0.0};
#pragma unroll
      for (int k4 = 0; k4 < NK4; ++k4) {
        const int k = k4 * 4 + t4;
        const double av = (r < q && k < q) ? Ms[r * ld + k] : 0.0;
        if (k4 & 1)
          dmma884(acc1[0], acc1[1], av, b[k4]);
        else
          dmma884(acc0[0], acc0[1], av, b[k4]);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (out[h] && r < q) out[h][r] = acc0[h] + acc1[h];
    }
  }
  if (flops) {
    __shared__ unsigned long long s_fl;
    if (threadIdx.x == 0) s_fl = 0;
    __syncthreads();
    if (lane == 0 && useful) atomicAdd(&s_fl, useful);
    __syncthreads();
    if (threadIdx.x == 0 && s_fl) atomicAdd(flops, s_fl);
  }
}

// The same for any order (q up to 256: the boosted orders 9..16 of the coarse levels): M_d and
// the source coefficients are read from global memory (L1 / L2), 8 row tiles per pass, one
// accumulator chain per tile over ascending k -- the arithmetic of the former per-offset generic
// pass, so its results bit for bit, with the 40 offsets of the level side by side in one launch.
__global__ void __launch_bounds__(256) m2l_prod_generic_kernel(M2LProd a, int q, unsigned long long* __restrict__ flops) {
  __shared__ int s_d;
  if (threadIdx.x < 40) {
    const int d = threadIdx.x;
    if ((int64_t)blockIdx.x >= a.blk[d] && (int64_t)blockIdx.x < a.blk[d + 1]) s_d = d;
  }
  __syncthreads();
  const int d = s_d;
  const double* __restrict__ M = a.M + (int64_t)d * q * q;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t4 = lane & 3;
  const int64_t e_end = a.off[d + 1];
  const int64_t i0 = a.off[d] + ((int64_t)blockIdx.x - a.blk[d]) * 64 + warp * 8;
  if (i0 >= e_end) return;
  int2 pe = make_int2(-1, -1);
  if (i0 + g < e_end) pe = a.ent[i0 + g];
  if (flops && lane == 0) atomicAdd(flops, 2ull * (unsigned long long)(e_end - i0 < 8 ? e_end - i0 : 8) * q * q);
  if (t4 == 0 && pe.x >= 0) a.tab[(int64_t)pe.y * 40 + d] = (int32_t)(i0 + g);
  double* out[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t i = i0 + 2 * t4 + h;
    out[h] = i < e_end ? a.Pr + i * q : nullptr;
  }
  const int nrt = (q + 7) >> 3, nk4 = (q + 3) >> 2;
  const double* __restrict__ w = a.W + (int64_t)(pe.x >= 0 ? pe.x : 0) * q;
  for (int r0 = 0; r0 < nrt; r0 += 8) {
    double acc[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
    for (int k4 = 0; k4 < nk4; ++k4) {
      const int k = k4 * 4 + t4;
      const double b = (pe.x >= 0 && k < q) ? w[k] : 0.0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = (r0 + i) * 8 + g;
        if (r0 + i < nrt) {
          const double av = (r < q && k < q) ? __ldg(M + (int64_t)r * q + k) : 0.0;
          dmma884(acc[i][0], acc[i][1], av, b);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = (r0 + i) * 8 + g;
      if (r0 + i < nrt && r < q) {
        if (out[0]) out[0][r] = acc[i][0];
        if (out[1]) out[1][r] = acc[i][1];
      }
    }
  }
}

// S[slot][:] = ((0 + Pr[e_1]) + Pr[e_2]) + ... over the slot's entries in ascending offset
// order: the adds of the per-offset passes (which start from a zeroed scratch), same order.
// One warp per slot; the products of up to four entries are loaded before they are added.
__global__ void __launch_bounds__(256, 8) m2l_reduce_kernel(int64_t nslots, int q, const int32_t* __restrict__ tab,
                                                        const double* __restrict__ Pr, double* __restrict__ S) {
  const int64_t slot = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (slot >= nslots) return;
  const int32_t t0 = tab[slot * 40 + lane];
  const int32_t t1 = lane < 8 ? tab[slot * 40 + 32 + lane] : -1;
  const unsigned mask0 = __ballot_sync(0xffffffffu, t0 >= 0), mask1 = __ballot_sync(0xffffffffu, t1 >= 0);
  for (int rb = 0; rb < q; rb += 64) {  // 64 coefficients per sweep over the slot's entries
    unsigned m0 = mask0, m1 = mask1;
    const int r0 = rb + lane, r1 = rb + lane + 32;
    double acc0 = 0.0, acc1 = 0.0;
    while (m0 | m1) {
      int64_t idx[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        idx[k] = -1;
        if (m0) {
          const int dsel = __ffs(m0) - 1;
          m0 &= m0 - 1;
          idx[k] = __shfl_sync(0xffffffffu, t0, dsel);
        } else if (m1) {
          const int dsel = __ffs(m1) - 1;
          m1 &= m1 - 1;
          idx[k] = __shfl_sync(0xffffffffu, t1, dsel);
        }
      }
      double v0[4], v1[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        v0[k] = (idx[k] >= 0 && r0 < q) ? Pr[idx[k] * q + r0] : 0.0;
        v1[k] = (idx[k] >= 0 && r1 < q) ? Pr[idx[k] * q + r1] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (idx[k] >= 0) {
          acc0 += v0[k];
          acc1 += v1[k];
        }
    }
    if (r0 < q) S[slot * q + r0] = acc0;
    if (r1 < q) S[slot * q + r1] = acc1;
  }
}

// Pair-major M2L scratch S[T][j][a] -> box-major locals L[T][a][j] for the
// occupied boxes (CTA = box x 32-column chunk, smem-staged transpose).
constexpr int kTrCols = 32;
__global__ void __launch_bounds__(256) pair_to_box_kernel(const int32_t* __restrict__ occ, int q, int64_t n,
                                                          const double* __restrict__ S,
                                                          const int32_t* __restrict__ tmap, double* __restrict__ L) {
  extern __shared__ double tile[];  // kTrCols x (q + 1)
  const int64_t T = occ[blockIdx.x];
  const int64_t j0 = (int64_t)blockIdx.y * kTrCols;
  const int cw = (int)((n - j0) < kTrCols ? (n - j0) : kTrCols);
  const int qs = q + 1;
  for (int e = threadIdx.x; e < cw * q; e += blockDim.x) {
    const int jj = e / q, a = e % q;
    const int32_t slot = tmap[T * n + j0 + jj];
    tile[jj * qs + a] = slot >= 0 ? S[(int64_t)slot * q + a] : 0.0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < cw * q; e += blockDim.x) {
    int a = e / cw, jj = e % cw;
    L[(T * q + a) * n + j0 + jj] = tile[jj * qs + a];
  }
}

}  // namespace

int pair_to_box(const hikf_tree* t, int l, const double* S, const int32_t* tmap, int64_t n, double* L,
                cudaStream_t st) {
  if (t->n_occ[l] == 0 || n == 0) return HIKF_OK;
  const int q = t->orders[l] * t->orders[l];
  const size_t smem = sizeof(double) * kTrCols * (q + 1);
  static size_t configured = 0;
  if (smem > configured) {
    HIKF_CHECK_CUDA(cudaFuncSetAttribute(pair_to_box_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::max<size_t>(smem, 48 << 10)));
    configured = std::max<size_t>(smem, 48 << 10);
  }
  dim3 grid((unsigned)t->n_occ[l], (unsigned)((n + kTrCols - 1) / kTrCols));
  pair_to_box_kernel<<<grid, 256, smem, st>>>(t->occ[l], q, n, S, tmap, L);
  HIKF_CHECK_LAUNCH();
  return HIKF_OK;
}

namespace {

int grid_cap(int64_t n) {
  int64_t b = (n + kT - 1) / kT;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)num_sms() * 64));
}

}  // namespace

void pairs_free(PairLevel* p, cudaStream_t st) {
  if (p->key) cudaFreeAsync(p->key, st);
  if (p->W) cudaFreeAsync(p->W, st);
  if (p->np_dev) cudaFreeAsync(p->np_dev, st);
  *p = PairLevel();
}

int pairs_leaf(const hikf_tree* t, const SparseHt& s, PairLevel* out, cudaStream_t st, cudaEvent_t keys_ready) {
  *out = PairLevel();
  const int q = t->orders[t->depth] * t->orders[t->depth];
  out->np = s.ngroups;
  HIKF_TRY(aalloc(&out->key, s.ngroups, st));
  HIKF_TRY(aalloc(&out->W, s.ngroups * q, st));
  if (s.ngroups == 0) return HIKF_OK;
  leaf_pair_keys<<<grid_cap(s.ngroups), kT, 0, st>>>(s.ngroups, s.n, s.g_leaf, s.g_j, t->leaf_box, out->key);
  HIKF_CHECK_LAUNCH();
  if (keys_ready) HIKF_CHECK_CUDA(cudaEventRecord(keys_ready, st));
  p2m_pairs<<<grid_cap(s.ngroups * q), kT, 0, st>>>(s.ngroups, q, s.g_start, s.e_sp, s.e_v, t->W2s, out->W,
                                                     prof_flops_ptr(ST_P2M));
  HIKF_CHECK_LAUNCH();
  return HIKF_OK;
}

int pairs_keys(const hikf_tree* t, int l, int lc, const PairLevel& child, int64_t n, PairLevel* out, cudaStream_t st,
               bool deferred) {
  *out = PairLevel();
  const int64_t Gc = (int64_t)1 << lc, Gp = (int64_t)1 << l;
  if (child.np == 0) {
    HIKF_TRY(aalloc(&out->key, 1, st));
    return HIKF_OK;
  }
  int64_t *pk = nullptr, *pk_s = nullptr;
  int32_t* d_num = nullptr;
  HIKF_TRY(aalloc(&pk, child.np, st));
  HIKF_TRY(aalloc(&pk_s, child.np, st));
  HIKF_TRY(aalloc(&out->key, child.np, st));
  HIKF_TRY(aalloc(&d_num, 1, st));
  int end_bit = 1;
  while (end_bit < 62 && ((int64_t)1 << end_bit) <= Gp * Gp * n) ++end_bit;  // keys and the sentinel below 2^end_bit
  const int64_t sentinel = Gp * Gp * n;
  parent_keys<<<grid_cap(child.np), kT, 0, st>>>(child.np, child.np_dev, child.key, n, Gc, lc - l, sentinel, pk);
  HIKF_CHECK_LAUNCH();
  size_t b1 = 0, b2 = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, b1, pk, pk_s, (int)child.np, 0, end_bit, st);
  cub::DeviceSelect::Unique(nullptr, b2, pk_s, out->key, d_num, (int)child.np, st);
  void* tmp = nullptr;
  HIKF_CHECK_CUDA(cudaMallocAsync(&tmp, std::max<size_t>(std::max(b1, b2), 1), st));
  cub::DeviceRadixSort::SortKeys(tmp, b1, pk, pk_s, (int)child.np, 0, end_bit, st);
  cub::DeviceSelect::Unique(tmp, b2, pk_s, out->key, d_num, (int)child.np, st);
  if (child.np_dev) {
    drop_sentinel<<<1, 1, 0, st>>>(d_num, out->key, sentinel);
    HIKF_CHECK_LAUNCH();
  }
  if (deferred) {
    // no host read-back: the level is sized by its bound (ancestor pairs <= pairs, <= boxes x rays)
    // and its consumers read the count on the device
    out->np = std::min<int64_t>(child.np, Gp * Gp * n);
    out->np_dev = d_num;
  } else {
    int32_t np = 0;
    HIKF_CHECK_CUDA(cudaMemcpyAsync(&np, d_num, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    HIKF_CHECK_CUDA(cudaStreamSynchronize(st));
    out->np = np;
    cudaFreeAsync(d_num, st);
  }
  cudaFreeAsync(tmp, st);
  cudaFreeAsync(pk, st);
  cudaFreeAsync(pk_s, st);
  return HIKF_OK;
}

int pairs_m2m(const hikf_tree* t, int l, const PairLevel& child, int64_t n, PairLevel* out, cudaStream_t st) {
  const int64_t Gc = (int64_t)1 << (l + 1);
  const int qp = t->orders[l] * t->orders[l], qc = t->orders[l + 1] * t->orders[l + 1];
  HIKF_TRY(aalloc(&out->W, out->np * qp, st));
  if (out->np == 0 || child.np == 0) return HIKF_OK;
  int32_t* cidx = nullptr;
  HIKF_TRY(aalloc(&cidx, out->np * 4, st));
  HIKF_CHECK_CUDA(cudaMemsetAsync(cidx, 0xff, sizeof(int32_t) * out->np * 4, st));
  child_index<<<grid_cap(child.np), kT, 0, st>>>(child.np, child.np_dev, child.key, n, Gc, out->np, out->np_dev,
                                                out->key, cidx);
  HIKF_CHECK_LAUNCH();
  m2m_pairs<<<grid_cap(out->np * 32), kT, 0, st>>>(out->np, out->np_dev, qp, qc, t->shift[l], cidx, child.W, out->W,
                                                   prof_flops_ptr(ST_M2M));
  HIKF_CHECK_LAUNCH();
  cudaFreeAsync(cidx, st);
  return HIKF_OK;
}

namespace {

// flags[T * n + j] = 1 for every target of an active source pair (any of the 40 offsets)
// target (T * n + j) of source pair p at offset slot d, or -1 when the offset is not
// admissible for it (parent adjacency, bounds), T is empty, or outside [xlo, xhi]
__device__ __forceinline__ int64_t m2l_target_of(const int64_t* __restrict__ key, int64_t p, int d, int64_t n,
                                                 int64_t G, const uint8_t* __restrict__ occ, const M2LOffsets& offs,
                                                 int64_t xlo, int64_t xhi) {
  const int64_t S = key[p] / n, j = key[p] % n;
  const int dx = offs.dx[d], dy = offs.dy[d];
  const int64_t tx = S / G - dx, ty = S % G - dy;
  int64_t s2;
  if (tx >= xlo && tx <= xhi && tx >= 0 && ty >= 0 && tx < G && ty < G && m2l_source(tx, ty, dx, dy, G, s2) &&
      s2 == S && occ[tx * G + ty])
    return (tx * G + ty) * n + j;
  return -1;
}

// flags[T * n + j] = 1 for every target of an active source pair; eflag[d * np + p] = 1
// for every (offset, source pair) that has a target (offset-major)
// (np: allocated pairs = the stride of the (offset, pair) codes; np_dev: the actual count or null)
__global__ void m2l_mark_targets(int64_t np, const int32_t* __restrict__ np_dev, const int64_t* __restrict__ key,
                                 int64_t n, int64_t G, const uint8_t* __restrict__ occ, M2LOffsets offs, int64_t xlo,
                                 int64_t xhi, uint8_t* __restrict__ flags, uint8_t* __restrict__ eflag) {
  const int64_t nv = np_dev ? *np_dev : np;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < np * 40; e += (int64_t)gridDim.x * blockDim.x) {
    const int d = (int)(e / np);
    const int64_t p = e % np;
    const int64_t tk = p < nv ? m2l_target_of(key, p, d, n, G, occ, offs, xlo, xhi) : -1;
    if (tk >= 0) flags[tk] = 1;
    eflag[e] = tk >= 0 ? 1 : 0;
  }
}

// entries (source pair, target slot) of the selected (offset, pair) codes, and the
// first entry of every offset (codes are offset-major and ascending)
__global__ void m2l_entries(const int64_t* __restrict__ codes, const int32_t* __restrict__ count, int64_t np,
                            const int64_t* __restrict__ key, int64_t n, int64_t G, const uint8_t* __restrict__ occ,
                            M2LOffsets offs, int64_t xlo, int64_t xhi, const int32_t* __restrict__ tmap,
                            int2* __restrict__ ent) {
  const int64_t c = *count;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c; i += (int64_t)gridDim.x * blockDim.x) {
    const int d = (int)(codes[i] / np);
    const int64_t p = codes[i] % np;
    const int64_t tk = m2l_target_of(key, p, d, n, G, occ, offs, xlo, xhi);
    ent[i] = make_int2((int)p, tmap[tk]);
  }
}

__global__ void m2l_offset_starts(const int64_t* __restrict__ codes, const int32_t* __restrict__ count, int64_t np,
                                  int64_t* __restrict__ off) {
  const int d = threadIdx.x;
  if (d > 40) return;
  int64_t lo = 0, hi = *count;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (codes[mid] < (int64_t)d * np) lo = mid + 1; else hi = mid;
  }
  off[d] = lo;
}

__global__ void m2l_slots(const int64_t* __restrict__ keys, const int32_t* __restrict__ count,
                          int32_t* __restrict__ tmap) {
  const int64_t c = *count;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c; i += (int64_t)gridDim.x * blockDim.x)
    tmap[keys[i]] = (int32_t)i;
}

}  // namespace

int m2l_targets(const hikf_tree* t, int l, const PairLevel& src, int64_t n, int32_t* tmap, int32_t* count_dev,
                M2LPlan* plan, cudaStream_t st, int64_t xlo, int64_t xhi) {
  const int64_t G = (int64_t)1 << l;
  const int64_t total = G * G * n;
  *plan = M2LPlan();
  HIKF_CHECK_CUDA(cudaMemsetAsync(tmap, 0xff, sizeof(int32_t) * total, st));
  HIKF_CHECK_CUDA(cudaMemsetAsync(count_dev, 0, 2 * sizeof(int32_t), st));
  HIKF_TRY(aalloc(&plan->off, 41, st));
  HIKF_CHECK_CUDA(cudaMemsetAsync(plan->off, 0, 41 * sizeof(int64_t), st));
  if (src.np == 0 || total == 0) return HIKF_OK;
  if (total > INT32_MAX || src.np * 40 > INT32_MAX) {
    set_error("M2L target map of level %d too large (%lld entries)", l, (long long)total);
    return HIKF_BAD_ARGUMENT;
  }
  uint8_t *flags = nullptr, *eflag = nullptr;
  int64_t *keys = nullptr, *codes = nullptr;
  HIKF_TRY(aalloc(&flags, total, st));
  HIKF_TRY(aalloc(&eflag, src.np * 40, st));
  HIKF_CHECK_CUDA(cudaMemsetAsync(flags, 0, total, st));
  M2LOffsets offs;
  m2l_mark_targets<<<grid_cap(src.np * 40), kT, 0, st>>>(src.np, src.np_dev, src.key, n, G, t->occ_flag[l], offs, xlo,
                                                         xhi, flags, eflag);
  HIKF_CHECK_LAUNCH();
  // target slots (ascending T * n + j)
  const int64_t cap = std::min<int64_t>(total, src.np * 40);
  HIKF_TRY(aalloc(&keys, cap, st));
  HIKF_TRY(aalloc(&codes, src.np * 40, st));
  size_t tb = 0, tb2 = 0;
  cub::CountingInputIterator<int64_t> it(0);
  cub::DeviceSelect::Flagged(nullptr, tb, it, flags, keys, count_dev, (int)total, st);
  cub::DeviceSelect::Flagged(nullptr, tb2, it, eflag, codes, count_dev + 1, (int)(src.np * 40), st);
  void* tmp = nullptr;
  HIKF_CHECK_CUDA(cudaMallocAsync(&tmp, std::max<size_t>(std::max(tb, tb2), 1), st));
  cub::DeviceSelect::Flagged(tmp, tb, it, flags, keys, count_dev, (int)total, st);
  m2l_slots<<<grid_cap(cap), kT, 0, st>>>(keys, count_dev, tmap);
  HIKF_CHECK_LAUNCH();
  // the (source pair, target slot) entries of every offset, offset-major
  cub::DeviceSelect::Flagged(tmp, tb2, it, eflag, codes, count_dev + 1, (int)(src.np * 40), st);
  HIKF_TRY(aalloc(&plan->ent, src.np * 40, st));
  m2l_entries<<<grid_cap(src.np * 40), kT, 0, st>>>(codes, count_dev + 1, src.np, src.key, n, G, t->occ_flag[l], offs,
                                                    xlo, xhi, tmap, plan->ent);
  HIKF_CHECK_LAUNCH();
  m2l_offset_starts<<<1, 64, 0, st>>>(codes, count_dev + 1, src.np, plan->off);
  HIKF_CHECK_LAUNCH();
  cudaFreeAsync(tmp, st);
  cudaFreeAsync(keys, st);
  cudaFreeAsync(codes, st);
  cudaFreeAsync(eflag, st);
  cudaFreeAsync(flags, st);
  return HIKF_OK;
}

void m2l_plan_free(M2LPlan* plan, cudaStream_t st) {
  if (plan->ent) cudaFreeAsync(plan->ent, st);
  if (plan->off) cudaFreeAsync(plan->off, st);
  *plan = M2LPlan();
}

int m2l_products(const hikf_tree* t, int l, const PairLevel& src, const M2LPlan& plan, const int64_t* hoff,
                 int64_t nslots, double* S, cudaStream_t st) {
  const int q = t->orders[l] * t->orders[l];
  const int64_t nent = hoff[40];
  if (nslots <= 0 || nent <= 0) return HIKF_OK;
  if (nent > INT32_MAX) {
    set_error("M2L products of level %d: %lld entries do not fit 32-bit indices", l, (long long)nent);
    return HIKF_BAD_ARGUMENT;
  }
  M2LProd a{};
  a.ent = plan.ent;
  a.W = src.W;
  a.M = t->m2l[l];
  const bool inst = q == 4 || q == 9 || q == 16 || q == 25 || q == 36 || q == 49 || q == 64;
  // enough CTAs for every SM before a warp takes more than one group of 8 entries
  const int gpw = (inst && nent / 64 >= (int64_t)num_sms() * 24) ? 4 : 1;
  int64_t blocks = 0;
  for (int d = 0; d < 40; ++d) {
    a.off[d] = hoff[d];
    a.blk[d] = blocks;
    blocks += (hoff[d + 1] - hoff[d] + 64 * gpw - 1) / (64 * gpw);
  }
  a.off[40] = hoff[40];
  a.blk[40] = blocks;
  HIKF_TRY(aalloc(&a.Pr, nent * q, st));
  HIKF_TRY(aalloc(&a.tab, nslots * 40, st));
  HIKF_CHECK_CUDA(cudaMemsetAsync(a.tab, 0xff, sizeof(int32_t) * nslots * 40, st));
  const size_t smem = sizeof(double) * q * m2l_ld(q);
  unsigned long long* fl = prof_flops_ptr(ST_M2L);
#define HIKF_M2LP(QQ, K4, RT)                                                    \
  case QQ:                                                                      \
    m2l_prod_kernel<K4, RT><<<(unsigned)blocks, kT, smem, st>>>(a, q, gpw, fl); \
    break;
  switch (q) {
    HIKF_M2LP(4, 1, 1)
    HIKF_M2LP(9, 3, 2)
    HIKF_M2LP(16, 4, 2)
    HIKF_M2LP(25, 7, 4)
    HIKF_M2LP(36, 9, 5)
    HIKF_M2LP(49, 13, 7)
    HIKF_M2LP(64, 16, 8)
    default:
      m2l_prod_generic_kernel<<<(unsigned)blocks, kT, 0, st>>>(a, q, fl);
  }
#undef HIKF_M2LP
  HIKF_CHECK_LAUNCH();
  m2l_reduce_kernel<<<(unsigned)((nslots * 32 + kT - 1) / kT), kT, 0, st>>>(nslots, q, a.tab, a.Pr, S);
  HIKF_CHECK_LAUNCH();
  cudaFreeAsync(a.Pr, st);
  cudaFreeAsync(a.tab, st);
  return HIKF_OK;
}

bool m2l_list_supported(const hikf_tree* t, int l) {
  const int q = t->orders[l] * t->orders[l];
  return q >= 1 && q <= 256;  // instantiated kernels for orders 2..8, the generic product kernel above them
}

}  // namespace hikf

// 3D octree bbFMM for the cfg3 / cfg5 scenarios.
//
// PARITY UNPINNED: the reference is 2D and isotropic.  The algorithm is the
// direct 3D extension of fmm.py, restated in oracle/hikf_oracle3d.py (which is
// checked against the exact direct sum) -- see that file for the rules.  The
// anisotropic kernel variance exp(-|A (x - y)|^p) is handled by building the
// whole FMM on the scaled points A x with the isotropic unit kernel.
//
// Expansions are dense per level (box-major W[box][coeff][col]) and the
// product runs in column chunks of 64, so device memory stays bounded at cfg5
// (m = 2M).  Every transfer is a DMMA (m8n8k4 f64) warp GEMM: the operator
// sits in shared memory, each warp owns one (box, 8-column) output unit and
// streams its B fragments from global memory.
//
//   P2P   U[t] = sum over the 27 neighbour leaves of K(t, s) V[s]   (kernel block generated in smem)
//   P2M   W_D[leaf] = W2_leaf^T V_leaf
//   M2M   W_l[P] = sum_c S_c^T W_{l+1}[child c]
//   M2L   L_l[t] = sum over the offsets o valid for t's child class of M_o W_l[t + o]
//   L2L   L_l[t] += S_c L_{l-1}[parent]
//   L2P   U[p] += W2[p] L_D[leaf(p)]
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <numeric>
#include <vector>

#include "fmm3d.h"
#include "host_ops.h"
#include "prof.h"

struct hikf_tree3 {
  int64_t m = 0;
  int n = 0, q = 0, depth = 0;
  int64_t G = 1;
  double lo[3] = {0, 0, 0}, size = 0;
  hikf_kernel3 k{};
  // host copies (export / sizes)
  std::vector<int64_t> order_h, leaf_key_h;
  std::vector<int32_t> leaf_start_h, leaf_count_h;
  int32_t max_count = 0;
  // device
  double* pts = nullptr;  // m x 3 scaled, sorted (leaf) order
  int64_t* order = nullptr;
  int64_t* leaf_key = nullptr;
  int32_t *leaf_start = nullptr, *leaf_count = nullptr, *box2leaf = nullptr;
  double* W2 = nullptr;      // m x q, sorted order
  double* shift = nullptr;   // 8 x q x q: [c][child coeff][parent coeff]
  double* shiftT = nullptr;  // 8 x q x q: [c][parent coeff][child coeff]
  double* m2l[hikf::kMaxDepth + 1] = {nullptr};  // 316 x q x q per level
};

namespace hikf {

namespace {

// trivially-copyable view of the tree for kernel arguments
struct T3v {
  int64_t m, G;
  int n, q, max_count;
  hikf_kernel3 k;
  const double* pts;
  const int64_t *order, *leaf_key;
  const int32_t *leaf_start, *leaf_count, *box2leaf;
  const double* W2;
};

T3v view(const hikf_tree3* t) {
  return T3v{t->m, t->G, t->n, t->q, t->max_count, t->k, t->pts, t->order, t->leaf_key,
             t->leaf_start, t->leaf_count, t->box2leaf, t->W2};
}

constexpr int T3 = 256;    // threads per CTA (8 warps)
constexpr int MAXRT = 16;  // row tiles per warp unit (rows <= 128)
constexpr int KC = 64;     // columns per chunk
constexpr int NOFF = 316;  // M2L offsets in [-3, 3]^3 with max |o| >= 2

__host__ __device__ inline int pad4(int k) { return k + ((4 - k % 16) + 16) % 16; }  // == 4 mod 16

__device__ __forceinline__ double k3_of_r(int family, double variance, double r) {
  const double t = family == HIKF_GAUSSIAN ? __dmul_rn(r, r) : r;
  return __dmul_rn(variance, exp(-t));
}

__device__ __forceinline__ double d3(double ax, double ay, double az, double bx, double by, double bz) {
  const double dx = __dsub_rn(ax, bx), dy = __dsub_rn(ay, by), dz = __dsub_rn(az, bz);
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
}

__host__ __device__ inline int64_t box_coord3(double x, double lo, double h, int64_t G) {
  const double u = (x - lo) / h;
  int64_t b = (int64_t)floor(u);
  if ((double)b == u && b > 0) --b;  // split plane -> low box
  return b < 0 ? 0 : (b > G - 1 ? G - 1 : b);
}

void offsets3(int o[NOFF][3]) {
  int k = 0;
  for (int a = -3; a <= 3; ++a)
    for (int b = -3; b <= 3; ++b)
      for (int c = -3; c <= 3; ++c)
        if (std::max(std::abs(a), std::max(std::abs(b), std::abs(c))) >= 2) {
          o[k][0] = a;
          o[k][1] = b;
          o[k][2] = c;
          ++k;
        }
}

// ---- W2[p][(ix n + iy) n + iz] = S_ix(xi) S_iy(eta) S_iz(zeta), sorted order ----
__global__ void interp3_kernel(const double* __restrict__ pts, int64_t m, double lo0, double lo1, double lo2,
                               double h, int64_t G, int n, const double* __restrict__ Tn, double* __restrict__ W2) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
    double w[3][12];
    for (int d = 0; d < 3; ++d) {
      const double x = pts[3 * p + d], lo = d == 0 ? lo0 : (d == 1 ? lo1 : lo2);
      const int64_t b = box_coord3(x, lo, h, G);
      const double ctr = __dadd_rn(lo, __dmul_rn(__dadd_rn((double)b, 0.5), h));
      const double xi = __ddiv_rn(__dsub_rn(x, ctr), __ddiv_rn(h, 2.0));
      double T[12];
      T[0] = 1.0;
      if (n > 1) T[1] = xi;
      const double two_x = __dmul_rn(2.0, xi);
      for (int j = 2; j < n; ++j) T[j] = __dsub_rn(__dmul_rn(two_x, T[j - 1]), T[j - 2]);
      for (int k = 0; k < n; ++k) {
        double dot = 0.0;
        for (int j = 1; j < n; ++j) dot = __dadd_rn(dot, __dmul_rn(T[j], Tn[k * n + j]));
        w[d][k] = __ddiv_rn(__dadd_rn(1.0, __dmul_rn(2.0, dot)), (double)n);
      }
    }
    double* out = W2 + p * (int64_t)(n * n * n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        for (int l = 0; l < n; ++l) out[(i * n + j) * n + l] = __dmul_rn(__dmul_rn(w[0][i], w[1][j]), w[2][l]);
  }
}

// ---- M2L operators of one level: M[o][a][b] = K(|t_a - (o h + t_b)|), t = nodes3 h / 2 ----
__global__ void m2l3_ops_kernel(int n, double h, const double* __restrict__ nodes, const int* __restrict__ offs,
                                int family, double variance, double* __restrict__ ops) {
  const int q = n * n * n;
  const int64_t total = (int64_t)NOFF * q * q;
  const double hh = __ddiv_rn(h, 2.0);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int o = (int)(e / ((int64_t)q * q));
    const int ab = (int)(e % ((int64_t)q * q)), a = ab / q, b = ab % q;
    const double ta[3] = {__dmul_rn(nodes[a / (n * n)], hh), __dmul_rn(nodes[(a / n) % n], hh),
                          __dmul_rn(nodes[a % n], hh)};
    double sb[3];
    const int bi[3] = {b / (n * n), (b / n) % n, b % n};
    for (int d = 0; d < 3; ++d)
      sb[d] = __dadd_rn(__dmul_rn(nodes[bi[d]], hh), __dmul_rn((double)offs[3 * o + d], h));
    ops[e] = k3_of_r(family, variance, d3(ta[0], ta[1], ta[2], sb[0], sb[1], sb[2]));
  }
}

// ---- warp GEMM core: acc[rt] (+)= A[rt*8 + g][k] * B[k][j0 + g], k < nk4 * 4 ----
// The B fragments (global loads) are fetched 8 k-steps at a time ahead of
// their DMMAs, so a batch pays one memory latency instead of eight.
template <class BFrag>
__device__ __forceinline__ void warp_gemm(const double* As, int lda, int nrt, int nk4, int gq, int t4, BFrag bf,
                                          double (&acc)[MAXRT][2]) {
  constexpr int KB = 8;
  for (int kb = 0; kb < nk4; kb += KB) {
    double b[KB];
#pragma unroll
    for (int i = 0; i < KB; ++i) b[i] = kb + i < nk4 ? bf((kb + i) * 4 + t4) : 0.0;
#pragma unroll
    for (int i = 0; i < KB; ++i) {
      if (kb + i >= nk4) break;
      const int k4 = kb + i;
#pragma unroll
      for (int rt = 0; rt < MAXRT; ++rt)
        if (rt < nrt) dmma884(acc[rt][0], acc[rt][1], As[(rt * 8 + gq) * lda + k4 * 4 + t4], b[i]);
    }
  }
}

__device__ __forceinline__ void zero_acc(double (&acc)[MAXRT][2]) {
#pragma unroll
  for (int rt = 0; rt < MAXRT; ++rt) acc[rt][0] = acc[rt][1] = 0.0;
}

// load a rows x cols block (row-major, element (r, c) = src(r, c)) into smem, zero-padded to
// prow x pcol with leading dimension lda
template <class Src>
__device__ __forceinline__ void load_A(double* As, int lda, int prow, int pcol, int rows, int cols, Src src) {
  for (int e = threadIdx.x; e < prow * pcol; e += blockDim.x) {
    const int r = e / pcol, c = e % pcol;
    As[r * lda + c] = (r < rows && c < cols) ? src(r, c) : 0.0;
  }
}

struct Chunk {
  const double* V;  // m x ldv, original order (this chunk's first column at V)
  int64_t ldv;
  int kc;           // columns in this chunk
  double* U;        // m x ldu, original order
  int64_t ldu;
  unsigned long long* flops;  // performed-flop counter of the stage (profiling on), or null
};

// one atomic per CTA: thread 0's tally of the flops the CTA performed
__device__ __forceinline__ void count_flops(unsigned long long* c, unsigned long long v) {
  if (c && threadIdx.x == 0 && v) atomicAdd(c, v);
}

// ---- P2P: U[t] = sum_nbr K(t, s) V[s] (first write of the chunk's U columns) ----
__global__ void __launch_bounds__(T3, 2) p2p3_kernel(const T3v t, Chunk ch, const uint8_t* __restrict__ leafnz) {
  // the kernel block K(target, source) is built in shared memory 64 target rows at a
  // time (~68 KB: 2 CTAs per SM, one CTA's exp / sqrt build overlaps the other's DMMAs)
  extern __shared__ double As[];
  constexpr int TR = 64;
  const int leaf = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, gq = lane >> 2, t4 = lane & 3;
  const int ts = t.leaf_start[leaf], tc = t.leaf_count[leaf];
  const int64_t key = t.leaf_key[leaf], G = t.G;
  const int64_t bx = key / (G * G), by = (key / G) % G, bz = key % G;
  const int lda = pad4(((t.max_count + 3) / 4) * 4);
  const int j0 = warp * 8;  // this warp's 8 columns of the chunk (kc <= 64)
  double acc[MAXRT][2];
  zero_acc(acc);
  unsigned long long done = 0;
  for (int s = 0; s < 27; ++s) {
    const int64_t x = bx + s / 9 - 1, y = by + (s / 3) % 3 - 1, z = bz + s % 3 - 1;
    if (x < 0 || y < 0 || z < 0 || x >= G || y >= G || z >= G) continue;
    const int sl = t.box2leaf[(x * G + y) * G + z];
    if (sl < 0 || !leafnz[sl]) continue;  // no leaf / all-zero charges: uniform across the CTA
    const int ss = t.leaf_start[sl], sc = t.leaf_count[sl];
    const bool mine = j0 < ch.kc && ((leafnz[sl] >> warp) & 1);  // this warp's 8 columns hold a nonzero charge
    if (mine) done += 2ull * tc * sc * min(8, ch.kc - j0);
    const int jc = j0 + gq, nk4 = (sc + 3) / 4;
    static_assert(2 * TR >= MAXRT * 8, "two row blocks cover a leaf");
    for (int r0 = 0; r0 < tc; r0 += TR) {
      const int nr = min(TR, tc - r0), nrt = (nr + 7) >> 3;
      __syncthreads();
      load_A(As, lda, nrt * 8, nk4 * 4, nr, sc, [&](int r, int c) {
        const double* a = t.pts + 3 * (int64_t)(ts + r0 + r);
        const double* b = t.pts + 3 * (int64_t)(ss + c);
        return k3_of_r(t.k.family, t.k.variance, d3(a[0], a[1], a[2], b[0], b[1], b[2]));
      });
      __syncthreads();
      if (!mine) continue;
      for (int k4 = 0; k4 < nk4; ++k4) {
        const int k = k4 * 4 + t4;
        const double b = (k < sc && jc < ch.kc) ? ch.V[t.order[ss + k] * ch.ldv + jc] : 0.0;
        if (r0 == 0) {  // static accumulator indices: rows 0..63 -> acc[0..7], 64..127 -> acc[8..15]
#pragma unroll
          for (int rt = 0; rt < TR / 8; ++rt)
            if (rt < nrt) dmma884(acc[rt][0], acc[rt][1], As[(rt * 8 + gq) * lda + k4 * 4 + t4], b);
        } else {
#pragma unroll
          for (int rt = 0; rt < TR / 8; ++rt)
            if (rt < nrt) dmma884(acc[TR / 8 + rt][0], acc[TR / 8 + rt][1], As[(rt * 8 + gq) * lda + k4 * 4 + t4], b);
        }
      }
    }
  }
  if (ch.flops && lane == 0 && done) atomicAdd(ch.flops, done);
  if (j0 >= ch.kc) return;
  const int nrt = (tc + 7) >> 3;
#pragma unroll
  for (int rt = 0; rt < MAXRT; ++rt) {
    const int r = rt * 8 + gq;
    if (rt >= nrt || r >= tc) continue;
    double* urow = ch.U + t.order[ts + r] * ch.ldu;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int c = j0 + 2 * t4 + hh;
      if (c < ch.kc) urow[c] = acc[rt][hh];
    }
  }
}

// Leaf operators stage W2 (points x q, row-major as stored: coalesced loads) in
// blocks of LP = 64 points, ~68 KB of shared memory, so 3 CTAs share an SM and
// one CTA's staging overlaps another's DMMAs.
constexpr int LP = 64;
__host__ __device__ inline int w2_ld(int q) { return pad4(((q + 3) / 4) * 4); }  // == 4 mod 16 doubles

// ---- P2M: W_D[box(leaf)] = W2_leaf^T V_leaf; A[a][p] = W2[p][a] read transposed from the
// staged W2 block (conflict-free: the row stride is 4 mod 16 doubles) ----
__global__ void __launch_bounds__(T3, 3) p2m3_kernel(const T3v t, Chunk ch, double* __restrict__ W,
                                                     const uint8_t* __restrict__ leafnz) {
  extern __shared__ double As[];
  const int leaf = blockIdx.x;
  if (!leafnz[leaf]) return;  // W stays zero (memset)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, gq = lane >> 2, t4 = lane & 3;
  const int ts = t.leaf_start[leaf], tc = t.leaf_count[leaf], q = t.q;
  const int nrt = (q + 7) >> 3, ld = w2_ld(q);
  const int j0 = warp * 8, jc = j0 + gq;
  const bool mine = j0 < ch.kc && ((leafnz[leaf] >> warp) & 1);
  if (mine && ch.flops && lane == 0) atomicAdd(ch.flops, 2ull * q * tc * min(8, ch.kc - j0));
  double acc[MAXRT][2];
  zero_acc(acc);
  for (int p0 = 0; p0 < tc; p0 += LP) {
    const int np = min(LP, tc - p0);
    __syncthreads();
    for (int e = threadIdx.x; e < LP * ld; e += T3) {
      const int p = e / ld, a = e % ld;
      As[e] = (p < np && a < q) ? t.W2[(int64_t)(ts + p0 + p) * q + a] : 0.0;
    }
    __syncthreads();
    if (!mine) continue;
    const int nk4 = (np + 3) / 4;
    for (int k4 = 0; k4 < nk4; ++k4) {
      const int p = k4 * 4 + t4;
      const double b = (p < np && jc < ch.kc) ? ch.V[t.order[ts + p0 + p] * ch.ldv + jc] : 0.0;
#pragma unroll
      for (int rt = 0; rt < MAXRT; ++rt)
        if (rt < nrt) dmma884(acc[rt][0], acc[rt][1], As[p * ld + rt * 8 + gq], b);
    }
  }
  if (!mine) return;  // W stays zero (memset) for all-zero columns
  double* out = W + t.leaf_key[leaf] * (int64_t)q * KC;
#pragma unroll
  for (int rt = 0; rt < MAXRT; ++rt) {
    const int a = rt * 8 + gq;
    if (rt >= nrt || a >= q) continue;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) out[(int64_t)a * KC + j0 + 2 * t4 + hh] = acc[rt][hh];
  }
}

// ---- L2P: U[p] += W2[p] L_D[box(leaf)], LP points per pass ----
__global__ void __launch_bounds__(T3, 3) l2p3_kernel(const T3v t, Chunk ch, const double* __restrict__ L) {
  extern __shared__ double As[];
  const int leaf = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, gq = lane >> 2, t4 = lane & 3;
  const int ts = t.leaf_start[leaf], tc = t.leaf_count[leaf], q = t.q;
  count_flops(ch.flops, 2ull * tc * q * ch.kc);
  const int ld = w2_ld(q), nk4 = (q + 3) / 4;
  const int j0 = warp * 8, jc = j0 + gq;
  const double* Lb = L + t.leaf_key[leaf] * (int64_t)q * KC;
  for (int p0 = 0; p0 < tc; p0 += LP) {
    const int np = min(LP, tc - p0), nrt = (np + 7) >> 3;
    __syncthreads();
    for (int e = threadIdx.x; e < LP * ld; e += T3) {
      const int p = e / ld, a = e % ld;
      As[e] = (p < np && a < q) ? t.W2[(int64_t)(ts + p0 + p) * q + a] : 0.0;
    }
    __syncthreads();
    if (j0 >= ch.kc) continue;
    double acc[LP / 8][2];
#pragma unroll
    for (int rt = 0; rt < LP / 8; ++rt) acc[rt][0] = acc[rt][1] = 0.0;
    for (int k4 = 0; k4 < nk4; ++k4) {
      const int k = k4 * 4 + t4;
      const double b = (k < q && jc < ch.kc) ? Lb[(int64_t)k * KC + jc] : 0.0;  // L1 hit on the second pass
#pragma unroll
      for (int rt = 0; rt < LP / 8; ++rt)
        if (rt < nrt) dmma884(acc[rt][0], acc[rt][1], As[(rt * 8 + gq) * ld + k4 * 4 + t4], b);
    }
#pragma unroll
    for (int rt = 0; rt < LP / 8; ++rt) {
      const int r = rt * 8 + gq;
      if (rt >= nrt || r >= np) continue;
      double* urow = ch.U + t.order[ts + p0 + r] * ch.ldu;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int c = j0 + 2 * t4 + hh;
        if (c < ch.kc) urow[c] += acc[rt][hh];  // U = near + far
      }
    }
  }
}

// ---- box operators: M2M / M2L / L2L, one CTA = 8 output boxes of one child class ----
enum { OP_M2M = 0, OP_M2L = 1, OP_L2L = 2 };

struct BoxOpArgs {
  int mode, q, lev;          // lev = level of the output boxes
  int cls;                   // child class (cx cy cz bits) for M2L / L2L
  int64_t Gout;              // boxes per axis at the output level
  const double* in;          // source expansions (level lev for M2L, lev + 1 for M2M, lev - 1 for L2L)
  double* out;               // output expansions (level lev)
  const double* ops;         // M2L: 316 x q x q; M2M: shiftT (8 x q x q); L2L: shift (8 x q x q)
  const int* offs;           // M2L: 316 x 3
  int kc;
  const uint8_t* nz;         // M2L: per source box, 1 if its expansion has a nonzero in this chunk
  const uint8_t* occ;        // M2L / L2L: per output box, 1 if any point lies below it (else skipped:
                             // its locals are never read -- L2L children and L2P leaves are occupied)
  unsigned long long* flops; // performed-flop counter (profiling on), or null
};

// occupancy of the boxes of each level: occ_D[box] = has a leaf; occ_l = OR of the 8 children
__global__ void occ_leaf(const int32_t* __restrict__ box2leaf, int64_t nb, uint8_t* __restrict__ occ) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x)
    occ[b] = box2leaf[b] >= 0 ? 1 : 0;
}
__global__ void occ_parent(const uint8_t* __restrict__ occc, int64_t G, uint8_t* __restrict__ occp) {
  const int64_t nb = G * G * G, Gc = 2 * G;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = b / (G * G), y = (b / G) % G, z = b % G;
    uint8_t o = 0;
    for (int c = 0; c < 8; ++c)
      o |= occc[((2 * x + ((c >> 2) & 1)) * Gc + (2 * y + ((c >> 1) & 1))) * Gc + (2 * z + (c & 1))];
    occp[b] = o;
  }
}

// leafnz[l] = per-warp mask of any(V[order[p]][j] != 0) over the leaf's points p and the warp's 8
// columns: P2P / P2M skip all-zero source leaves per CTA and per warp (exact: they contribute zeros)
__global__ void nonzero_leaves(const T3v t, const double* __restrict__ V, int64_t ldv, int kc, int64_t nl,
                               uint8_t* __restrict__ nz) {
  const int64_t leaf = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (leaf >= nl) return;
  const int ts = t.leaf_start[leaf], tc = t.leaf_count[leaf];
  // bit w: some charge in columns 8w .. 8w + 7 (warp w's columns in the leaf / box kernels)
  unsigned mask = 0;
  for (int e = lane; e < tc * kc; e += 32)
    if (V[t.order[ts + e / kc] * ldv + e % kc] != 0.0) mask |= 1u << ((e % kc) >> 3);
  mask = __reduce_or_sync(0xffffffffu, mask);
  if (lane == 0) nz[leaf] = (uint8_t)mask;
}

// nz masks without scanning the dense expansions: leaf boxes take their leaf's charge mask (a
// superset of the nonzero groups of W_D), parents the OR of their children; empty boxes 0
__global__ void nz_leaf_boxes(const int64_t* __restrict__ leaf_key, const uint8_t* __restrict__ lnz, int64_t nl,
                              uint8_t* __restrict__ nz) {
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < nl; l += (int64_t)gridDim.x * blockDim.x)
    nz[leaf_key[l]] = lnz[l];
}
__global__ void nz_parent(const uint8_t* __restrict__ nzc, int64_t G, uint8_t* __restrict__ nzp) {
  const int64_t nb = G * G * G, Gc = 2 * G;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = b / (G * G), y = (b / G) % G, z = b % G;
    uint8_t o = 0;
    for (int c = 0; c < 8; ++c)
      o |= nzc[((2 * x + ((c >> 2) & 1)) * Gc + (2 * y + ((c >> 1) & 1))) * Gc + (2 * z + (c & 1))];
    nzp[b] = o;
  }
}


// one CTA = one output box; warp w owns chunk columns 8w .. 8w + 7.  The
// operators stream through shared memory in K-slices of 32 with a two-slot
// cp.async ring, so the next slice (of this term or the next valid term)
// loads while the current one is multiplied.
constexpr int KS = 32;                    // k per slice
constexpr int KLD = KS + 4;               // == 4 mod 16 doubles
constexpr int SLICE = MAXRT * 8 * KLD;    // doubles per slot (128 rows)

__global__ void __launch_bounds__(T3, 2) boxop3_kernel(BoxOpArgs g) {
  extern __shared__ double As[];  // 2 slots
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, gq = lane >> 2, t4 = lane & 3;
  const int q = g.q, nrt = (q + 7) >> 3, nslices = (q + KS - 1) / KS;
  const int64_t G = g.Gout;
  // M2L / L2L launch all 8 child classes at once: blockIdx.x = class * parents + parent
  const int64_t nunit = g.mode == OP_M2M ? (int64_t)gridDim.x : (int64_t)gridDim.x / 8;
  const int64_t unit = blockIdx.x % nunit;
  const int cls = g.mode == OP_M2M ? 0 : (int)(blockIdx.x / nunit);
  int64_t ox, oy, oz;
  if (g.mode == OP_M2M) {
    ox = unit / (G * G);
    oy = (unit / G) % G;
    oz = unit % G;
  } else {  // the class-c child of parent `unit`
    const int64_t Gp = G / 2;
    const int64_t px = unit / (Gp * Gp), py = (unit / Gp) % Gp, pz = unit % Gp;
    ox = 2 * px + ((cls >> 2) & 1);
    oy = 2 * py + ((cls >> 1) & 1);
    oz = 2 * pz + (cls & 1);
  }
  const int64_t obox = (ox * G + oy) * G + oz;
  if (g.occ && !g.occ[obox]) return;  // empty output box (CTA-uniform, before any barrier)
  const int nterms = g.mode == OP_M2L ? NOFF : (g.mode == OP_M2M ? 8 : 1);
  // term -> (operator, source box); -1 when the term does not apply (CTA-uniform)
  auto term_src = [&](int term, const double** A) -> int64_t {
    if (g.mode == OP_M2L) {
      const int dx = g.offs[3 * term], dy = g.offs[3 * term + 1], dz = g.offs[3 * term + 2];
      // parents adjacent per axis (fmm.py:301-302); floor((c + d) / 2) is the parent offset
      const int cx = (cls >> 2) & 1, cy = (cls >> 1) & 1, cz = cls & 1;
      const int pdx = (cx + dx) >> 1, pdy = (cy + dy) >> 1, pdz = (cz + dz) >> 1;
      if (pdx < -1 || pdx > 1 || pdy < -1 || pdy > 1 || pdz < -1 || pdz > 1) return -1;
      const int64_t sx = ox + dx, sy = oy + dy, sz = oz + dz;
      if (sx < 0 || sy < 0 || sz < 0 || sx >= G || sy >= G || sz >= G) return -1;
      const int64_t sb = (sx * G + sy) * G + sz;
      if (g.nz && !g.nz[sb]) return -1;  // all-zero source expansion
      *A = g.ops + (int64_t)term * q * q;
      return sb;
    }
    if (g.mode == OP_M2M) {
      const int64_t Gc = 2 * G;
      const int64_t cx = 2 * ox + ((term >> 2) & 1), cy = 2 * oy + ((term >> 1) & 1), cz = 2 * oz + (term & 1);
      const int64_t cb = (cx * Gc + cy) * Gc + cz;
      if (g.nz && !g.nz[cb]) return -1;  // all-zero child expansion
      *A = g.ops + (int64_t)term * q * q;  // shiftT[c]: parent coeff x child coeff
      return cb;
    }
    const int64_t Gp = G / 2;
    *A = g.ops + (int64_t)cls * q * q;  // shift[c]: child coeff x parent coeff
    return ((ox >> 1) * Gp + (oy >> 1)) * Gp + (oz >> 1);
  };
  auto next_term = [&](int from) {
    const double* A;
    for (int t = from; t < nterms; ++t)
      if (term_src(t, &A) >= 0) return t;
    return nterms;
  };
  // issue the copy of slice `sl` of term `term`'s operator into slot `slot` (zero-filled padding)
  auto issue = [&](int term, int sl, int slot) {
    const double* A;
    term_src(term, &A);
    double* dst = As + slot * SLICE;
    const int k0 = sl * KS;
    for (int e = threadIdx.x; e < MAXRT * 8 * KS; e += T3) {
      const int r = e / KS, k = e % KS;
      const bool ok = r < q && k0 + k < q;
      cp_async8(dst + r * KLD + k, ok ? A + (int64_t)r * q + k0 + k : A, ok);
    }
  };
  const int j0 = warp * 8, jc = j0 + gq;
  double acc[MAXRT][2];
  zero_acc(acc);
  int term = next_term(0), sl = 0, slot = 0;
  if (term < nterms) issue(term, 0, 0);
  cp_async_commit();
  unsigned long long done = 0;
  // this warp's part of a term: M2L / M2M skip the 8 columns that are all zero in the source
  auto mine = [&](int tm) -> bool {
    if (g.mode == OP_L2L || !g.nz) return true;
    const double* A;
    return (g.nz[term_src(tm, &A)] >> warp) & 1;
  };
  // B fragments of a slice (this lane's column jc, k = k0 + 4 k4 + t4), one register per
  // k-step; the next slice's are loaded while this slice's DMMAs run
  constexpr int NK4S = KS / 4;
  auto load_bs = [&](int tm, int s, double (&b)[NK4S]) {
    const double* Aop;
    const int64_t sbox = term_src(tm, &Aop);
    const double* B = g.in + sbox * (int64_t)q * KC;
    const int k0 = s * KS;
#pragma unroll
    for (int k4 = 0; k4 < NK4S; ++k4) {
      const int k = k0 + k4 * 4 + t4;
      b[k4] = (k < q && jc < g.kc) ? B[(int64_t)k * KC + jc] : 0.0;
    }
  };
  double bcur[NK4S];
  bool mcur = term < nterms && j0 < g.kc && mine(term);
  if (mcur) load_bs(term, 0, bcur);
  while (term < nterms) {
    if (sl == 0 && mcur) done += 2ull * q * q * min(8, g.kc - j0);
    // next step (slice of this term, or the first slice of the next valid term)
    int nterm = term, nsl = sl + 1;
    if (nsl == nslices) {
      nterm = next_term(term + 1);
      nsl = 0;
    }
    if (nterm < nterms) issue(nterm, nsl, slot ^ 1);
    cp_async_commit();
    double bnext[NK4S];
    const bool mnext = nterm < nterms && j0 < g.kc && (nterm == term ? mcur : mine(nterm));
    if (mnext) load_bs(nterm, nsl, bnext);
    cp_async_wait<1>();
    __syncthreads();
    if (mcur) {
      const double* Asl = As + slot * SLICE;
      const int k0 = sl * KS;
      const int nk4 = (min(KS, q - k0) + 3) / 4;
#pragma unroll
      for (int k4 = 0; k4 < NK4S; ++k4) {
        if (k4 >= nk4) break;
#pragma unroll
        for (int rt = 0; rt < MAXRT; ++rt)
          if (rt < nrt) dmma884(acc[rt][0], acc[rt][1], Asl[(rt * 8 + gq) * KLD + k4 * 4 + t4], bcur[k4]);
      }
    }
    __syncthreads();  // everyone is done with `slot` before it is refilled
#pragma unroll
    for (int k4 = 0; k4 < NK4S; ++k4) bcur[k4] = bnext[k4];
    mcur = mnext;
    term = nterm;
    sl = nsl;
    slot ^= 1;
  }
  cp_async_wait<0>();
  if (g.flops && lane == 0 && done) atomicAdd(g.flops, done);
  if (j0 >= g.kc) return;
  double* O = g.out + obox * (int64_t)q * KC;
#pragma unroll
  for (int rt = 0; rt < MAXRT; ++rt) {
    const int a = rt * 8 + gq;
    if (rt >= nrt || a >= q) continue;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int c = j0 + 2 * t4 + hh;
      if (c >= g.kc) continue;
      if (g.mode == OP_L2L)
        O[(int64_t)a * KC + c] += acc[rt][hh];  // L = M2L sum + L2L
      else
        O[(int64_t)a * KC + c] = acc[rt][hh];
    }
  }
}


// ---- M2L, row-split: one CTA per (output box, 8-column group of the chunk) ----
// The 8 warps split the q output rows (RTW row tiles each) and read their rows
// of each operator straight from L2 (no shared-memory staging, no barriers), so
// a term costs operator traffic only for the column groups whose source
// expansion is nonzero.  The B fragments (the source's 8 columns) are the same
// for all warps (L1 hits after the first).
template <int RTW, int G2>
__global__ void __launch_bounds__(T3) m2l3_rows_kernel(BoxOpArgs g) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, gq = lane >> 2, t4 = lane & 3;
  const int q = g.q, nk4 = (q + 3) / 4;
  const int64_t G = g.Gout, Gp = G / 2;
  constexpr int NGB = KC / 8 / G2;  // blocks of G2 column groups per chunk
  const int gb = blockIdx.x % NGB;
  const int64_t rest = blockIdx.x / NGB;
  const int64_t nunit = (int64_t)(gridDim.x / NGB) / 8;
  const int64_t unit = rest % nunit;
  const int cls = (int)(rest / nunit);
  const int j0 = gb * G2 * 8;
  if (j0 >= g.kc) return;
  const int64_t px = unit / (Gp * Gp), py = (unit / Gp) % Gp, pz = unit % Gp;
  const int64_t ox = 2 * px + ((cls >> 2) & 1), oy = 2 * py + ((cls >> 1) & 1), oz = 2 * pz + (cls & 1);
  const int64_t obox = (ox * G + oy) * G + oz;
  if (g.occ && !g.occ[obox]) return;
  const int cx = (cls >> 2) & 1, cy = (cls >> 1) & 1, cz = cls & 1;
  double acc[RTW][G2][2];
#pragma unroll
  for (int i = 0; i < RTW; ++i)
#pragma unroll
    for (int c = 0; c < G2; ++c) acc[i][c][0] = acc[i][c][1] = 0.0;
  unsigned long long done = 0;
  for (int term = 0; term < NOFF; ++term) {
    const int dx = g.offs[3 * term], dy = g.offs[3 * term + 1], dz = g.offs[3 * term + 2];
    const int pdx = (cx + dx) >> 1, pdy = (cy + dy) >> 1, pdz = (cz + dz) >> 1;
    if (pdx < -1 || pdx > 1 || pdy < -1 || pdy > 1 || pdz < -1 || pdz > 1) continue;
    const int64_t sx = ox + dx, sy = oy + dy, sz = oz + dz;
    if (sx < 0 || sy < 0 || sz < 0 || sx >= G || sy >= G || sz >= G) continue;
    const int64_t sb = (sx * G + sy) * G + sz;
    // active column groups of this block (CTA-uniform): the source's nonzero 8-column groups
    const unsigned act = g.nz ? ((unsigned)g.nz[sb] >> (gb * G2)) & ((1u << G2) - 1) : (1u << G2) - 1;
    if (!act) continue;
    const double* A = g.ops + (int64_t)term * q * q;
    const double* B = g.in + sb * (int64_t)q * KC;
#pragma unroll
    for (int c = 0; c < G2; ++c)
      if ((act >> c) & 1) done += 2ull * q * q * max(0, min(8, g.kc - j0 - 8 * c));
    constexpr int KB = 8;  // k-steps per batch of loads
    for (int kb = 0; kb < nk4; kb += KB) {
      double b[KB][G2], a[KB][RTW];
#pragma unroll
      for (int i = 0; i < KB; ++i) {
        const int k = (kb + i) * 4 + t4;
        const bool ok = kb + i < nk4 && k < q;
#pragma unroll
        for (int c = 0; c < G2; ++c) {
          const int jc = j0 + 8 * c + gq;
          b[i][c] = ok && ((act >> c) & 1) && jc < g.kc ? __ldg(B + (int64_t)k * KC + jc) : 0.0;
        }
#pragma unroll
        for (int r = 0; r < RTW; ++r) {
          const int row = (warp * RTW + r) * 8 + gq;
          a[i][r] = ok && row < q ? __ldg(A + (int64_t)row * q + k) : 0.0;
        }
      }
#pragma unroll
      for (int i = 0; i < KB; ++i)
#pragma unroll
        for (int c = 0; c < G2; ++c)
          if ((act >> c) & 1)
#pragma unroll
            for (int r = 0; r < RTW; ++r) dmma884(acc[r][c][0], acc[r][c][1], a[i][r], b[i][c]);
    }
  }
  if (g.flops && threadIdx.x == 0 && done) atomicAdd(g.flops, done);
  double* O = g.out + obox * (int64_t)q * KC;
#pragma unroll
  for (int r = 0; r < RTW; ++r) {
    const int a = (warp * RTW + r) * 8 + gq;
    if (a >= q) continue;
#pragma unroll
    for (int c = 0; c < G2; ++c)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int col = j0 + 8 * c + 2 * t4 + hh;
        if (col < g.kc) O[(int64_t)a * KC + col] = acc[r][c][hh];
      }
  }
}

size_t boxop_smem(int) { return sizeof(double) * 2 * (size_t)SLICE; }
size_t leafop_smem(int rows, int cols) {
  return sizeof(double) * (size_t)(((rows + 7) >> 3) * 8) * pad4(((cols + 3) / 4) * 4);
}

template <class K>
int set_smem(K kern, size_t smem) {
  HIKF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return HIKF_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// tree build
// ---------------------------------------------------------------------------
int tree3_build(const double* xyz, int64_t m, const hikf_kernel3& kern, int n_cheb, int64_t max_leaf,
                cudaStream_t st, hikf_tree3** out) {
  if (!xyz || m < 1 || n_cheb < 2 || n_cheb > 5 || max_leaf < 1 || max_leaf > 128) {
    set_error("tree3: need m >= 1, 2 <= n_cheb <= 5, 1 <= max_leaf <= 128");
    return HIKF_BAD_ARGUMENT;
  }
  if ((kern.family != HIKF_GAUSSIAN && kern.family != HIKF_EXPONENTIAL) || !(kern.lx > 0) || !(kern.ly > 0) ||
      !(kern.lz > 0) || !(kern.variance >= 0)) {
    set_error("tree3: kernel must be gaussian or exponential with positive length scales");
    return HIKF_BAD_ARGUMENT;
  }
  auto* t = new hikf_tree3();
  t->m = m;
  t->n = n_cheb;
  t->q = n_cheb * n_cheb * n_cheb;
  t->k = kern;
  // scaled points (anisotropy folded into the coordinates)
  std::vector<double> p(3 * m);
  const double ls[3] = {kern.lx, kern.ly, kern.lz};
  for (int64_t i = 0; i < m; ++i)
    for (int d = 0; d < 3; ++d) {
      const double v = xyz[3 * i + d] / ls[d];
      if (!std::isfinite(v)) {
        delete t;
        set_error("coordinates must be finite");
        return HIKF_BAD_ARGUMENT;
      }
      p[3 * i + d] = v;
    }
  double hi[3];
  for (int d = 0; d < 3; ++d) {
    t->lo[d] = hi[d] = p[d];
    for (int64_t i = 1; i < m; ++i) {
      t->lo[d] = std::min(t->lo[d], p[3 * i + d]);
      hi[d] = std::max(hi[d], p[3 * i + d]);
    }
  }
  t->size = std::max(hi[0] - t->lo[0], std::max(hi[1] - t->lo[1], hi[2] - t->lo[2])) * (1.0 + 1e-12);
  // uniform depth: smallest with every leaf <= max_leaf (stop when 8^(d+1) > max(32768, 8 m))
  std::vector<int64_t> key(m);
  auto keys_at = [&](int depth) {
    const int64_t G = (int64_t)1 << depth;
    const double h = t->size / (double)G;
    for (int64_t i = 0; i < m; ++i) {
      int64_t b[3];
      for (int d = 0; d < 3; ++d) b[d] = box_coord3(p[3 * i + d], t->lo[d], h, G);
      key[i] = (b[0] * G + b[1]) * G + b[2];
    }
  };
  int depth = 0;
  for (;; ++depth) {
    keys_at(depth);
    std::vector<int64_t> sk(key);
    std::sort(sk.begin(), sk.end());
    int64_t best = 0;
    for (int64_t i = 0; i < m;) {
      int64_t j = i;
      while (j < m && sk[j] == sk[i]) ++j;
      best = std::max(best, j - i);
      i = j;
    }
    if (best <= max_leaf) break;
    const double next = std::pow(8.0, depth + 1);
    if (next > std::max(32768.0, 8.0 * (double)m) || depth + 1 >= 8) break;
  }
  t->depth = depth;
  t->G = (int64_t)1 << depth;
  t->order_h.resize(m);
  std::iota(t->order_h.begin(), t->order_h.end(), 0);
  std::stable_sort(t->order_h.begin(), t->order_h.end(), [&](int64_t a, int64_t b) { return key[a] < key[b]; });
  for (int64_t i = 0; i < m;) {
    int64_t j = i;
    while (j < m && key[t->order_h[j]] == key[t->order_h[i]]) ++j;
    t->leaf_key_h.push_back(key[t->order_h[i]]);
    t->leaf_start_h.push_back((int32_t)i);
    t->leaf_count_h.push_back((int32_t)(j - i));
    t->max_count = std::max<int32_t>(t->max_count, (int32_t)(j - i));
    i = j;
  }
  if (t->max_count > 128) {
    tree3_free(t);
    set_error("tree3: a leaf holds %d > 128 points (coincident points?)", t->max_count);
    return HIKF_BAD_ARGUMENT;
  }
  const int64_t nl = (int64_t)t->leaf_key_h.size();
  std::vector<double> ps(3 * m);
  for (int64_t i = 0; i < m; ++i)
    for (int d = 0; d < 3; ++d) ps[3 * i + d] = p[3 * t->order_h[i] + d];
  std::vector<int32_t> b2l(t->G * t->G * t->G, -1);
  for (int64_t l = 0; l < nl; ++l) b2l[t->leaf_key_h[l]] = (int32_t)l;
  HIKF_CHECK_CUDA(cudaMalloc((void**)&t->pts, sizeof(double) * 3 * m));
  HIKF_CHECK_CUDA(cudaMalloc((void**)&t->order, sizeof(int64_t) * m));
  HIKF_CHECK_CUDA(cudaMalloc((void**)&t->leaf_key, sizeof(int64_t) * nl));
  HIKF_CHECK_CUDA(cudaMalloc((void**)&t->leaf_start, sizeof(int32_t) * nl));
  HIKF_CHECK_CUDA(cudaMalloc((void**)&t->leaf_count, sizeof(int32_t) * nl));
  HIKF_CHECK_CUDA(cudaMalloc((void**)&t->box2leaf, sizeof(int32_t) * b2l.size()));
  HIKF_CHECK_CUDA(cudaMemcpy(t->pts, ps.data(), sizeof(double) * 3 * m, cudaMemcpyHostToDevice));
  HIKF_CHECK_CUDA(cudaMemcpy(t->order, t->order_h.data(), sizeof(int64_t) * m, cudaMemcpyHostToDevice));
  HIKF_CHECK_CUDA(cudaMemcpy(t->leaf_key, t->leaf_key_h.data(), sizeof(int64_t) * nl, cudaMemcpyHostToDevice));
  HIKF_CHECK_CUDA(cudaMemcpy(t->leaf_start, t->leaf_start_h.data(), sizeof(int32_t) * nl, cudaMemcpyHostToDevice));
  HIKF_CHECK_CUDA(cudaMemcpy(t->leaf_count, t->leaf_count_h.data(), sizeof(int32_t) * nl, cudaMemcpyHostToDevice));
  HIKF_CHECK_CUDA(cudaMemcpy(t->box2leaf, b2l.data(), sizeof(int32_t) * b2l.size(), cudaMemcpyHostToDevice));
  // interpolation weights
  const int n = t->n, q = t->q;
  {
    std::vector<double> Tn = cheb_node_table(n);
    double* dTn = nullptr;
    HIKF_CHECK_CUDA(cudaMalloc((void**)&dTn, sizeof(double) * Tn.size()));
    HIKF_CHECK_CUDA(cudaMemcpy(dTn, Tn.data(), sizeof(double) * Tn.size(), cudaMemcpyHostToDevice));
    HIKF_CHECK_CUDA(cudaMalloc((void**)&t->W2, sizeof(double) * m * q));
    const int blocks = (int)std::min<int64_t>((m + 255) / 256, (int64_t)num_sms() * 16);
    interp3_kernel<<<blocks, 256, 0, st>>>(t->pts, m, t->lo[0], t->lo[1], t->lo[2], t->size / (double)t->G, t->G, n,
                                           dTn, t->W2);
    HIKF_CHECK_LAUNCH();
    HIKF_CHECK_CUDA(cudaStreamSynchronize(st));
    cudaFree(dTn);
  }
  // shift operators: kron(Bx, By, Bz) for child class c = (cx cy cz)
  {
    std::vector<double> cn = cheb_nodes(n), S((size_t)8 * q * q), ST((size_t)8 * q * q);
    for (int c = 0; c < 8; ++c) {
      const int cc[3] = {(c >> 2) & 1, (c >> 1) & 1, c & 1};
      std::vector<double> B[3];
      for (int d = 0; d < 3; ++d) {
        std::vector<double> xs(n);
        for (int i = 0; i < n; ++i) xs[i] = (cn[i] + (double)(2 * cc[d] - 1)) / 2.0;
        B[d] = cheb_weights(xs, n);
      }
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
          for (int l = 0; l < n; ++l)
            for (int a = 0; a < n; ++a)
              for (int b = 0; b < n; ++b)
                for (int e = 0; e < n; ++e) {
                  const int row = (i * n + j) * n + l, col = (a * n + b) * n + e;
                  const double v = (B[0][i * n + a] * B[1][j * n + b]) * B[2][l * n + e];
                  S[(size_t)c * q * q + (size_t)row * q + col] = v;
                  ST[(size_t)c * q * q + (size_t)col * q + row] = v;
                }
    }
    HIKF_CHECK_CUDA(cudaMalloc((void**)&t->shift, sizeof(double) * S.size()));
    HIKF_CHECK_CUDA(cudaMalloc((void**)&t->shiftT, sizeof(double) * ST.size()));
    HIKF_CHECK_CUDA(cudaMemcpy(t->shift, S.data(), sizeof(double) * S.size(), cudaMemcpyHostToDevice));
    HIKF_CHECK_CUDA(cudaMemcpy(t->shiftT, ST.data(), sizeof(double) * ST.size(), cudaMemcpyHostToDevice));
  }
  // M2L operators per level
  if (depth >= 2) {
    int offs[NOFF][3];
    offsets3(offs);
    std::vector<double> nodes = cheb_nodes(n);
    double *dn = nullptr;
    int* doffs = nullptr;
    HIKF_CHECK_CUDA(cudaMalloc((void**)&dn, sizeof(double) * n));
    HIKF_CHECK_CUDA(cudaMalloc((void**)&doffs, sizeof(offs)));
    HIKF_CHECK_CUDA(cudaMemcpy(dn, nodes.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
    HIKF_CHECK_CUDA(cudaMemcpy(doffs, offs, sizeof(offs), cudaMemcpyHostToDevice));
    for (int l = 2; l <= depth; ++l) {
      HIKF_CHECK_CUDA(cudaMalloc((void**)&t->m2l[l], sizeof(double) * NOFF * q * q));
      const double h = t->size / (double)((int64_t)1 << l);
      m2l3_ops_kernel<<<num_sms() * 8, 256, 0, st>>>(n, h, dn, doffs, kern.family, kern.variance, t->m2l[l]);
      HIKF_CHECK_LAUNCH();
    }
    HIKF_CHECK_CUDA(cudaStreamSynchronize(st));
    cudaFree(dn);
    cudaFree(doffs);
  }
  *out = t;
  return HIKF_OK;
}

void tree3_free(hikf_tree3* t) {
  if (!t) return;
  for (void* p : {(void*)t->pts, (void*)t->order, (void*)t->leaf_key, (void*)t->leaf_start, (void*)t->leaf_count,
                  (void*)t->box2leaf, (void*)t->W2, (void*)t->shift, (void*)t->shiftT})
    if (p) cudaFree(p);
  for (auto* p : t->m2l)
    if (p) cudaFree(p);
  delete t;
}

// ---------------------------------------------------------------------------
// U (m x k) = Q V (m x k), both original order, row-major, device
// ---------------------------------------------------------------------------
int tree3_matmat(const hikf_tree3* t, const double* V, int64_t ldv, int64_t k, double* U, int64_t ldu,
                 cudaStream_t st) {
  if (k <= 0) return HIKF_OK;
  const int q = t->q, D = t->depth;
  const int64_t nl = (int64_t)t->leaf_key_h.size();
  static int offs_h[NOFF][3];
  static int* doffs = nullptr;
  if (!doffs) {
    offsets3(offs_h);
    HIKF_CHECK_CUDA(cudaMalloc((void**)&doffs, sizeof(offs_h)));
    HIKF_CHECK_CUDA(cudaMemcpy(doffs, offs_h, sizeof(offs_h), cudaMemcpyHostToDevice));
  }
  const size_t sm_p2p = leafop_smem(std::min(t->max_count, 64), t->max_count), sm_box = boxop_smem(q);
  const size_t sm_p2m = sizeof(double) * (size_t)LP * w2_ld(q), sm_l2p = sm_p2m;
  HIKF_TRY(set_smem(p2p3_kernel, std::max<size_t>(sm_p2p, 1)));
  HIKF_TRY(set_smem(p2m3_kernel, std::max<size_t>(sm_p2m, 1)));
  HIKF_TRY(set_smem(l2p3_kernel, std::max<size_t>(sm_l2p, 1)));
  HIKF_TRY(set_smem(boxop3_kernel, sm_box));
  // expansion buffers for one chunk: W_l, L_l (dense per level, KC columns)
  double* W[kMaxDepth + 1] = {nullptr};
  double* L[kMaxDepth + 1] = {nullptr};
  uint8_t* NZ[kMaxDepth + 1] = {nullptr};
  if (D >= 2)
    for (int l = 2; l <= D; ++l) {
      const int64_t nb = (int64_t)1 << (3 * l);
      HIKF_CHECK_CUDA(cudaMallocAsync((void**)&W[l], sizeof(double) * nb * q * KC, st));
      HIKF_CHECK_CUDA(cudaMallocAsync((void**)&L[l], sizeof(double) * nb * q * KC, st));
      HIKF_CHECK_CUDA(cudaMallocAsync((void**)&NZ[l], nb, st));
    }
  uint8_t* LNZ = nullptr;
  HIKF_CHECK_CUDA(cudaMallocAsync((void**)&LNZ, std::max<int64_t>(nl, 1), st));
  uint8_t* OCC[kMaxDepth + 1] = {nullptr};
  if (D >= 2) {
    for (int l = 2; l <= D; ++l) HIKF_CHECK_CUDA(cudaMallocAsync((void**)&OCC[l], (int64_t)1 << (3 * l), st));
    const int64_t nbD = (int64_t)1 << (3 * D);
    occ_leaf<<<(unsigned)std::min<int64_t>((nbD + 255) / 256, num_sms() * 16), 256, 0, st>>>(t->box2leaf, nbD,
                                                                                             OCC[D]);
    HIKF_CHECK_LAUNCH();
    for (int l = D - 1; l >= 2; --l) {
      const int64_t nb = (int64_t)1 << (3 * l);
      occ_parent<<<(unsigned)std::min<int64_t>((nb + 255) / 256, num_sms() * 16), 256, 0, st>>>(OCC[l + 1],
                                                                                                (int64_t)1 << l, OCC[l]);
      HIKF_CHECK_LAUNCH();
    }
  }
  const T3v tv = view(t);
  int status = HIKF_OK;
  for (int64_t c0 = 0; c0 < k && status == HIKF_OK; c0 += KC) {
    Chunk ch{V + c0, ldv, (int)std::min<int64_t>(KC, k - c0), U + c0, ldu, nullptr};
    nonzero_leaves<<<(unsigned)((nl * 32 + 255) / 256), 256, 0, st>>>(tv, ch.V, ch.ldv, ch.kc, nl, LNZ);
    HIKF_CHECK_LAUNCH();
    {
      ProfScope ps(ST_P2P, st);
      ch.flops = prof_flops_ptr(ST_P2P);
      p2p3_kernel<<<(unsigned)nl, T3, sm_p2p, st>>>(tv, ch, LNZ);
      HIKF_CHECK_LAUNCH();
    }
    if (D < 2) continue;
    {
      ProfScope ps(ST_P2M, st);
      // W_D is not cleared: a box / column group is read only where its nz bit is set, and
      // P2M writes every group its leaf's charge mask flags
      ch.flops = prof_flops_ptr(ST_P2M);
      p2m3_kernel<<<(unsigned)nl, T3, sm_p2m, st>>>(tv, ch, W[D], LNZ);
      HIKF_CHECK_LAUNCH();
      const int64_t nbD = (int64_t)1 << (3 * D);
      HIKF_CHECK_CUDA(cudaMemsetAsync(NZ[D], 0, nbD, st));
      nz_leaf_boxes<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((nl + 255) / 256, num_sms() * 8)), 256, 0,
                      st>>>(t->leaf_key, LNZ, nl, NZ[D]);
      HIKF_CHECK_LAUNCH();
    }
    for (int l = D - 1; l >= 2; --l) {
      ProfScope ps(ST_M2M, st);
      const int64_t nb = (int64_t)1 << (3 * l);
      nz_parent<<<(unsigned)std::min<int64_t>((nb + 255) / 256, num_sms() * 16), 256, 0, st>>>(NZ[l + 1],
                                                                                             (int64_t)1 << l, NZ[l]);
      HIKF_CHECK_LAUNCH();
      // only boxes with a nonzero child are read later (nz), so M2M skips the others
      BoxOpArgs a{OP_M2M, q, l, 0, (int64_t)1 << l, W[l + 1], W[l], t->shiftT, nullptr, ch.kc, NZ[l + 1], NZ[l],
                  prof_flops_ptr(ST_M2M)};
      boxop3_kernel<<<(unsigned)nb, T3, sm_box, st>>>(a);
      HIKF_CHECK_LAUNCH();
    }
    for (int l = 2; l <= D; ++l) {
      {
        ProfScope ps(ST_M2L, st);
        const int64_t units = (int64_t)1 << (3 * (l - 1));  // parents x 8 child classes, one launch
        BoxOpArgs a{OP_M2L, q, l, 0, (int64_t)1 << l, W[l], L[l], t->m2l[l], doffs, ch.kc, NZ[l], OCC[l],
                    prof_flops_ptr(ST_M2L)};
        // row-split kernel: 8 warps x 2 row tiles (q <= 128), 2 column groups per CTA (measured
        // best: 1 group under-fills, 4 groups need 168 registers; profiles/r01_m2l3_sweep.log)
        if (q <= 8 * 8 * 2) {
          m2l3_rows_kernel<2, 2><<<(unsigned)(8 * units * (KC / 16)), T3, 0, st>>>(a);
        } else {
          boxop3_kernel<<<(unsigned)(8 * units), T3, sm_box, st>>>(a);
        }
        HIKF_CHECK_LAUNCH();
      }
      if (l > 2) {
        ProfScope ps(ST_L2L, st);
        const int64_t units = (int64_t)1 << (3 * (l - 1));
        BoxOpArgs a{OP_L2L, q, l, 0, (int64_t)1 << l, L[l - 1], L[l], t->shift, nullptr, ch.kc, nullptr, OCC[l],
                    prof_flops_ptr(ST_L2L)};
        boxop3_kernel<<<(unsigned)(8 * units), T3, sm_box, st>>>(a);
        HIKF_CHECK_LAUNCH();
      }
    }
    {
      ProfScope ps(ST_L2P, st);
      ch.flops = prof_flops_ptr(ST_L2P);
      l2p3_kernel<<<(unsigned)nl, T3, sm_l2p, st>>>(tv, ch, L[D]);
      HIKF_CHECK_LAUNCH();
    }
  }
  for (int l = 2; l <= D; ++l) {
    cudaFreeAsync(W[l], st);
    cudaFreeAsync(L[l], st);
    cudaFreeAsync(NZ[l], st);
    cudaFreeAsync(OCC[l], st);
  }
  cudaFreeAsync(LNZ, st);
  return status;
}

// dense H^T chunk (m x 64, original order) from CSR H (n x m): Ht[cell][r - r0] = H[r][cell]
namespace {
__global__ void scatter_ht_chunk(int64_t r0, int64_t rows, const int32_t* __restrict__ ip,
                                 const int32_t* __restrict__ ix, const double* __restrict__ val,
                                 double* __restrict__ Ht) {
  const int64_t r = r0 + blockIdx.x;
  if (blockIdx.x >= rows) return;
  for (int64_t e = ip[r] + threadIdx.x; e < ip[r + 1]; e += blockDim.x) Ht[(int64_t)ix[e] * KC + blockIdx.x] = val[e];
}
}  // namespace

int tree3_matmat_csrT(const hikf_tree3* t, int64_t n, const int32_t* ip, const int32_t* ix, const double* val,
                      double* U, cudaStream_t st) {
  if (n <= 0) return HIKF_OK;
  double* Ht = nullptr;
  HIKF_CHECK_CUDA(cudaMallocAsync((void**)&Ht, sizeof(double) * t->m * KC, st));
  int status = HIKF_OK;
  for (int64_t r0 = 0; r0 < n && status == HIKF_OK; r0 += KC) {
    const int64_t rows = std::min<int64_t>(KC, n - r0);
    HIKF_CHECK_CUDA(cudaMemsetAsync(Ht, 0, sizeof(double) * t->m * KC, st));
    scatter_ht_chunk<<<(unsigned)rows, 128, 0, st>>>(r0, rows, ip, ix, val, Ht);
    HIKF_CHECK_LAUNCH();
    status = tree3_matmat(t, Ht, KC, rows, U + r0, n, st);
  }
  cudaFreeAsync(Ht, st);
  return status;
}

int tree3_info(const hikf_tree3* t, int64_t* m, int32_t* depth, int32_t* n_cheb, int64_t* n_leaves, double* lo3,
               double* size) {
  if (!t) return HIKF_BAD_ARGUMENT;
  if (m) *m = t->m;
  if (depth) *depth = t->depth;
  if (n_cheb) *n_cheb = t->n;
  if (n_leaves) *n_leaves = (int64_t)t->leaf_key_h.size();
  if (lo3)
    for (int d = 0; d < 3; ++d) lo3[d] = t->lo[d];
  if (size) *size = t->size;
  return HIKF_OK;
}

void tree3_kernel(const hikf_tree3* t, hikf_kernel3* k) { *k = t->k; }

int tree3_export(const hikf_tree3* t, int64_t* order, int64_t* leaf_keys, int64_t* leaf_starts,
                 int64_t* leaf_counts) {
  if (!t) return HIKF_BAD_ARGUMENT;
  if (order) std::copy(t->order_h.begin(), t->order_h.end(), order);
  for (size_t l = 0; l < t->leaf_key_h.size(); ++l) {
    if (leaf_keys) leaf_keys[l] = t->leaf_key_h[l];
    if (leaf_starts) leaf_starts[l] = t->leaf_start_h[l];
    if (leaf_counts) leaf_counts[l] = t->leaf_count_h[l];
  }
  return HIKF_OK;
}

}  // namespace hikf

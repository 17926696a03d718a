// Warp-streaming DMMA GEMM for the downward FMM transfers whose inner
// dimension is one small operator (L2L, L2P):
//
//   out_task (R x n) = A_task (R x K) * B_task (K x n)  [+ init]
//
// A (the four stacked shift operators of a level, or a leaf's interpolation
// rows) sits in shared memory; after that every warp works independently on
// 8-column units (task, j0..j0+8): it loads its K x 8 B block straight into
// DMMA fragments (one register per k-step), runs the R/8 x K/4 DMMA chains,
// and writes its output columns -- no block barriers in the stream, so the
// latency of the HBM stream is hidden by the many warps in flight.
//
//   L2L (fmm.py:361-363, sparse path): R = 4 q (children), K = q_parent,
//        B = L_{l-1}[parent], init = the pair-major M2L scratch S[child][j][a]
//        (M2L sum first, then + L2L -- the reference's order); writes the
//        box-major locals L_l[child][a][j].  A is level-constant: one CTA
//        loads it once and its warps stride over (parent, 8 columns) units.
//   L2P (fmm.py:366): R = leaf points, K = q_leaf, B = L_D[leaf],
//        out rows = U[order[p]] (store; the sparse near field is added after).
//        One CTA per (leaf, 64-row block); its warps stride over the columns.
#include <algorithm>
#include <cstdlib>

#include "boxgemm.h"
#include "fmm_device.cuh"
#include "prof.h"

namespace hikf {

namespace {

constexpr int BW_THREADS = 256;
constexpr int BW_MAXK4 = 16;   // K <= 64
constexpr int BW_RT = 8;       // row tiles per register pass (64 rows)

__host__ __device__ inline int pad4(int k) { return k + ((4 - k % 16) + 16) % 16; }  // == 4 mod 16

struct BoxArgs {
  int mode;                // 0 = L2L, 1 = L2P
  int64_t n;               // columns
  int K;                   // inner dimension
  // L2L
  const int32_t* occp;     // occupied parents
  int64_t nparents;
  int q;                   // child coefficients
  int64_t Gp;
  const double* Lp;        // parent locals (box-major)
  const double* shift;     // 4 q x qp
  const double* S;         // compact M2L scratch of the child level (q per slot)
  const int32_t* tmap;     // (child box, ray) -> slot in S, or -1
  double* L;               // child locals (box-major)
  // L2P
  const int32_t *leaf_box, *leaf_start, *leaf_count;
  const double* W2s;
  const int64_t* order;
  const double* Lleaf;
  double* U;
  int64_t ldu;
  int64_t r0, r1;  // L2P row window: only original rows in [r0, r1) are written, at U + (row - r0) ldu
  int64_t pxlo, pxhi;  // L2L: parents outside this box-column range are skipped (leaf-aligned shard)
  int64_t leaf0;       // L2P: first leaf of the launch (blockIdx.x + leaf0)
  int64_t s0;          // L2P: >= 0: leaf-aligned shard, U row = sorted position - s0
  unsigned long long* flops;
};

template <int NK4, int NRT, int MODE, bool PF, int CW>
__global__ void __launch_bounds__(BW_THREADS, 2) box_warp_kernel(BoxArgs g) {
  extern __shared__ double As[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, t4 = lane & 3;
  const int K = g.K, lda = pad4(NK4 * 4);  // rows hold NK4*4 >= K entries (zero beyond K)
  int R, row_off = 0;
  const double* Ag;
  if (MODE == 0) {
    R = 4 * g.q;
    Ag = g.shift;
  } else {
    row_off = blockIdx.y * 64;
    const int cnt = g.leaf_count[blockIdx.x + g.leaf0];
    if (row_off >= cnt) return;
    R = min(64, cnt - row_off);
    Ag = g.W2s + (int64_t)(g.leaf_start[blockIdx.x + g.leaf0] + row_off) * K;
  }
  const int nrt = (R + 7) >> 3;
  for (int e = tid; e < nrt * 8 * NK4 * 4; e += BW_THREADS) {
    int r = e / (NK4 * 4), k = e % (NK4 * 4);
    As[r * lda + k] = (r < R && k < K) ? Ag[(int64_t)r * K + k] : 0.0;
  }
  __syncthreads();

  // a unit = one task x 8 CW columns: every A fragment read from shared memory
  // feeds CW DMMAs (CW column tiles of 8)
  constexpr int UW = 8 * CW;
  const int64_t ncb = (g.n + UW - 1) / UW;
  int64_t unit0, unit_stride, units;
  if (MODE == 0) {
    units = g.nparents * ncb;
    unit0 = (int64_t)blockIdx.x * (BW_THREADS / 32) + warp;
    unit_stride = (int64_t)gridDim.x * (BW_THREADS / 32);
  } else {
    units = ncb;
    unit0 = warp;
    unit_stride = BW_THREADS / 32;
  }
  unsigned long long useful = 0;
  // B fragments of a unit: one register per k-step and column tile (this lane's columns j0 + 8c + gq)
  auto load_b = [&](int64_t u, double (&b)[CW][NK4]) {
    const int64_t task = MODE == 0 ? u / ncb : blockIdx.x + g.leaf0;
    const int64_t j0 = (u % ncb) * UW;
    const double* Bg = MODE == 0 ? g.Lp + (int64_t)g.occp[task] * K * g.n
                                 : g.Lleaf + (int64_t)g.leaf_box[task] * K * g.n;
#pragma unroll
    for (int c = 0; c < CW; ++c) {
      const int64_t jb = j0 + 8 * c + gq;
#pragma unroll
      for (int k4 = 0; k4 < NK4; ++k4) {
        const int k = k4 * 4 + t4;
        b[c][k4] = (k < K && jb < g.n) ? Bg[(int64_t)k * g.n + jb] : 0.0;
      }
    }
  };
  double bn[CW][NK4];  // software pipeline (PF): the next unit's fragments are in flight during this unit
  if (PF && unit0 < units) load_b(unit0, bn);
  for (int64_t u = unit0; u < units; u += unit_stride) {
    const int64_t task = MODE == 0 ? u / ncb : blockIdx.x + g.leaf0;
    const int64_t j0 = (u % ncb) * UW;
    double b[CW][NK4];
    if (PF) {
#pragma unroll
      for (int c = 0; c < CW; ++c)
#pragma unroll
        for (int k4 = 0; k4 < NK4; ++k4) b[c][k4] = bn[c][k4];
      if (u + unit_stride < units) load_b(u + unit_stride, bn);
    } else {
      load_b(u, b);
    }
    const int cols = (int)(g.n - j0 < UW ? g.n - j0 : UW);
    if (lane == 0) useful += 2ull * R * K * cols;
    int64_t X = 0, Y = 0;
    if (MODE == 0) {
      const int64_t P = g.occp[task];
      X = P / g.Gp;
      Y = P % g.Gp;
      if (X < g.pxlo || X > g.pxhi) continue;  // warp-uniform: no ancestor of a shard's leaves
    }
    auto child_of = [&](int r, int& a) {
      const int ci = r / g.q;
      a = r - ci * g.q;
      return (2 * X + (ci >> 1)) * (2 * g.Gp) + (2 * Y + (ci & 1));
    };
    for (int r0 = 0; r0 < nrt; r0 += NRT) {
      // L2L: the M2L-sum init values are loaded before the DMMA chain (their
      // latency hides under it) and added after it -- the reference's order
      // (M2L sum, then + L2L) and the same rounding as adding them afterwards
      double init[MODE == 0 ? NRT : 1][CW][2];
      if (MODE == 0) {
#pragma unroll
        for (int i = 0; i < NRT; ++i) {
          const int r = (r0 + i) * 8 + gq;
#pragma unroll
          for (int c = 0; c < CW; ++c) init[i][c][0] = init[i][c][1] = 0.0;
          if (r0 + i < nrt && r < R) {
            int a;
            const int64_t crow = child_of(r, a) * g.n;
#pragma unroll
            for (int c = 0; c < CW; ++c)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int64_t jc = j0 + 8 * c + 2 * t4 + h;
                if (jc < g.n) {
                  const int32_t slot = g.tmap[crow + jc];
                  if (slot >= 0) init[i][c][h] = g.S[(int64_t)slot * g.q + a];
                }
              }
          }
        }
      }
      double acc[NRT][CW][2];
#pragma unroll
      for (int i = 0; i < NRT; ++i)
#pragma unroll
        for (int c = 0; c < CW; ++c) acc[i][c][0] = acc[i][c][1] = 0.0;
#pragma unroll
      for (int k4 = 0; k4 < NK4; ++k4)
#pragma unroll
        for (int i = 0; i < NRT; ++i)
          if (r0 + i < nrt) {
            const double af = As[((r0 + i) * 8 + gq) * lda + k4 * 4 + t4];
#pragma unroll
            for (int c = 0; c < CW; ++c) dmma884(acc[i][c][0], acc[i][c][1], af, b[c][k4]);
          }
      // epilogue: rows (r0+i)*8+gq, columns j0 + 8 c + 2 t4 + h
#pragma unroll
      for (int i = 0; i < NRT; ++i) {
        const int r = (r0 + i) * 8 + gq;
        if (r0 + i >= nrt || r >= R) continue;
        double* orow;
        if (MODE == 0) {
          int a;
          orow = g.L + (child_of(r, a) * g.q + a) * g.n;
        } else {
          if (g.s0 >= 0) {
            orow = g.U + (g.leaf_start[task] + row_off + r - g.s0) * g.ldu;
          } else {
            const int64_t orw = g.order[g.leaf_start[task] + row_off + r];
            if (orw < g.r0 || orw >= g.r1) continue;
            orow = g.U + (orw - g.r0) * g.ldu;
          }
        }
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          const int64_t jc = j0 + 8 * c + 2 * t4;
          if (jc + 1 < g.n && (((uintptr_t)(orow + jc)) & 15) == 0) {
            const double v0 = MODE == 0 ? acc[i][c][0] + init[MODE == 0 ? i : 0][c][0] : acc[i][c][0];
            const double v1 = MODE == 0 ? acc[i][c][1] + init[MODE == 0 ? i : 0][c][1] : acc[i][c][1];
            *reinterpret_cast<double2*>(orow + jc) = make_double2(v0, v1);
          } else {
#pragma unroll
            for (int h = 0; h < 2; ++h)
              if (jc + h < g.n) orow[jc + h] = MODE == 0 ? acc[i][c][h] + init[MODE == 0 ? i : 0][c][h] : acc[i][c][h];
          }
        }
      }
    }
  }
  if (g.flops && lane == 0 && useful) atomicAdd(g.flops, useful);
}

// exact k-steps per operator size (one instantiation per ceil(K/4)): a padded
// bucket would spend DMMAs on all-zero k-steps (49 -> 64 is 30 % at order 7)
int k4_bucket(int K) { return (K + 3) / 4; }

// shared memory of the A block: rows padded to 8, leading dimension pad4(4 * NK4)
size_t box_smem(int R, int K) {
  return sizeof(double) * (size_t)(((R + 7) >> 3) * 8) * pad4(4 * k4_bucket(K));
}

template <int NK4, int NRT, int MODE, bool PF, int CW>
int launch_box_t(const BoxArgs& a, dim3 grid, size_t smem, cudaStream_t st) {
  static size_t configured = 0;
  auto kern = box_warp_kernel<NK4, NRT, MODE, PF, CW>;
  if (smem > configured) {
    HIKF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::max<size_t>(smem, 48 << 10)));
    configured = std::max<size_t>(smem, 48 << 10);
  }
  kern<<<grid, BW_THREADS, smem, st>>>(a);
  HIKF_CHECK_LAUNCH();
  return HIKF_OK;
}

template <int K4>
int launch_box_k(const BoxArgs& a, dim3 grid, size_t smem, cudaStream_t st) {
  // L2L: 4 row tiles per pass, L2P: 8; both with the next unit's B fragments in flight
  // (one 8-column tile per unit; 2-tile units were measured slower, profiles/r01_box_sweep.log)
  if (a.mode == 0) return launch_box_t<K4, 4, 0, true, 1>(a, grid, smem, st);
  return launch_box_t<K4, 8, 1, true, 1>(a, grid, smem, st);
}

// compile-time k-steps: exactly ceil(K/4)
int launch_box(const BoxArgs& a, int R, dim3 grid, cudaStream_t st) {
  const size_t smem = box_smem(R, a.K);
  const int nk4 = (a.K + 3) / 4;

#define HIKF_BOX(K4)          \
  if (nk4 <= K4)              \
    return launch_box_k<K4>(a, grid, smem, st);
  HIKF_BOX(1) HIKF_BOX(2) HIKF_BOX(3) HIKF_BOX(4) HIKF_BOX(5) HIKF_BOX(6) HIKF_BOX(7) HIKF_BOX(8)
  HIKF_BOX(9) HIKF_BOX(10) HIKF_BOX(11) HIKF_BOX(12) HIKF_BOX(13) HIKF_BOX(14) HIKF_BOX(15) HIKF_BOX(16)
#undef HIKF_BOX
  set_error("box-streaming kernel supports K <= %d (got %d)", 4 * BW_MAXK4, a.K);
  return HIKF_BAD_ARGUMENT;
}

// ---------------------------------------------------------------------------
// Fused leaf-level downward step: L2L into the leaves + L2P, the leaf locals
// never stored.  One CTA per occupied leaf T (points <= 64), its warps stride
// over 8-column units:
//   l[a][j]     = S[T][j][a] + sum_b C_ci[a][b] L_{D-1}[parent][b][j]   (fmm.py:361-363:
//                 the M2L sum first, then + L2L; the same DMMA k-order as l2l_boxes)
//   U[p][j]     = sum_a W2[p][a] l[a][j]                                 (fmm.py:366)
// l goes from the accumulator layout to B fragments through a per-warp
// shared-memory tile (q x 8).  A operands (the leaf's child-class shift rows and
// its W2 rows) are staged once per CTA.  Results are bit-identical to
// l2l_boxes + l2p_boxes (same products in the same order); the saving is the
// G_D^2 x q x n leaf-local array (written and read back: 9.6 GB at cfg4).
// ---------------------------------------------------------------------------
constexpr int kLeafUnits = 2048;  // near-field fold: up to 2048 units of 8 columns (n <= 16384)
struct LeafArgs {
  int64_t n;
  int q, qp;
  int64_t G;  // leaf-level grid
  const int32_t *leaf_box, *leaf_start, *leaf_count;
  const double* W2s;
  const int64_t* order;
  const double* Lp;     // parent-level locals (box-major)
  const double* shift;  // 4 q x qp stacked child operators of the parent level
  const double* S;      // compact M2L scratch of the leaf level (q per slot)
  const int32_t* tmap;  // (leaf box, ray) -> slot in S, or -1
  double* U;
  int64_t ldu, r0, r1;
  int64_t leaf0;  // first leaf of the launch (blockIdx.x + leaf0)
  int64_t s0;     // >= 0: leaf-aligned shard, U row = sorted position - s0 (else original rows, r0 / r1 window)
  unsigned long long *fl_l2l, *fl_l2p;
  // near-field sums of the (leaf, ray) items (p2p_sparse), added to U here: U = far + near
  const double* Pnear;  // item-major, maxc per item; null: not added here
  const int64_t* items;
  const int32_t* item_start;
  int32_t maxc;
};

// 8-byte asynchronous global -> shared copy; !pred: the destination is zero-filled
__device__ __forceinline__ void cp_async8_zfill(double* dst, const double* src, bool pred) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(sz) : "memory");
}

// shared-memory load the compiler cannot hoist out of the unit loop (the A
// operands are loop-invariant; keeping them all in registers would spill)
__device__ __forceinline__ double lds64(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}

// NT: 8-column tiles per warp unit.  With NT = 2 every A fragment read from shared memory feeds
// two DMMAs (the kernel is otherwise co-limited by the shared-memory data pipe: one 256-byte
// fragment per DMMA); the larger register tile runs as 3 CTAs of 4 warps per SM.
template <int NK1, int NRT1, int NK2, int NT>
__global__ void __launch_bounds__(NT == 2 ? 128 : BW_THREADS, NT == 2 ? 3 : 2) leaf_down_kernel(LeafArgs g) {
  extern __shared__ double sm[];
  constexpr int THREADS = NT == 2 ? 128 : BW_THREADS;
  constexpr int UC = 8 * NT;  // columns per unit
  constexpr int LDA1 = NK1 * 4 + ((4 - (NK1 * 4) % 16) + 16) % 16;
  constexpr int LDA2 = NK2 * 4 + ((4 - (NK2 * 4) % 16) + 16) % 16;
  constexpr int KR2 = NK2 * 4;              // rows of the per-warp l tile
  constexpr int LDL = NT == 2 ? 20 : 8;     // its row stride: conflict-free 16-byte stores and fragment loads
  double* A1 = sm;                          // NRT1*8 x LDA1
  double* A2 = A1 + NRT1 * 8 * LDA1;        // 64 x LDA2
  double* Lw = A2 + 64 * LDA2;              // warps x KR2 x LDL
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, t4 = lane & 3;
  const int q = g.q, qp = g.qp;
  const int64_t T = blockIdx.x + g.leaf0;
  const int64_t box = g.leaf_box[T];
  const int64_t X = box / g.G, Y = box % g.G;
  const int ci = (int)(((X & 1) << 1) | (Y & 1));
  const int64_t P = (X >> 1) * (g.G >> 1) + (Y >> 1);
  const int cnt = g.leaf_count[T];
  const int64_t ls = g.leaf_start[T];
  const double* Cg = g.shift + (int64_t)ci * q * qp;
  // A operands: asynchronous 8-byte copies, all in flight at once (zero fill for the padding)
  for (int e = tid; e < NRT1 * 8 * NK1 * 4; e += THREADS) {
    const int r = e / (NK1 * 4), k = e % (NK1 * 4);
    const bool ok = r < q && k < qp;
    cp_async8_zfill(A1 + r * LDA1 + k, ok ? Cg + (int64_t)r * qp + k : Cg, ok);
  }
  // near-field items of this leaf: per 8-column tile, the columns that hold an item (one byte)
  // and the tile's first item (a tile's items are consecutive, in ascending ray order)
  __shared__ uint32_t umask[kLeafUnits / 4];
  __shared__ int32_t ufirst[kLeafUnits];
  const int32_t is0 = g.Pnear ? g.item_start[T] : 0, is1 = g.Pnear ? g.item_start[T + 1] : 0;
  if (g.Pnear)
    for (int e = tid; e < (int)((g.n + 7) / 8); e += THREADS) {
      ufirst[e] = INT32_MAX;
      if ((e & 3) == 0) umask[e >> 2] = 0;
    }
  const double* Wg = g.W2s + ls * q;
  for (int e = tid; e < 64 * NK2 * 4; e += THREADS) {
    const int r = e / (NK2 * 4), k = e % (NK2 * 4);
    const bool ok = r < cnt && k < q;
    cp_async8_zfill(A2 + r * LDA2 + k, ok ? Wg + (int64_t)r * q + k : Wg, ok);
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  double* lw = Lw + warp * KR2 * LDL;
  const int64_t n = g.n;
  const int64_t ncb = (n + UC - 1) / UC;
  const double* Lpar = g.Lp + P * qp * n;
  const int32_t* tm = g.tmap + box * n;
  // output row in U of each leaf point (or -1 outside the row window), shared by the warps
  __shared__ int32_t orow[64];
  if (tid < 64) {
    int32_t r = -1;
    if (tid < cnt) {
      if (g.s0 >= 0) {
        r = (int32_t)(ls + tid - g.s0);
      } else {
        const int64_t o = g.order[ls + tid];
        if (o >= g.r0 && o < g.r1) r = (int32_t)(o - g.r0);
      }
    }
    orow[tid] = r;
  }
  for (int32_t i = is0 + tid; i < is1; i += THREADS) {
    const int j = (int)(g.items[i] % g.n), u = j >> 3;
    atomicOr(&umask[u >> 2], (1u << (j & 7)) << ((u & 3) * 8));
    atomicMin(&ufirst[u], i);
  }
  __syncthreads();
  // A unit's parent columns are loaded during the previous unit's L2P phase, straight into the
  // registers its L2L chain reads (dead by then); its M2L slot indices too, so that the M2L
  // sums, loaded at the start of the unit and added after the L2L chain, are not a dependent load.
  auto load_cols = [&](int64_t u, double (&b1)[NT][NK1]) {
#pragma unroll
    for (int tt = 0; tt < NT; ++tt) {
      const int64_t jb = u * UC + tt * 8 + gq;
      // one running row pointer (opaque to the compiler: NK1 hoisted row addresses would cost 2 NK1 registers)
      const double* pr = Lpar + (int64_t)t4 * n + (jb < n ? jb : 0);
      asm volatile("" : "+l"(pr));
#pragma unroll
      for (int k4 = 0; k4 < NK1; ++k4) {
        const int k = k4 * 4 + t4;
        b1[tt][k4] = (k < qp && jb < n) ? *pr : 0.0;
        pr += 4 * n;
      }
    }
  };
  auto load_slots = [&](int64_t u, int32_t (&sl)[NT][2]) {
#pragma unroll
    for (int tt = 0; tt < NT; ++tt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t jc = u * UC + tt * 8 + 2 * t4 + h;
        sl[tt][h] = jc < n ? tm[jc] : -1;
      }
  };
  constexpr int kStep = THREADS / 32;
  unsigned long long useful1 = 0, useful2 = 0;
  double b1[NT][NK1];
  int32_t slot[NT][2];
  if (warp < ncb) {
    load_cols(warp, b1);
    load_slots(warp, slot);
  }
  for (int64_t u = warp; u < ncb; u += kStep) {
    const bool more = u + kStep < ncb;
    const int64_t j0 = u * UC;
    const int cols = (int)(n - j0 < UC ? n - j0 : UC);
    if (lane == 0) {
      useful1 += 2ull * q * qp * cols;
      useful2 += 2ull * cnt * q * cols;
    }
    // the M2L sums of this unit: asynchronous copies into the warp's l tile, each thread into the
    // positions it will add its own L2L results to (no registers held while they are in flight
    // under the DMMA chain; the previous unit's L2P has finished reading the tile)
    __syncwarp();
#pragma unroll
    for (int tt = 0; tt < NT; ++tt)
#pragma unroll
      for (int i = 0; i < NRT1; ++i) {
        const int r = i * 8 + gq;
        if (r < KR2) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const bool ok = r < q && slot[tt][h] >= 0;
            cp_async8_zfill(lw + r * LDL + tt * 8 + 2 * t4 + h, ok ? g.S + (int64_t)slot[tt][h] * q + r : g.S, ok);
          }
        }
      }
    asm volatile("cp.async.commit_group;" ::: "memory");
    // L2L into the leaf: acc1 = C_ci L_parent, then l = acc1 + S
    double acc1[NT][NRT1][2];
#pragma unroll
    for (int tt = 0; tt < NT; ++tt)
#pragma unroll
      for (int i = 0; i < NRT1; ++i) acc1[tt][i][0] = acc1[tt][i][1] = 0.0;
#pragma unroll
    for (int k4 = 0; k4 < NK1; ++k4)
#pragma unroll
      for (int i = 0; i < NRT1; ++i) {
        const double af = lds64(A1 + (i * 8 + gq) * LDA1 + k4 * 4 + t4);
#pragma unroll
        for (int tt = 0; tt < NT; ++tt) dmma884(acc1[tt][i][0], acc1[tt][i][1], af, b1[tt][k4]);
      }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
    for (int tt = 0; tt < NT; ++tt)
#pragma unroll
      for (int i = 0; i < NRT1; ++i) {
        const int r = i * 8 + gq;
        if (r < KR2) {  // 16-byte accesses: the warp's 32 chunks cover 4 wavefronts
          double2* pl = reinterpret_cast<double2*>(lw + r * LDL + tt * 8 + 2 * t4);
          const double2 in = *pl;
          *pl = make_double2(acc1[tt][i][0] + in.x, acc1[tt][i][1] + in.y);
        }
      }
    __syncwarp();
    // the next unit's parent columns and slots: in flight during this unit's L2P
    if (more) {
      load_cols(u + kStep, b1);
      load_slots(u + kStep, slot);
    }
    // L2P: U = W2 l  (the l fragments are read per k-step; rows q .. KR2 - 1 of the tile are zero)
    double acc2[NT][8][2];
#pragma unroll
    for (int tt = 0; tt < NT; ++tt)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc2[tt][i][0] = acc2[tt][i][1] = 0.0;
#pragma unroll
    for (int k4 = 0; k4 < NK2; ++k4) {
      double bf[NT];
#pragma unroll
      for (int tt = 0; tt < NT; ++tt) bf[tt] = lds64(lw + (k4 * 4 + t4) * LDL + tt * 8 + gq);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double af = lds64(A2 + (i * 8 + gq) * LDA2 + k4 * 4 + t4);
#pragma unroll
        for (int tt = 0; tt < NT; ++tt) dmma884(acc2[tt][i][0], acc2[tt][i][1], af, bf[tt]);
      }
    }
#pragma unroll
    for (int tt = 0; tt < NT; ++tt) {
      const int64_t ut = u * NT + tt;  // the 8-column tile
      const int64_t jc = ut * 8 + 2 * t4;
      const unsigned um = (g.Pnear && ut * 8 < n) ? (umask[ut >> 2] >> ((ut & 3) * 8)) & 0xffu : 0u;
      if (um) {  // rays of this tile cross the leaf's neighbourhood: + their near sums
        const int32_t f = ufirst[ut];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = 2 * t4 + h;
          if ((um >> c) & 1) {
            const double* pn = g.Pnear + (int64_t)(f + __popc(um & ((1u << c) - 1))) * g.maxc + gq;
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (i * 8 + gq < cnt) acc2[tt][i][h] += pn[i * 8];
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int32_t orw = orow[i * 8 + gq];
        if (orw < 0) continue;
        double* o = g.U + (int64_t)orw * g.ldu;
        if (jc + 1 < n && (((uintptr_t)(o + jc)) & 15) == 0) {
          *reinterpret_cast<double2*>(o + jc) = make_double2(acc2[tt][i][0], acc2[tt][i][1]);
        } else {
          if (jc < n) o[jc] = acc2[tt][i][0];
          if (jc + 1 < n) o[jc + 1] = acc2[tt][i][1];
        }
      }
    }
  }
  if (lane == 0) {
    if (g.fl_l2l && useful1) atomicAdd(g.fl_l2l, useful1);
    if (g.fl_l2p && useful2) atomicAdd(g.fl_l2p, useful2);
  }
}

template <int NK1, int NRT1, int NK2, int NT>
int launch_leaf_nt(const LeafArgs& a, unsigned nleaves, cudaStream_t st) {
  constexpr int THREADS = NT == 2 ? 128 : BW_THREADS;
  constexpr int LDL = NT == 2 ? 20 : 8;
  constexpr int LDA1 = NK1 * 4 + ((4 - (NK1 * 4) % 16) + 16) % 16;
  constexpr int LDA2 = NK2 * 4 + ((4 - (NK2 * 4) % 16) + 16) % 16;
  constexpr size_t smem = sizeof(double) * (NRT1 * 8 * LDA1 + 64 * LDA2 + (THREADS / 32) * NK2 * 4 * LDL);
  static bool configured = false;
  auto kern = leaf_down_kernel<NK1, NRT1, NK2, NT>;
  if (!configured) {
    HIKF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::max<size_t>(smem, 48 << 10)));
    configured = true;
  }
  kern<<<nleaves, THREADS, smem, st>>>(a);
  HIKF_CHECK_LAUNCH();
  return HIKF_OK;
}

// One 8-column tile per warp unit.  NT = 2 (every A fragment feeds two DMMAs; 168 registers, 3 CTAs
// of 4 warps) was measured equal and is not instantiated.
template <int NK1, int NRT1, int NK2>
int launch_leaf_t(const LeafArgs& a, unsigned nleaves, cudaStream_t st) {
  return launch_leaf_nt<NK1, NRT1, NK2, 1>(a, nleaves, st);
}

// ---------------------------------------------------------------------------
// L2L of one level, child-major: one CTA per occupied child box (the L2L half of
// leaf_down_kernel).  l[a][j] = S[child][j][a] + sum_b C_ci[a][b] L_parent[b][j], stored
// box-major.  Against the parent-major box_warp_kernel (4 q rows in passes of 4 row tiles,
// each pass with its own dependent slot -> M2L-sum gathers and integer divisions) a unit is one
// DMMA pass over ceil(q / 8) accumulators with the M2L sums copied asynchronously into the
// warp's shared tile; the products and their order are the same, so the locals are bit-identical.
// ---------------------------------------------------------------------------
struct ChildArgs {
  int64_t n;
  int q, qp;
  int64_t G;  // child-level grid
  const int32_t* occ;  // occupied child boxes
  const double *Lp, *shift, *S;
  const int32_t* tmap;
  double* L;
  int64_t pxlo, pxhi;  // parents outside this box-column range are skipped (leaf-aligned shard)
  unsigned long long* flops;
};

template <int NK1, int NRT1>
__global__ void __launch_bounds__(BW_THREADS, 2) l2l_child_kernel(ChildArgs g) {
  extern __shared__ double sm[];
  constexpr int LDA1 = NK1 * 4 + ((4 - (NK1 * 4) % 16) + 16) % 16;
  constexpr int TR = NRT1 * 8;  // rows of the per-warp tile
  double* A1 = sm;              // TR x LDA1
  double* Lw = A1 + TR * LDA1;  // 8 warps x TR x 8
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, t4 = lane & 3;
  const int q = g.q, qp = g.qp;
  const int64_t box = g.occ[blockIdx.x];
  const int64_t X = box / g.G, Y = box % g.G;
  if ((X >> 1) < g.pxlo || (X >> 1) > g.pxhi) return;  // CTA-uniform
  const int ci = (int)(((X & 1) << 1) | (Y & 1));
  const int64_t P = (X >> 1) * (g.G >> 1) + (Y >> 1);
  const double* Cg = g.shift + (int64_t)ci * q * qp;
  for (int e = tid; e < TR * NK1 * 4; e += BW_THREADS) {
    const int r = e / (NK1 * 4), k = e % (NK1 * 4);
    const bool ok = r < q && k < qp;
    cp_async8_zfill(A1 + r * LDA1 + k, ok ? Cg + (int64_t)r * qp + k : Cg, ok);
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  double* lw = Lw + warp * TR * 8;
  const int64_t n = g.n;
  const int64_t ncb = (n + 7) / 8;
  const double* Lpar = g.Lp + P * qp * n;
  const int32_t* tm = g.tmap + box * n;
  double* Lout = g.L + box * q * n;
  auto load_next = [&](int64_t u, double (&b1)[NK1], int32_t (&sl)[2]) {
    const int64_t jb = u * 8 + gq;
    // one running row pointer (opaque to the compiler: NK1 hoisted row addresses would cost 2 NK1 registers)
    const double* pr = Lpar + (int64_t)t4 * n + (jb < n ? jb : 0);
    asm volatile("" : "+l"(pr));
#pragma unroll
    for (int k4 = 0; k4 < NK1; ++k4) {
      const int k = k4 * 4 + t4;
      b1[k4] = (k < qp && jb < n) ? *pr : 0.0;
      pr += 4 * n;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t jc = u * 8 + 2 * t4 + h;
      sl[h] = jc < n ? tm[jc] : -1;
    }
  };
  constexpr int kStep = BW_THREADS / 32;
  unsigned long long useful = 0;
  double nb1[NK1];
  int32_t nslot[2];
  if (warp < ncb) load_next(warp, nb1, nslot);
  for (int64_t u = warp; u < ncb; u += kStep) {
    double b1[NK1];
    const int32_t slot[2] = {nslot[0], nslot[1]};
#pragma unroll
    for (int k4 = 0; k4 < NK1; ++k4) b1[k4] = nb1[k4];
    // the M2L sums: asynchronous copies into the positions this thread adds its results to
#pragma unroll
    for (int i = 0; i < NRT1; ++i) {
      const int r = i * 8 + gq;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const bool ok = r < q && slot[h] >= 0;
        cp_async8_zfill(lw + r * 8 + 2 * t4 + h, ok ? g.S + (int64_t)slot[h] * q + r : g.S, ok);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (u + kStep < ncb) load_next(u + kStep, nb1, nslot);
    const int64_t j0 = u * 8;
    if (lane == 0) useful += 2ull * q * qp * (unsigned long long)(n - j0 < 8 ? n - j0 : 8);
    double acc[NRT1][2];
#pragma unroll
    for (int i = 0; i < NRT1; ++i) acc[i][0] = acc[i][1] = 0.0;
#pragma unroll
    for (int k4 = 0; k4 < NK1; ++k4)
#pragma unroll
      for (int i = 0; i < NRT1; ++i) {
        const double af = lds64(A1 + (i * 8 + gq) * LDA1 + k4 * 4 + t4);
        dmma884(acc[i][0], acc[i][1], af, b1[k4]);
      }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    const int64_t jc = j0 + 2 * t4;
#pragma unroll
    for (int i = 0; i < NRT1; ++i) {
      const int r = i * 8 + gq;
      if (r >= q) continue;
      const double2 in = *reinterpret_cast<const double2*>(lw + r * 8 + 2 * t4);
      const double v0 = acc[i][0] + in.x, v1 = acc[i][1] + in.y;
      double* o = Lout + (int64_t)r * n;
      if (jc + 1 < n && (((uintptr_t)(o + jc)) & 15) == 0) {
        *reinterpret_cast<double2*>(o + jc) = make_double2(v0, v1);
      } else {
        if (jc < n) o[jc] = v0;
        if (jc + 1 < n) o[jc + 1] = v1;
      }
    }
  }
  if (g.flops && lane == 0 && useful) atomicAdd(g.flops, useful);
}

template <int NK1, int NRT1>
int launch_child_t(const ChildArgs& a, unsigned nboxes, cudaStream_t st) {
  constexpr int LDA1 = NK1 * 4 + ((4 - (NK1 * 4) % 16) + 16) % 16;
  constexpr size_t smem = sizeof(double) * (NRT1 * 8 * LDA1 + (BW_THREADS / 32) * NRT1 * 8 * 8);
  static bool configured = false;
  auto kern = l2l_child_kernel<NK1, NRT1>;
  if (!configured) {
    HIKF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::max<size_t>(smem, 48 << 10)));
    configured = true;
  }
  kern<<<nboxes, BW_THREADS, smem, st>>>(a);
  HIKF_CHECK_LAUNCH();
  return HIKF_OK;
}

// (child order o, parent order op) -> instantiation; -1 = not instantiated
int launch_child(const ChildArgs& a, int o, int op, unsigned nboxes, cudaStream_t st) {
#define HIKF_CHILD(O, OP) \
  if (o == O && op == OP) return launch_child_t<(OP * OP + 3) / 4, (O * O + 7) / 8>(a, nboxes, st);
  HIKF_CHILD(2, 2) HIKF_CHILD(2, 3) HIKF_CHILD(3, 3) HIKF_CHILD(3, 4) HIKF_CHILD(4, 4) HIKF_CHILD(4, 5)
  HIKF_CHILD(5, 5) HIKF_CHILD(5, 6) HIKF_CHILD(6, 6) HIKF_CHILD(6, 7) HIKF_CHILD(7, 7) HIKF_CHILD(7, 8)
  HIKF_CHILD(8, 8)
#undef HIKF_CHILD
  return -1;
}

// (leaf order o, parent order op) -> instantiation; 0 = not instantiated
int launch_leaf(const LeafArgs& a, int o, int op, unsigned nleaves, cudaStream_t st) {
#define HIKF_LEAF(O, OP)                                                                        \
  if (o == O && op == OP)                                                                       \
    return launch_leaf_t<(OP * OP + 3) / 4, (O * O + 7) / 8, (O * O + 3) / 4>(a, nleaves, st);
  HIKF_LEAF(2, 2) HIKF_LEAF(2, 3) HIKF_LEAF(3, 3) HIKF_LEAF(3, 4) HIKF_LEAF(4, 4) HIKF_LEAF(4, 5)
  HIKF_LEAF(5, 5) HIKF_LEAF(5, 6) HIKF_LEAF(6, 6) HIKF_LEAF(6, 7) HIKF_LEAF(7, 7) HIKF_LEAF(7, 8)
  HIKF_LEAF(8, 8)
#undef HIKF_LEAF
  return -1;
}

}  // namespace

bool box_supported(int rows, int K) { return K <= 4 * BW_MAXK4 && box_smem(rows, K) <= 200 * 1024; }

static int g_l2l_child = -1;  // child-major L2L (1, default) or the parent-major box kernel (0: HIKF_L2L_CHILD=0, tuning key 4)
static bool l2l_child_major() {
  if (g_l2l_child < 0) {
    const char* e = getenv("HIKF_L2L_CHILD");
    g_l2l_child = (e && e[0] == '0') ? 0 : 1;
  }
  return g_l2l_child != 0;
}
int l2l_set_child_major(int on) {
  const int prev = l2l_child_major() ? 1 : 0;
  g_l2l_child = on ? 1 : 0;
  return prev;
}

int l2l_boxes(const hikf_tree* t, int l, const double* S, const int32_t* tmap, const double* Lp, int64_t n,
              double* L, cudaStream_t st, int64_t pxlo, int64_t pxhi) {
  if (t->n_occ[l - 1] == 0 || n == 0) return HIKF_OK;
  if (l2l_child_major() && t->n_occ[l] > 0) {
    ChildArgs c{};
    c.n = n;
    c.q = t->orders[l] * t->orders[l];
    c.qp = t->orders[l - 1] * t->orders[l - 1];
    c.G = (int64_t)1 << l;
    c.occ = t->occ[l];
    c.Lp = Lp;
    c.shift = t->shift[l - 1];
    c.S = S;
    c.tmap = tmap;
    c.L = L;
    c.pxlo = pxlo;
    c.pxhi = pxhi;
    c.flops = prof_flops_ptr(ST_L2L);
    const int s = launch_child(c, t->orders[l], t->orders[l - 1], (unsigned)t->n_occ[l], st);
    if (s >= 0) return s;  // else: orders without a child-major instantiation
  }
  BoxArgs a{};
  a.tmap = tmap;
  a.pxlo = pxlo;
  a.pxhi = pxhi;
  a.s0 = -1;
  a.mode = 0;
  a.n = n;
  a.q = t->orders[l] * t->orders[l];
  a.K = t->orders[l - 1] * t->orders[l - 1];
  a.occp = t->occ[l - 1];
  a.nparents = t->n_occ[l - 1];
  a.Gp = (int64_t)1 << (l - 1);
  a.Lp = Lp;
  a.shift = t->shift[l - 1];
  a.S = S;
  a.L = L;
  a.flops = prof_flops_ptr(ST_L2L);
  const int64_t units = a.nparents * ((n + 7) / 8);
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((units + 7) / 8, (int64_t)num_sms() * 8));
  return launch_box(a, 4 * a.q, dim3((unsigned)blocks), st);
}

int l2p_boxes(const hikf_tree* t, const double* Lleaf, int64_t n, double* U, int64_t ldu, cudaStream_t st,
              int64_t r0, int64_t r1, const LeafWindow* lw) {
  const int64_t l0 = lw ? lw->leaf0 : 0, l1 = lw ? lw->leaf1 : t->n_leaves;
  if (l1 <= l0 || n == 0) return HIKF_OK;
  BoxArgs a{};
  a.leaf0 = l0;
  a.s0 = lw ? lw->s0 : -1;
  a.r0 = r0;
  a.r1 = r1 < 0 ? INT64_MAX : r1;
  a.pxhi = INT64_MAX;
  a.mode = 1;
  a.n = n;
  a.K = t->orders[t->depth] * t->orders[t->depth];
  a.leaf_box = t->leaf_box;
  a.leaf_start = t->leaf_start;
  a.leaf_count = t->leaf_count;
  a.W2s = t->W2s;
  a.order = t->order;
  a.Lleaf = Lleaf;
  a.U = U;
  a.ldu = ldu;
  a.flops = prof_flops_ptr(ST_L2P);
  return launch_box(a, 64, dim3((unsigned)(l1 - l0), (unsigned)((t->max_count + 63) / 64)), st);
}

static int g_leaf_fused = -1;

bool leaf_fused_enabled() {
  if (g_leaf_fused < 0) {
    const char* e = getenv("HIKF_LEAF_FUSED");
    g_leaf_fused = (e && e[0] == '0') ? 0 : 1;
  }
  return g_leaf_fused != 0;
}

int leaf_set_fused(int on) {
  const int prev = leaf_fused_enabled() ? 1 : 0;
  g_leaf_fused = on ? 1 : 0;
  return prev;
}

bool leaf_down_supported(const hikf_tree* t) {
  const int D = t->depth;
  if (D < 3 || t->max_count > 64) return false;
  const int o = t->orders[D], op = t->orders[D - 1];
  return o >= 2 && o <= 8 && (op == o || op == o + 1);
}

bool leaf_down_adds_near(int64_t n) { return (n + 7) / 8 <= kLeafUnits; }

int leaf_down(const hikf_tree* t, const double* S, const int32_t* tmap, const double* Lp, int64_t n, double* U,
              int64_t ldu, cudaStream_t st, int64_t r0, int64_t r1, const LeafWindow* lw, const double* Pnear,
              const int64_t* items, const int32_t* item_start) {
  const int64_t l0 = lw ? lw->leaf0 : 0, l1 = lw ? lw->leaf1 : t->n_leaves;
  if (l1 <= l0 || n == 0) return HIKF_OK;
  const int D = t->depth;
  LeafArgs a{};
  a.n = n;
  a.q = t->orders[D] * t->orders[D];
  a.qp = t->orders[D - 1] * t->orders[D - 1];
  a.G = (int64_t)1 << D;
  a.leaf_box = t->leaf_box;
  a.leaf_start = t->leaf_start;
  a.leaf_count = t->leaf_count;
  a.W2s = t->W2s;
  a.order = t->order;
  a.Lp = Lp;
  a.shift = t->shift[D - 1];
  a.S = S;
  a.tmap = tmap;
  a.U = U;
  a.ldu = ldu;
  a.r0 = r0;
  a.r1 = r1 < 0 ? INT64_MAX : r1;
  a.leaf0 = l0;
  a.s0 = lw ? lw->s0 : -1;
  a.fl_l2l = prof_flops_ptr(ST_L2L);
  a.fl_l2p = prof_flops_ptr(ST_L2P);
  if (Pnear && !leaf_down_adds_near(n)) {
    set_error("fused leaf step: near-field fold supports n <= %d", 8 * kLeafUnits);
    return HIKF_BAD_ARGUMENT;
  }
  a.Pnear = Pnear;
  a.items = items;
  a.item_start = item_start;
  a.maxc = (int32_t)t->max_count;
  const int s = launch_leaf(a, t->orders[D], t->orders[D - 1], (unsigned)(l1 - l0), st);
  if (s < 0) {
    set_error("fused leaf downward step: orders (%d, %d) not instantiated", t->orders[D], t->orders[D - 1]);
    return HIKF_BAD_ARGUMENT;
  }
  return s;
}

}  // namespace hikf

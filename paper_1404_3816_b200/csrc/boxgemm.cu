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
  const double* S;         // pair-major M2L scratch of the child level
  double* L;               // child locals (box-major)
  // L2P
  const int32_t *leaf_box, *leaf_start, *leaf_count;
  const double* W2s;
  const int64_t* order;
  const double* Lleaf;
  double* U;
  int64_t ldu;
  int64_t r0, r1;  // L2P row window: only original rows in [r0, r1) are written, at U + (row - r0) ldu
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
    const int cnt = g.leaf_count[blockIdx.x];
    if (row_off >= cnt) return;
    R = min(64, cnt - row_off);
    Ag = g.W2s + (int64_t)(g.leaf_start[blockIdx.x] + row_off) * K;
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
    const int64_t task = MODE == 0 ? u / ncb : blockIdx.x;
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
    const int64_t task = MODE == 0 ? u / ncb : blockIdx.x;
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
            const int64_t irow = child_of(r, a) * g.n * g.q + a;
#pragma unroll
            for (int c = 0; c < CW; ++c)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int64_t jc = j0 + 8 * c + 2 * t4 + h;
                if (jc < g.n) init[i][c][h] = g.S[irow + jc * g.q];
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
          const int64_t orw = g.order[g.leaf_start[task] + row_off + r];
          if (orw < g.r0 || orw >= g.r1) continue;
          orow = g.U + (orw - g.r0) * g.ldu;
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

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

template <int K4>
int launch_box_k(const BoxArgs& a, dim3 grid, size_t smem, cudaStream_t st) {
  // tuning knobs (profiles/r01_box_sweep.log): column tiles per unit (CW) per mode; the
  // L2L uses 4 row tiles per pass with the B prefetch, the L2P 8
  static const int cw0 = env_int("HIKF_BOX_CW0", 1), cw1 = env_int("HIKF_BOX_CW1", 1);
  if (a.mode == 0)
    return cw0 == 2 ? launch_box_t<K4, 4, 0, false, 2>(a, grid, smem, st)
                    : launch_box_t<K4, 4, 0, true, 1>(a, grid, smem, st);
  return cw1 == 2 ? launch_box_t<K4, 8, 1, false, 2>(a, grid, smem, st) : launch_box_t<K4, 8, 1, true, 1>(a, grid, smem, st);
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

}  // namespace

bool box_supported(int rows, int K) { return K <= 4 * BW_MAXK4 && box_smem(rows, K) <= 200 * 1024; }

int l2l_boxes(const hikf_tree* t, int l, const double* S, const double* Lp, int64_t n, double* L, cudaStream_t st) {
  if (t->n_occ[l - 1] == 0 || n == 0) return HIKF_OK;
  BoxArgs a{};
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
              int64_t r0, int64_t r1) {
  if (t->n_leaves == 0 || n == 0) return HIKF_OK;
  BoxArgs a{};
  a.r0 = r0;
  a.r1 = r1 < 0 ? INT64_MAX : r1;
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
  return launch_box(a, 64, dim3((unsigned)t->n_leaves, (unsigned)((t->max_count + 63) / 64)), st);
}

}  // namespace hikf

// Fused n x n chain of the per-step update (filters.py:144-156, linalg.py:30-37)
// for n <= NN_FUSED_MAX: one cooperative launch runs a whole phase program.
//
// The multi-launch chain (update.cu: build_S, the recursive chol_inv with 64 x 64
// base blocks and DMMA GEMMs, the transpose, S^-1 = Li^T Li, the HC chain and
// the look-ahead) is about 40 dependent launches per step.  At small n each is
// a few microseconds of latency for almost no work, so at cfg1 / cfg2 the chain,
// not the m x n GEMM, set the step time.  Here the same operations are a
// program of phases -- lists of 64 x 64 GEMM tiles, Cholesky base blocks and
// grid-strided elementwise passes -- executed by one persistent cooperative
// grid with a grid barrier between phases.
//
// Bit-identical to the multi-launch chain: each GEMM tile accumulates every
// output element over k in ascending k4 groups from a multiple of 16 with the
// same DMMA instruction (the skipped triangle blocks of the library GEMM are
// exact zeros), the epilogues are alpha acc (+ beta Cin) as in dgemm.cu, and
// the base blocks run the same device function (chol_block.cuh).
//
// The look-ahead probe is on the device: the pre program compares HC / HC_Q
// with the look-ahead's inputs and takes the hit or miss branch itself, so the
// update needs no host round trip before its GEMM.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <tuple>

#include "chol_block.cuh"
#include "nnchain.h"

namespace cg = cooperative_groups;

namespace hikf {

namespace {

constexpr int kThreads = 256;
constexpr int TILE = 64;   // GEMM output tile (64 x 64), 8 warps of 32 x 16
constexpr int KC = 32;     // k-chunk staged in shared memory
constexpr int AS = KC + 4; // == 4 (mod 16) doubles: conflict-free fragment loads
constexpr int BS = TILE + 4;
constexpr int STG = TILE * AS + KC * BS;
constexpr size_t GEMM_SMEM = 2 * STG * sizeof(double);
constexpr size_t PROG_SMEM = GEMM_SMEM > CHOL_SMEM ? GEMM_SMEM : CHOL_SMEM;

enum : int16_t {
  K_GEMM = 0,    // one 64 x 64 tile of C = alpha A B (+ beta Cin)
  K_CHOL,        // one base block (chol_inv_block)
  K_ADD,         // grid: c = a + b (count elements)
  K_BUILD_S,     // grid: c = 0.5 ((a + r I) + (a + r I)^T), n x n
  K_TRANSPOSE,   // grid: c = a^T, n x n
  K_COPY,        // grid: c = a
  K_ZERO,        // grid: c = 0
  K_DIFF,        // grid: flag |= bits(a) != bits(b)
  K_ICOPY,       // grid: int c = int a (count)
  K_IZERO,       // grid: int c = 0 (count)
  K_INNOV,       // grid: innov = z - H mean (one warp per row)
};

struct NnTask {
  int16_t kind = 0;
  int16_t a = -1, b = -1, c = -1, cin = -1;  // buffer ids (int buffers for K_ICOPY / K_IZERO / K_CHOL status)
  int64_t offA = 0, offB = 0, offC = 0, offCin = 0;
  int64_t i0 = 0, j0 = 0;            // GEMM tile origin
  int64_t M = 0, N = 0, kbeg = 0, kend = 0;  // GEMM bounds (rows, cols, k range); elementwise: count in M
  int64_t sa_r = 0, sa_c = 1, sb_r = 0, sb_c = 1, ldc = 0, ldcin = 0;
  double alpha = 1.0, beta = 0.0;
  int64_t ld = 0, pivot = 0;          // K_CHOL: leading dimension, global pivot offset (nb in M)
};

__device__ __forceinline__ bool is_grid_task(int k) { return k >= K_ADD; }

// ---- 64 x 64 GEMM tile: all 256 threads, register-prefetched two-stage smem ring ----
__device__ void gemm_tile(const NnTask& t, const NnPtrs& p, double* sm) {
  const double* A = p.d[t.a] + t.offA;
  const double* B = p.d[t.b] + t.offB;
  double* C = p.d[t.c] + t.offC;
  const double* Cin = t.cin >= 0 ? p.d[t.cin] + t.offCin : nullptr;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1, gq = lane >> 2, t4 = lane & 3;
  const bool arow = t.sa_c == 1, brow = t.sb_c == 1;
  const int64_t span = t.kend - t.kbeg;
  const int nch = span > 0 ? (int)((span + KC - 1) / KC) : 0;
  double ra[8], rb[8];
  auto gload = [&](int c) {
    const int64_t k0 = t.kbeg + (int64_t)c * KC;
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int e = tid + it * kThreads;
      const int r = arow ? e / KC : e % TILE, kk = arow ? e % KC : e / TILE;
      const int64_t row = t.i0 + r, k = k0 + kk;
      ra[it] = (row < t.M && k < t.kend) ? A[row * t.sa_r + k * t.sa_c] : 0.0;
      const int kb = brow ? e / TILE : e % KC, cc = brow ? e % TILE : e / KC;
      const int64_t kb2 = k0 + kb, col = t.j0 + cc;
      rb[it] = (kb2 < t.kend && col < t.N) ? B[kb2 * t.sb_r + col * t.sb_c] : 0.0;
    }
  };
  auto sstore = [&](int stage) {
    double* As = sm + stage * STG;
    double* Bs = As + TILE * AS;
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int e = tid + it * kThreads;
      const int r = arow ? e / KC : e % TILE, kk = arow ? e % KC : e / TILE;
      As[r * AS + kk] = ra[it];
      const int kb = brow ? e / TILE : e % KC, cc = brow ? e % TILE : e / KC;
      Bs[kb * BS + cc] = rb[it];
    }
  };
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if (nch > 0) {
    gload(0);
    sstore(0);
  }
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) gload(c + 1);
    const double* As = sm + (c & 1) * STG + (wm * 32 + gq) * AS + t4;
    const double* Bs = sm + (c & 1) * STG + TILE * AS + t4 * BS + wn * 16 + gq;
#pragma unroll
    for (int kb = 0; kb < KC; kb += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[i * 8 * AS + kb];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = Bs[kb * BS + j * 8];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if (c + 1 < nch) sstore((c + 1) & 1);
    __syncthreads();
  }
  // epilogue as dgemm.cu's gemm_epilogue: alpha acc + beta Cin, else alpha acc
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = t.i0 + wm * 32 + i * 8 + gq;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t col = t.j0 + wn * 16 + j * 8 + 2 * t4 + h;
        if (row < t.M && col < t.N) {
          double v;
          if (Cin) {
            const double cv = Cin[row * t.ldcin + col];
            v = t.alpha * acc[i][j][h] + t.beta * cv;
          } else {
            v = t.alpha * acc[i][j][h];
          }
          C[row * t.ldc + col] = v;
        }
      }
  }
  __syncthreads();  // the next task reuses the ring
}

// ---- grid-strided elementwise tasks (every CTA takes its share) ----
__device__ void grid_task(const NnTask& t, const NnPtrs& p) {
  const int64_t g0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gs = (int64_t)gridDim.x * blockDim.x;
  const int64_t cnt = t.M, n = p.n;
  switch (t.kind) {
    case K_ADD: {  // 4 independent elements per thread in flight (the grid is small)
      const double* __restrict__ a = p.d[t.a];
      const double* __restrict__ b = p.d[t.b];
      double* __restrict__ c = p.d[t.c];
      int64_t e = g0;
      for (; e + 3 * gs < cnt; e += 4 * gs) {
        double x[4], y[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = a[e + u * gs], y[u] = b[e + u * gs];
#pragma unroll
        for (int u = 0; u < 4; ++u) c[e + u * gs] = x[u] + y[u];
      }
      for (; e < cnt; e += gs) c[e] = a[e] + b[e];
      break;
    }
    case K_BUILD_S: {  // update.cu build_S
      const double* __restrict__ HC = p.d[t.a];
      double* __restrict__ S = p.d[t.c];
      int64_t e = g0;
      for (; e + 3 * gs < n * n; e += 4 * gs) {
        double x[4], y[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t i = (e + u * gs) / n, j = (e + u * gs) % n;
          x[u] = HC[i * n + j];
          y[u] = HC[j * n + i];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t i = (e + u * gs) / n, j = (e + u * gs) % n;
          double a = x[u], b = y[u];
          if (i == j) {
            a = a + p.r;
            b = b + p.r;
          }
          S[e + u * gs] = 0.5 * (a + b);
        }
      }
      for (; e < n * n; e += gs) {
        const int64_t i = e / n, j = e % n;
        double a = HC[i * n + j], b = HC[j * n + i];
        if (i == j) {
          a = a + p.r;
          b = b + p.r;
        }
        S[e] = 0.5 * (a + b);
      }
      break;
    }
    case K_TRANSPOSE: {
      const double* X = p.d[t.a];
      double* Y = p.d[t.c];
      for (int64_t e = g0; e < n * n; e += gs) {
        const int64_t i = e / n, j = e % n;
        Y[j * n + i] = X[e];
      }
      break;
    }
    case K_COPY: {
      const double* __restrict__ a = p.d[t.a];
      double* __restrict__ c = p.d[t.c];
      int64_t e = g0;
      for (; e + 3 * gs < cnt; e += 4 * gs) {
        double x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = a[e + u * gs];
#pragma unroll
        for (int u = 0; u < 4; ++u) c[e + u * gs] = x[u];
      }
      for (; e < cnt; e += gs) c[e] = a[e];
      break;
    }
    case K_ZERO: {
      double* c = p.d[t.c];
      for (int64_t e = g0; e < cnt; e += gs) c[e] = 0.0;
      break;
    }
    case K_DIFF: {
      const uint64_t* __restrict__ a = reinterpret_cast<const uint64_t*>(p.d[t.a]);
      const uint64_t* __restrict__ b = reinterpret_cast<const uint64_t*>(p.d[t.b]);
      uint64_t d = 0;
      int64_t e = g0;
      for (; e + 3 * gs < cnt; e += 4 * gs)
#pragma unroll
        for (int u = 0; u < 4; ++u) d |= a[e + u * gs] ^ b[e + u * gs];
      for (; e < cnt; e += gs) d |= a[e] ^ b[e];
      if (__syncthreads_or(d != 0) && threadIdx.x == 0) atomicOr(p.i[NI_FLAG], 1);
      break;
    }
    case K_ICOPY: {
      for (int64_t e = g0; e < cnt; e += gs) p.i[t.c][e] = p.i[t.a][e];
      break;
    }
    case K_IZERO: {
      for (int64_t e = g0; e < cnt; e += gs) p.i[t.c][e] = 0;
      break;
    }
    case K_INNOV: {  // update.cu innovation, one warp per row
      const int lane = threadIdx.x & 31;
      for (int64_t row = g0 >> 5; row < n; row += gs >> 5) {
        double s = 0.0;
        if (p.Hmean) {
          s = p.Hmean[row];
        } else {
          for (int64_t e = p.ip[row] + lane; e < p.ip[row + 1]; e += 32) s += p.val[e] * p.mean[p.ix[e]];
          for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        }
        if (lane == 0) p.innov[row] = p.z[row] - s;
      }
      break;
    }
    default:
      break;
  }
}

// cond: 0 always, 1 only on a look-ahead miss, 2 only on a hit.  The flag is
// written in phase 0 only, so every CTA takes the same branches (and the same
// number of grid barriers).
__global__ void __launch_bounds__(kThreads, 1) nn_program_kernel(const NnTask* __restrict__ tasks,
                                                                  const int* __restrict__ phase_off,
                                                                  const int* __restrict__ phase_cond, int nphases,
                                                                  NnPtrs p) {
  extern __shared__ __align__(16) double nn_smem[];
  cg::grid_group grid = cg::this_grid();
  bool synced = true;
  for (int ph = 0; ph < nphases; ++ph) {
    const int cond = phase_cond[ph];
    if (cond) {
      if (!synced) {
        grid.sync();
        synced = true;
      }
      const bool miss = p.force_miss || __ldcg(p.i[NI_FLAG]) != 0;
      if ((cond == 1) != miss) continue;
    }
    if (!synced) grid.sync();
    synced = false;
    int tile = 0;
    for (int ti = phase_off[ph]; ti < phase_off[ph + 1]; ++ti) {
      const NnTask& t = tasks[ti];
      if (is_grid_task(t.kind)) {
        grid_task(t, p);
        continue;
      }
      if ((tile++ % (int)gridDim.x) != (int)blockIdx.x) continue;
      if (t.kind == K_GEMM) {
        gemm_tile(t, p, nn_smem);
      } else {  // K_CHOL
        chol_inv_block(p.d[t.a] + t.offA, t.ld, (int)t.M, t.pivot, p.d[t.b] + t.offB, p.d[t.c] + t.offC,
                       p.i[t.cin], nn_smem);
        __syncthreads();
      }
    }
  }
}

// ---------------------------------------------------------------------------
// program construction (host)
// ---------------------------------------------------------------------------
struct Program {
  std::vector<NnTask> tasks;
  std::vector<int> off{0}, cond;
  int max_tiles = 1;
  int cur = 0, cur_tiles = 0;
  void task(const NnTask& t) {
    tasks.push_back(t);
    if (t.kind == K_GEMM || t.kind == K_CHOL) max_tiles = std::max(max_tiles, ++cur_tiles);
  }
  void phase(int c = 0) {  // close the current phase (taken under condition c)
    off.push_back((int)tasks.size());
    cond.push_back(c);
    cur_tiles = 0;
  }
};

NnTask ew(int16_t kind, int16_t a, int16_t b, int16_t c, int64_t count) {
  NnTask t;
  t.kind = kind;
  t.a = a;
  t.b = b;
  t.c = c;
  t.M = count;
  return t;
}

// C (M x N) = alpha A (M x K) B (K x N) [+ beta Cin], split into 64 x 64 tiles;
// kmode as dgemm: KB_UPPER (B upper triangular: k < j0 + 64), KB_LOWER (k >= j0 rounded to 16)
enum { TK_FULL = 0, TK_UPPER = 1, TK_LOWER = 2 };
void gemm(Program& P, int64_t M, int64_t N, int64_t K, int16_t a, int64_t offA, int64_t sa_r, int64_t sa_c, int16_t b,
          int64_t offB, int64_t sb_r, int64_t sb_c, int16_t c, int64_t offC, int64_t ldc, double alpha = 1.0,
          int16_t cin = -1, int64_t offCin = 0, int64_t ldcin = 0, double beta = 0.0, int kmode = TK_FULL) {
  for (int64_t i0 = 0; i0 < M; i0 += TILE)
    for (int64_t j0 = 0; j0 < N; j0 += TILE) {
      NnTask t;
      t.kind = K_GEMM;
      t.a = a; t.offA = offA; t.sa_r = sa_r; t.sa_c = sa_c;
      t.b = b; t.offB = offB; t.sb_r = sb_r; t.sb_c = sb_c;
      t.c = c; t.offC = offC; t.ldc = ldc;
      t.cin = cin; t.offCin = offCin; t.ldcin = ldcin;
      t.alpha = alpha; t.beta = beta;
      t.i0 = i0; t.j0 = j0; t.M = M; t.N = N;
      t.kbeg = kmode == TK_LOWER ? (j0 / 16) * 16 : 0;
      t.kend = kmode == TK_UPPER ? std::min(K, j0 + TILE) : K;
      P.task(t);
    }
}

// update.cu chol_inv (recursive blocked Cholesky with inverse) as phases; the
// T = L21 Li11 product joins the S22 update's phase, so every recursion level
// keeps its own tmp slice (toff).
void chol_program(Program& P, int16_t S, int16_t L, int16_t Li, int16_t tmp, int16_t status, int64_t n, int64_t ld,
                  int64_t off, int64_t pivot, int64_t toff, int c) {
  if (n <= CHOL_NB) {
    NnTask t;
    t.kind = K_CHOL;
    t.a = S; t.offA = off;
    t.b = L; t.offB = off;
    t.c = Li; t.offC = off;
    t.cin = status;
    t.ld = ld;
    t.M = n;
    t.pivot = pivot;
    P.task(t);
    P.phase(c);
    return;
  }
  const int64_t n1 = ((n / 2 + CHOL_NB - 1) / CHOL_NB) * CHOL_NB, n2 = n - n1;
  const int64_t o11 = off, o21 = off + n1 * ld, o22 = off + n1 * ld + n1;
  chol_program(P, S, L, Li, tmp, status, n1, ld, o11, pivot, toff + n2 * n1, c);
  // L21 = S21 Li11^T
  gemm(P, n2, n1, n1, S, o21, ld, 1, Li, o11, 1, ld, L, o21, ld);
  P.phase(c);
  // S22 -= L21 L21^T ; T = L21 Li11
  gemm(P, n2, n2, n1, L, o21, ld, 1, L, o21, 1, ld, S, o22, ld, -1.0, S, o22, ld, 1.0);
  gemm(P, n2, n1, n1, L, o21, ld, 1, Li, o11, ld, 1, tmp, toff, n1);
  P.phase(c);
  chol_program(P, S, L, Li, tmp, status, n2, ld, o22, pivot + n1, toff + n2 * n1, c);
  // Li21 = -Li22 T
  gemm(P, n2, n1, n2, Li, o22, ld, 1, tmp, toff, n1, 1, Li, o21, ld, -1.0);
  P.phase(c);
}

// factorisation of S = sym(HCsrc) + r I into (L scratch, Li, LiT, Sinv, status)
void factor_program(Program& P, int16_t HCsrc, int16_t Li, int16_t LiT, int16_t Sinv, int16_t status, int64_t n,
                    int c) {
  P.task(ew(K_BUILD_S, HCsrc, -1, NB_S, n * n));
  P.task(ew(K_ZERO, -1, -1, NB_L, n * n));
  P.task(ew(K_ZERO, -1, -1, Li, n * n));
  P.phase(c);
  chol_program(P, NB_S, NB_L, Li, NB_TMP, status, n, n, 0, 0, 0, c);
  // S^-1 = Li^T Li (B lower triangular); A = Li^T read through transposed strides
  gemm(P, n, n, n, Li, 0, 1, n, Li, 0, n, 1, Sinv, 0, n, 1.0, -1, 0, 0, 0.0, TK_LOWER);
  P.task(ew(K_TRANSPOSE, Li, -1, LiT, n * n));
  P.phase(c);
}

Program pre_program(int64_t n, bool probe) {
  Program P;
  P.task(ew(K_IZERO, -1, -1, NI_STATUS, 4));  // the step's pivot / check / block-count words
  P.task(ew(K_ADD, NB_HC, NB_HCQ, NB_HCP, n * n));
  P.task(ew(K_INNOV, -1, -1, -1, n));
  if (probe) {
    P.task(ew(K_DIFF, NB_HC, NB_LA_HC, -1, n * n));
    P.task(ew(K_DIFF, NB_HCQ, NB_LA_HCQ, -1, n * n));
  }
  P.phase(0);
  // hit: this step's factor is the look-ahead's
  P.task(ew(K_COPY, NB_LA_LI, -1, NB_LI, n * n));
  P.task(ew(K_COPY, NB_LA_LIT, -1, NB_LIT, n * n));
  P.task(ew(K_COPY, NB_LA_SINV, -1, NB_SINV, n * n));
  P.task(ew(K_ICOPY, NI_LA_STATUS, -1, NI_STATUS, 1));
  P.phase(2);
  // miss: factorise in line
  factor_program(P, NB_HCP, NB_LI, NB_LIT, NB_SINV, NI_STATUS, n, 1);
  return P;
}

Program post_program(int64_t n, bool lookahead) {
  Program P;
  // P = Li HC', R = HC' Li^T (Li^T upper triangular, read through transposed strides)
  gemm(P, n, n, n, NB_LI, 0, n, 1, NB_HCP, 0, n, 1, NB_P, 0, n);
  gemm(P, n, n, n, NB_HCP, 0, n, 1, NB_LI, 0, 1, n, NB_R, 0, n, 1.0, -1, 0, 0, 0.0, TK_UPPER);
  P.phase(0);
  // HC_out = HC' - R P
  gemm(P, n, n, n, NB_R, 0, n, 1, NB_P, 0, n, 1, NB_HCOUT, 0, n, -1.0, NB_HCP, 0, n, 1.0);
  P.task(ew(K_IZERO, -1, -1, NI_FLAG, 1));  // the next step's probe flag (the pre program has used it)
  P.phase(0);
  if (!lookahead) return P;
  P.task(ew(K_ADD, NB_HCOUT, NB_HCQ, NB_LA_HCP, n * n));
  P.task(ew(K_COPY, NB_HCOUT, -1, NB_LA_HC, n * n));
  P.task(ew(K_COPY, NB_HCQ, -1, NB_LA_HCQ, n * n));
  P.task(ew(K_IZERO, -1, -1, NI_LA_STATUS, 1));
  P.phase(0);
  factor_program(P, NB_LA_HCP, NB_LA_LI, NB_LA_LIT, NB_LA_SINV, NI_LA_STATUS, n, 0);
  return P;
}

struct DevProgram {
  NnTask* tasks = nullptr;
  int *off = nullptr, *cond = nullptr;
  int nphases = 0, grid = 1;
};

int upload(const Program& P, DevProgram* d) {
  d->nphases = (int)P.cond.size();
  HIKF_CHECK_CUDA(cudaMalloc((void**)&d->tasks, sizeof(NnTask) * std::max<size_t>(1, P.tasks.size())));
  HIKF_CHECK_CUDA(cudaMalloc((void**)&d->off, sizeof(int) * P.off.size()));
  HIKF_CHECK_CUDA(cudaMalloc((void**)&d->cond, sizeof(int) * std::max<size_t>(1, P.cond.size())));
  HIKF_CHECK_CUDA(cudaMemcpy(d->tasks, P.tasks.data(), sizeof(NnTask) * P.tasks.size(), cudaMemcpyHostToDevice));
  HIKF_CHECK_CUDA(cudaMemcpy(d->off, P.off.data(), sizeof(int) * P.off.size(), cudaMemcpyHostToDevice));
  HIKF_CHECK_CUDA(cudaMemcpy(d->cond, P.cond.data(), sizeof(int) * P.cond.size(), cudaMemcpyHostToDevice));
  static int max_grid = 0;
  if (!max_grid) {
    HIKF_CHECK_CUDA(cudaFuncSetAttribute(nn_program_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)PROG_SMEM));
    int per_sm = 0;
    HIKF_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nn_program_kernel, kThreads, PROG_SMEM));
    max_grid = std::max(1, per_sm) * num_sms();
  }
  // enough CTAs for the widest phase, capped by co-residency (cooperative launch)
  d->grid = std::max(1, std::min({std::max(P.max_tiles, 32), max_grid, num_sms()}));
  return HIKF_OK;
}

int run(int kind, int64_t n, bool flag, const NnPtrs& p, cudaStream_t st) {
  static std::map<std::tuple<int, int, int64_t, bool>, DevProgram> cache;
  int dev = 0;
  HIKF_CHECK_CUDA(cudaGetDevice(&dev));
  auto key = std::make_tuple(dev, kind, n, flag);
  auto it = cache.find(key);
  if (it == cache.end()) {
    DevProgram d;
    HIKF_TRY(upload(kind == 0 ? pre_program(n, flag) : post_program(n, flag), &d));
    it = cache.emplace(key, d).first;
  }
  const DevProgram& d = it->second;
  NnPtrs pp = p;
  void* args[] = {(void*)&d.tasks, (void*)&d.off, (void*)&d.cond, (void*)&d.nphases, (void*)&pp};
  HIKF_CHECK_CUDA(cudaLaunchCooperativeKernel((void*)nn_program_kernel, dim3(d.grid), dim3(kThreads), args,
                                              PROG_SMEM, st));
  HIKF_CHECK_LAUNCH();
  return HIKF_OK;
}

}  // namespace

static int g_nn_fused = -1;

bool nn_fused_enabled(int64_t n) {
  if (g_nn_fused < 0) {
    const char* e = getenv("HIKF_NN_FUSED");
    g_nn_fused = (e && e[0] == '0') ? 0 : 1;
  }
  return g_nn_fused && n >= 1 && n <= NN_FUSED_MAX;
}

int nn_set_fused(int on) {
  nn_fused_enabled(1);
  const int prev = g_nn_fused;
  g_nn_fused = on ? 1 : 0;
  return prev;
}

int nn_pre(const NnPtrs& p, bool probe, cudaStream_t st) { return run(0, p.n, probe, p, st); }

int nn_post(const NnPtrs& p, bool lookahead, cudaStream_t st) { return run(1, p.n, lookahead, p, st); }

}  // namespace hikf

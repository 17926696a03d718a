// FP64 DMMA GEMM (see dgemm.cuh).  One templated kernel; the tile shape is
// a compile-time variant (dgemm_variant() picks it; HIKF_DGEMM_VARIANT
// overrides for tuning sweeps).
#include <algorithm>
#include <cstdlib>

#include "dgemm.cuh"

// CUTLASS 2.x SM80 FP64 tensor-op threadblock mainloop (headers only; the
// tree vendored with flashinfer, see Makefile CUTLASS_INC).  Used as the
// mainloop of the K-GEMM variant below; the epilogue is ours.
#include "cutlass/gemm/gemm.h"
#include "cutlass/gemm/threadblock/default_mma.h"
#include "cutlass/layout/matrix.h"

namespace hikf {

namespace {

// Shared epilogue: alpha/beta, fused row partials, stores.  Accumulator
// acc[i][j][h] holds C[row = i*8 + gq][col] of the warp tile with
//   SPLIT = false: col = j*8 + 2 t4 + h        (8-column DMMA tiles)
//   SPLIT = true:  col = (2 t4 + h) * TN + j   (interleaved tiles: each thread
//                  owns two runs of TN contiguous columns)
template <int BM, int BN, int WM, int WN, bool PARTIALS, bool SPLIT = false>
__device__ __forceinline__ void gemm_epilogue(const GemmArgs& g, double (&acc)[BM / WM / 8][BN / WN / 8][2], double* C,
                                              const double* Cin, int64_t m0, int64_t n0, int tid, int wm, int wn,
                                              int gq, int t4, double (*red_sq)[PARTIALS ? BM : 1],
                                              double (*red_dot)[PARTIALS ? BM : 1]) {
  constexpr int THREADS = WM * WN * 32;
  constexpr int TM = BM / WM / 8;
  constexpr int TN = BN / WN / 8;
  const int64_t cw = n0 + wn * TN * 8;
  auto colh = [&](int j, int h) -> int64_t { return cw + (SPLIT ? (2 * t4 + h) * TN + j : j * 8 + 2 * t4 + h); };
  // beta * Cin is read for the whole warp tile before any store: C may alias
  // Cin (in-place C_new = C' - Y P), and separating the phases lets the loads
  // overlap instead of serialising load -> store round trips.
  if (Cin) {
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int64_t row = m0 + wm * TM * 8 + i * 8 + gq;
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t col = colh(j, h);
          double c = 0.0;
          if (row < g.M && col < g.N) c = Cin[row * g.ldcin + col];
          acc[i][j][h] = g.alpha * acc[i][j][h] + g.beta * c;
        }
    }
  }
  // row partials first (they read w / px), then the stores: keeping the
  // loads ahead of the stores avoids load-after-store serialisation on
  // possibly aliasing pointers
  if (PARTIALS) {
    const double sc = g.px ? 1.0 : (Cin ? 1.0 : g.alpha);
    if (g.sp_ip) {  // sparse-row addend (see GemmArgs): folded into the accumulators first
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const int64_t row = m0 + wm * TM * 8 + i * 8 + gq;
        if (row >= g.M) continue;
        const int32_t e0 = g.sp_ip[row], e1 = g.sp_ip[row + 1];
        for (int32_t e = e0; e < e1; ++e) {
          const double w = g.sp_alpha * g.sp_val[e];
          const double* yr = g.sp_Y + (int64_t)g.sp_ix[e] * g.sp_ldy;
#pragma unroll
          for (int j = 0; j < TN; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int64_t col = colh(j, h);
              if (col < g.N) acc[i][j][h] = fma(w, yr[col], acc[i][j][h]);
            }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int rl = wm * TM * 8 + i * 8 + gq;
      const int64_t row = m0 + rl;
      double ssq = 0.0, sdot = 0.0;
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t col = colh(j, h);
          if (row < g.M && col < g.N) {
            const double v = sc * acc[i][j][h];
            ssq += v * (g.px ? g.px[row * g.ldx + col] : v);
            if (g.w) sdot += v * g.w[col];
          }
        }
      ssq += __shfl_xor_sync(0xffffffffu, ssq, 1);
      ssq += __shfl_xor_sync(0xffffffffu, ssq, 2);
      sdot += __shfl_xor_sync(0xffffffffu, sdot, 1);
      sdot += __shfl_xor_sync(0xffffffffu, sdot, 2);
      if (t4 == 0) {
        red_sq[wn][rl] = ssq;
        red_dot[wn][rl] = sdot;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < TM && C; ++i) {  // C == null: partials only (no output store)
    const int64_t row = m0 + wm * TM * 8 + i * 8 + gq;
    if (SPLIT && (TN % 2 == 0) && row < g.M && cw + BN / WN <= g.N && g.ldc % 2 == 0 && ((uintptr_t)C & 15) == 0) {
      // two runs of TN contiguous columns: 16-byte stores
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int j = 0; j < TN; j += 2) {
          const double v0 = Cin ? acc[i][j][h] : g.alpha * acc[i][j][h];
          const double v1 = Cin ? acc[i][j + 1][h] : g.alpha * acc[i][j + 1][h];
          *reinterpret_cast<double2*>(C + row * g.ldc + colh(j, h)) = make_double2(v0, v1);
        }
    } else if (g.chain_out) {
      // also emit chain_out = C + chain_add (the next step's predict, fused);
      // columns 2 t4 and 2 t4 + 1 are adjacent: 16-byte accesses when aligned
      const bool v16 = !SPLIT && row < g.M && cw + BN / WN <= g.N && (g.ldc | g.ldch) % 2 == 0 &&
                       (((uintptr_t)C | (uintptr_t)g.chain_out | (uintptr_t)g.chain_add) & 15) == 0;
      if (v16) {
        double2 cv[TN];
#pragma unroll
        for (int j = 0; j < TN; ++j)
          cv[j] = *reinterpret_cast<const double2*>(g.chain_add + row * g.ldch + colh(j, 0));
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          const double v0 = Cin ? acc[i][j][0] : g.alpha * acc[i][j][0];
          const double v1 = Cin ? acc[i][j][1] : g.alpha * acc[i][j][1];
          *reinterpret_cast<double2*>(C + row * g.ldc + colh(j, 0)) = make_double2(v0, v1);
          *reinterpret_cast<double2*>(g.chain_out + row * g.ldch + colh(j, 0)) =
              make_double2(v0 + cv[j].x, v1 + cv[j].y);
        }
      } else {
        double cv[TN][2];
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t col = colh(j, h);
            cv[j][h] = (row < g.M && col < g.N) ? g.chain_add[row * g.ldch + col] : 0.0;
          }
#pragma unroll
        for (int j = 0; j < TN; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t col = colh(j, h);
            if (row < g.M && col < g.N) {
              const double v = Cin ? acc[i][j][h] : g.alpha * acc[i][j][h];
              C[row * g.ldc + col] = v;
              g.chain_out[row * g.ldch + col] = v + cv[j][h];
            }
          }
      }
    } else if (!SPLIT && row < g.M && cw + BN / WN <= g.N && g.ldc % 2 == 0 && ((uintptr_t)C & 15) == 0) {
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const double v0 = Cin ? acc[i][j][0] : g.alpha * acc[i][j][0];
        const double v1 = Cin ? acc[i][j][1] : g.alpha * acc[i][j][1];
        *reinterpret_cast<double2*>(C + row * g.ldc + colh(j, 0)) = make_double2(v0, v1);
      }
    } else {
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t col = colh(j, h);
          if (row < g.M && col < g.N) C[row * g.ldc + col] = Cin ? acc[i][j][h] : g.alpha * acc[i][j][h];
        }
    }
  }
  if (PARTIALS) {
    __syncthreads();
    for (int rl = tid; rl < BM; rl += THREADS) {
      int64_t row = m0 + rl;
      if (row < g.M) {
        double s = 0.0, d = 0.0;
#pragma unroll
        for (int w = 0; w < WN; ++w) {
          s += red_sq[w][rl];
          d += red_dot[w][rl];
        }
        g.psq[row * g.ldp + blockIdx.x] = s;
        if (g.pdot) g.pdot[row * g.ldp + blockIdx.x] = d;
      }
    }
  }
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int MINB, bool VEC, bool PARTIALS>
__global__ void __launch_bounds__(WM * WN * 32, MINB) dgemm_kernel(GemmArgs g) {
  constexpr int THREADS = WM * WN * 32;
  constexpr int AS = BK + 4;  // == 4 mod 16 doubles: conflict-free fragment loads
  constexpr int BS = BN + 4;
  constexpr int STAGE = BM * AS + BK * BS;
  constexpr int TM = BM / WM / 8;  // 8-row tiles per warp
  constexpr int TN = BN / WN / 8;  // 8-col tiles per warp
  extern __shared__ double smem[];
  __shared__ double red_sq[PARTIALS ? WN : 1][PARTIALS ? BM : 1];
  __shared__ double red_dot[PARTIALS ? WN : 1][PARTIALS ? BM : 1];

  const int64_t n0 = (int64_t)blockIdx.x * BN;
  const int64_t m0 = (int64_t)blockIdx.y * BM;
  const int z = blockIdx.z;
  const double* A = g.A + z * g.bsA;
  const double* B = g.B + z * g.bsB;
  double* C = g.C + z * g.bsC;
  const double* Cin = g.Cin ? g.Cin + z * g.bsCin : nullptr;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const int gq = lane >> 2, t4 = lane & 3;

  int64_t kbeg = 0, kend = g.K;
  if (g.kmode == KB_UPPER) kend = min(g.K, n0 + BN);
  if (g.kmode == KB_LOWER) kbeg = (n0 / BK) * BK;
  const int ntiles = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;

  // interior fast path (16-byte copies): per-thread offsets fixed, per-tile
  // bases uniform, no bounds tests
  constexpr int A_IT = (BM * BK / 2) / THREADS, B_IT = (BK * BN / 2) / THREADS;
  constexpr int RA = THREADS / (BK / 2), RB = THREADS / (BN / 2);
  const bool interior = VEC && m0 + BM <= g.M && n0 + BN <= g.N;
  const int r0 = tid / (BK / 2), kc0 = (tid % (BK / 2)) * 2;
  const int kr0 = tid / (BN / 2), c0 = (tid % (BN / 2)) * 2;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t sa0 = sbase + (uint32_t)(r0 * AS + kc0) * 8u;
  const uint32_t sb0 = sbase + (uint32_t)(BM * AS + kr0 * BS + c0) * 8u;
  const double* ga0 = A + (m0 + r0) * g.sa_r + kc0 + kbeg;
  const double* gb0 = B + (kr0 + kbeg) * g.sb_r + n0 + c0;
  const int64_t stepA = (int64_t)RA * g.sa_r, stepB = (int64_t)RB * g.sb_r;

  auto issue = [&](int tile, int stage) {
    double* As = smem + stage * STAGE;
    double* Bs = As + BM * AS;
    const int64_t k0 = kbeg + (int64_t)tile * BK;
    if (VEC && A_IT * THREADS == BM * BK / 2 && B_IT * THREADS == BK * BN / 2 && THREADS % (BK / 2) == 0 &&
        THREADS % (BN / 2) == 0 && interior && k0 + BK <= kend) {
      const uint32_t so = (uint32_t)(stage * STAGE) * 8u;
      const double* ga = ga0 + (int64_t)tile * BK;
      const double* gb = gb0 + (int64_t)tile * BK * g.sb_r;
#pragma unroll
      for (int it = 0; it < A_IT; ++it)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa0 + so + (uint32_t)(it * RA * AS * 8)),
                     "l"(ga + it * stepA));
#pragma unroll
      for (int it = 0; it < B_IT; ++it)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sb0 + so + (uint32_t)(it * RB * BS * 8)),
                     "l"(gb + it * stepB));
      return;
    }
    if (VEC) {
#pragma unroll
      for (int it = 0; it < (BM * BK / 2) / THREADS; ++it) {
        int e = tid + it * THREADS;
        int r = e / (BK / 2), kc = (e % (BK / 2)) * 2;
        int64_t row = m0 + r, kk = k0 + kc;
        int bytes = 0;
        const double* src = A;
        if (row < g.M && kk < kend) {
          bytes = (kend - kk) >= 2 ? 16 : 8;
          src = A + row * g.sa_r + kk;
        }
        cp_async16(As + r * AS + kc, src, bytes);
      }
#pragma unroll
      for (int it = 0; it < (BK * BN / 2) / THREADS; ++it) {
        int e = tid + it * THREADS;
        int kr = e / (BN / 2), c = (e % (BN / 2)) * 2;
        int64_t kk = k0 + kr, col = n0 + c;
        int bytes = 0;
        const double* src = B;
        if (kk < kend && col < g.N) {
          bytes = (g.N - col) >= 2 ? 16 : 8;
          src = B + kk * g.sb_r + col;
        }
        cp_async16(Bs + kr * BS + c, src, bytes);
      }
    } else {
#pragma unroll
      for (int it = 0; it < (BM * BK) / THREADS; ++it) {
        int e = tid + it * THREADS;
        int r = e / BK, kc = e % BK;
        int64_t row = m0 + r, kk = k0 + kc;
        bool ok = row < g.M && kk < kend;
        cp_async8(As + r * AS + kc, ok ? A + row * g.sa_r + kk * g.sa_c : A, ok);
      }
#pragma unroll
      for (int it = 0; it < (BK * BN) / THREADS; ++it) {
        int e = tid + it * THREADS;
        int kr = e / BN, c = e % BN;
        int64_t kk = k0 + kr, col = n0 + c;
        bool ok = kk < kend && col < g.N;
        cp_async8(Bs + kr * BS + c, ok ? B + kk * g.sb_r + col * g.sb_c : B, ok);
      }
    }
  };

  double acc[TM][TN][2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ntiles) issue(s, s);
    cp_async_commit();
  }
  auto tile_step = [&](int tile) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    int nt = tile + STAGES - 1;
    if (nt < ntiles) issue(nt, nt % STAGES);
    cp_async_commit();
    const double* As = smem + (tile % STAGES) * STAGE + (wm * TM * 8) * AS;
    const double* Bs = smem + (tile % STAGES) * STAGE + BM * AS + wn * TN * 8;
#pragma unroll
    for (int kb = 0; kb < BK; kb += 4) {
      double af[TM], bf[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) af[i] = As[(i * 8 + gq) * AS + kb + t4];
#pragma unroll
      for (int j = 0; j < TN; ++j) bf[j] = Bs[(kb + t4) * BS + j * 8 + gq];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  };
  for (int tile = 0; tile < ntiles; ++tile) tile_step(tile);
  cp_async_wait<0>();

  gemm_epilogue<BM, BN, WM, WN, PARTIALS>(g, acc, C, Cin, m0, n0, tid, wm, wn, gq, t4, red_sq, red_dot);
}

// LDS.128 variant (16-byte copies only).  The k-slots of the DMMA are
// remapped so each thread's operands are contiguous in shared memory:
//   step q (0..3) of a 16-deep k-tile uses k = 4 t4 + q for lane (gq, t4),
//   so a thread's A values A[row][4 t4 .. 4 t4 + 3] are two LDS.128;
//   the 8-column DMMA tile j is the column set {c * TN + j}, so a thread's B
//   values B[k][gq TN .. gq TN + TN - 1] are TN / 2 LDS.128.
// Per warp and k-tile that is 2 TM + 2 TN loads for 4 TM TN DMMAs (the
// 8-byte-fragment kernel needs 4 TM + 4 TN).  A rows are padded to 18 doubles
// and B rows swizzled (16-byte chunk c of k-row r stored at c ^ ((r >> 2) & 3))
// so every quarter-warp LDS.128 phase hits 8 distinct 16-byte bank groups.
template <int BM, int BN, int WM, int WN, int STAGES, int MINB, bool PARTIALS, int BK = 16>
__global__ void __launch_bounds__(WM * WN * 32, MINB) dgemm_kernel3(GemmArgs g) {
  static_assert(BK % 16 == 0, "k-tile is a multiple of 16");
  constexpr int THREADS = WM * WN * 32;
  constexpr int AS = BK + 2;
  constexpr int BS = BN;
  constexpr int STAGE = BM * AS + BK * BS;
  constexpr int TM = BM / WM / 8;
  constexpr int TN = BN / WN / 8;
  constexpr int A_IT = (BM * BK / 2) / THREADS;
  constexpr int B_IT = (BK * BN / 2) / THREADS;
  static_assert(TN == 8 || TN == 4, "B swizzle defined for TN = 4 or 8");
  // 16-byte chunk swizzle of B rows, by the row's t4 = (k >> 2) & 3: the 8 lanes
  // of a quarter-warp (gq in {0, 1}, t4 in 0..3) then hit 8 distinct bank groups
  auto swz = [](int t) { return TN == 8 ? t : ((t & 1) | ((t >> 1) << 2)); };
  static_assert(A_IT >= 1 && B_IT >= 1 && A_IT <= 32 && B_IT <= 32, "copy split");
  extern __shared__ double smem[];
  __shared__ double red_sq[PARTIALS ? WN : 1][PARTIALS ? BM : 1];
  __shared__ double red_dot[PARTIALS ? WN : 1][PARTIALS ? BM : 1];

  const int64_t n0 = (int64_t)blockIdx.x * BN;
  const int64_t m0 = (int64_t)blockIdx.y * BM;
  const int z = blockIdx.z;
  const double* A = g.A + z * g.bsA;
  const double* B = g.B + z * g.bsB;
  double* C = g.C + z * g.bsC;
  const double* Cin = g.Cin ? g.Cin + z * g.bsCin : nullptr;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const int gq = lane >> 2, t4 = lane & 3;

  int64_t kbeg = 0, kend = g.K;
  if (g.kmode == KB_UPPER) kend = min(g.K, n0 + BN);
  if (g.kmode == KB_LOWER) kbeg = (n0 / BK) * BK;
  const int ntiles = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;

  uint32_t a_ok = 0, b_ok = 0, b_half = 0;
#pragma unroll
  for (int it = 0; it < A_IT; ++it) {
    const int r = (tid + it * THREADS) / (BK / 2);
    if (m0 + r < g.M) a_ok |= 1u << it;
  }
#pragma unroll
  for (int it = 0; it < B_IT; ++it) {
    const int c = ((tid + it * THREADS) % (BN / 2)) * 2;
    if (n0 + c < g.N) b_ok |= 1u << it;
    if (n0 + c + 1 == g.N) b_half |= 1u << it;
  }
  const double* Ab = A + m0 * g.sa_r;
  const double* Bb = B + n0;

  // interior fast path: per-thread offsets fixed, per-tile bases uniform
  static_assert(THREADS % (BK / 2) == 0 && THREADS % (BN / 2) == 0, "copy rows");
  constexpr int RA = THREADS / (BK / 2), RB = THREADS / (BN / 2);
  const bool interior = m0 + BM <= g.M && n0 + BN <= g.N;
  const int r0 = tid / (BK / 2), kc0 = (tid % (BK / 2)) * 2;
  const int kr0 = tid / (BN / 2), ch0 = tid % (BN / 2);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t sa0 = sbase + (uint32_t)(r0 * AS + kc0) * 8u;
  const uint32_t sb0 = sbase + (uint32_t)(BM * AS + kr0 * BS) * 8u;
  const double* ga0 = Ab + r0 * g.sa_r + kc0 + kbeg;
  const double* gb0 = Bb + (kr0 + kbeg) * g.sb_r + 2 * ch0;
  const int64_t stepA = (int64_t)RA * g.sa_r, stepB = (int64_t)RB * g.sb_r;

  auto issue = [&](int tile, int stage) {
    const int64_t k0 = kbeg + (int64_t)tile * BK;
    if (interior && k0 + BK <= kend) {
      const uint32_t so = (uint32_t)(stage * STAGE) * 8u;
      const double* ga = ga0 + (int64_t)tile * BK;
      const double* gb = gb0 + (int64_t)tile * BK * g.sb_r;
#pragma unroll
      for (int it = 0; it < A_IT; ++it)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa0 + so + (uint32_t)(it * RA * AS * 8)),
                     "l"(ga + it * stepA));
#pragma unroll
      for (int it = 0; it < B_IT; ++it) {
        const int kr = kr0 + it * RB;
        const uint32_t d = sb0 + so + (uint32_t)(it * RB * BS * 8) + (uint32_t)((ch0 ^ swz((kr >> 2) & 3)) * 16);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gb + it * stepB));
      }
      return;
    }
    double* As = smem + stage * STAGE;
    double* Bs = As + BM * AS;
    const bool fullk = k0 + BK <= kend;
    const double* At = Ab + k0;
    const double* Bt = Bb + k0 * g.sb_r;
#pragma unroll
    for (int it = 0; it < A_IT; ++it) {
      const int e = tid + it * THREADS;
      const int r = e / (BK / 2), kc = (e % (BK / 2)) * 2;
      int bytes = (a_ok >> it) & 1 ? 16 : 0;
      if (!fullk) {
        const int64_t rem = kend - (k0 + kc);
        bytes = rem >= 2 ? bytes : (rem == 1 ? bytes / 2 : 0);
      }
      cp_async16(As + r * AS + kc, bytes ? At + r * g.sa_r + kc : A, bytes);
    }
#pragma unroll
    for (int it = 0; it < B_IT; ++it) {
      const int e = tid + it * THREADS;
      const int kr = e / (BN / 2), ch = e % (BN / 2);
      int bytes = (b_ok >> it) & 1 ? ((b_half >> it) & 1 ? 8 : 16) : 0;
      if (!fullk && k0 + kr >= kend) bytes = 0;
      cp_async16(Bs + kr * BS + 2 * (ch ^ swz((kr >> 2) & 3)), bytes ? Bt + kr * g.sb_r + 2 * ch : B, bytes);
    }
  };

  double acc[TM][TN][2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ntiles) issue(s, s);
    cp_async_commit();
  }
  int stage = 0;
  for (int tile = 0; tile < ntiles; ++tile) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nt = tile + STAGES - 1;
      const int ns = stage == 0 ? STAGES - 1 : stage - 1;  // == nt % STAGES
      if (nt < ntiles) issue(nt, ns);
      cp_async_commit();
    }
    const double* As = smem + stage * STAGE + (wm * TM * 8 + gq) * AS + 4 * t4;
    const double* Bs = smem + stage * STAGE + BM * AS + wn * TN * 8;
#pragma unroll
    for (int h16 = 0; h16 < BK / 16; ++h16) {
      double a[TM][4];
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const double2 x = *reinterpret_cast<const double2*>(As + i * 8 * AS + 16 * h16);
        const double2 y = *reinterpret_cast<const double2*>(As + i * 8 * AS + 16 * h16 + 2);
        a[i][0] = x.x; a[i][1] = x.y; a[i][2] = y.x; a[i][3] = y.y;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double* Br = Bs + (16 * h16 + 4 * t4 + q) * BS;
        double b[TN];
#pragma unroll
        for (int jj = 0; jj < TN / 2; ++jj) {
          const double2 v = *reinterpret_cast<const double2*>(Br + 2 * ((gq * (TN / 2) + jj) ^ swz(t4)));
          b[2 * jj] = v.x;
          b[2 * jj + 1] = v.y;
        }
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i][q], b[j]);
      }
    }
    stage = stage + 1 == STAGES ? 0 : stage + 1;
  }
  cp_async_wait<0>();
  gemm_epilogue<BM, BN, WM, WN, PARTIALS, true>(g, acc, C, Cin, m0, n0, tid, wm, wn, gq, t4, red_sq, red_dot);
}

template <int BM, int BN, int WM, int WN, int STAGES, int MINB, bool P, int BK = 16>
int launch_three(const GemmArgs& g, int batch, cudaStream_t st) {
  constexpr size_t smem = (size_t)STAGES * (BM * (BK + 2) + BK * BN) * sizeof(double);
  auto kern = dgemm_kernel3<BM, BN, WM, WN, STAGES, MINB, P, BK>;
  static bool configured = false;
  if (!configured) {
    HIKF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  dim3 grid((unsigned)ceil_div(g.N, BN), (unsigned)ceil_div(g.M, BM), (unsigned)batch);
  kern<<<grid, WM * WN * 32, smem, st>>>(g);
  HIKF_CHECK_LAUNCH();
  return HIKF_OK;
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int MINB, bool VEC, bool P>
int launch_one(const GemmArgs& g, int batch, cudaStream_t st) {
  constexpr size_t smem = (size_t)STAGES * (BM * (BK + 4) + BK * (BN + 4)) * sizeof(double);
  auto kern = dgemm_kernel<BM, BN, BK, WM, WN, STAGES, MINB, VEC, P>;
  static bool configured = false;
  if (!configured) {
    HIKF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  dim3 grid((unsigned)ceil_div(g.N, BN), (unsigned)ceil_div(g.M, BM), (unsigned)batch);
  kern<<<grid, WM * WN * 32, smem, st>>>(g);
  HIKF_CHECK_LAUNCH();
  return HIKF_OK;
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int MINB>
int launch_variant(const GemmArgs& g, int batch, bool vec, bool part, cudaStream_t st) {
  if (vec)
    return part ? launch_one<BM, BN, BK, WM, WN, STAGES, MINB, true, true>(g, batch, st)
                : launch_one<BM, BN, BK, WM, WN, STAGES, MINB, true, false>(g, batch, st);
  return part ? launch_one<BM, BN, BK, WM, WN, STAGES, MINB, false, true>(g, batch, st)
              : launch_one<BM, BN, BK, WM, WN, STAGES, MINB, false, false>(g, batch, st);
}

template <int BM, int BN, int WM, int WN, int STAGES, int MINB, int BK = 16>
int launch_variant3(const GemmArgs& g, int batch, bool vec, bool part, cudaStream_t st) {
  if (!vec) return launch_variant<BM, BN, 16, WM, WN, STAGES, MINB>(g, batch, vec, part, st);
  return part ? launch_three<BM, BN, WM, WN, STAGES, MINB, true, BK>(g, batch, st)
              : launch_three<BM, BN, WM, WN, STAGES, MINB, false, BK>(g, batch, st);
}

// ---------------------------------------------------------------------------
// Variant 30: CUTLASS multistage DMMA mainloop (cp.async ring, conflict-free
// 64-bit smem layouts, serpentine warp MMA order) + the fused epilogue above.
// profiles/r01_cutlass_probe.log: the plain CUTLASS 64x128x16 / 32x64 / 3-stage
// GEMM runs the cfg4 K-GEMM shape in 61.3 ms (cuBLAS 61.6 ms, our v7 66.5 ms).
template <int BM, int BN, int WTM, int WTN, int STAGES>
struct CutlassMain {
  using RM = cutlass::layout::RowMajor;
  using DefaultMma = cutlass::gemm::threadblock::DefaultMma<
      double, RM, 1, double, RM, 1, double, RM, cutlass::arch::OpClassTensorOp, cutlass::arch::Sm80,
      cutlass::gemm::GemmShape<BM, BN, 16>, cutlass::gemm::GemmShape<WTM, WTN, 16>, cutlass::gemm::GemmShape<8, 8, 4>,
      STAGES, cutlass::arch::OpMultiplyAdd>;
  using Mma = typename DefaultMma::ThreadblockMma;
  static constexpr int WM = BM / WTM, WN = BN / WTN, THREADS = WM * WN * 32;
};

template <int BM, int BN, int WTM, int WTN, int STAGES, bool PARTIALS>
__global__ void __launch_bounds__(CutlassMain<BM, BN, WTM, WTN, STAGES>::THREADS, 2)
    dgemm_cutlass_kernel(GemmArgs g, typename CutlassMain<BM, BN, WTM, WTN, STAGES>::Mma::IteratorA::Params pA,
                         typename CutlassMain<BM, BN, WTM, WTN, STAGES>::Mma::IteratorB::Params pB) {
  using CM = CutlassMain<BM, BN, WTM, WTN, STAGES>;
  using Mma = typename CM::Mma;
  constexpr int WM = CM::WM, WN = CM::WN;
  constexpr int TM = WTM / 8, TN = WTN / 8;
  extern __shared__ __align__(16) char smem_raw[];
  auto& ss = *reinterpret_cast<typename Mma::SharedStorage*>(smem_raw);
  __shared__ double red_sq[PARTIALS ? WN : 1][PARTIALS ? BM : 1];
  __shared__ double red_dot[PARTIALS ? WN : 1][PARTIALS ? BM : 1];

  const int64_t n0 = (int64_t)blockIdx.x * BN;
  const int64_t m0 = (int64_t)blockIdx.y * BM;
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  // triangular B: only the k-range that can hold nonzeros (as dgemm_kernel)
  int64_t kbeg = 0, kend = g.K;
  if (g.kmode == KB_UPPER) kend = min(g.K, n0 + BN);
  if (g.kmode == KB_LOWER) kbeg = (n0 / 16) * 16;
  typename Mma::IteratorA itA(pA, const_cast<double*>(g.A), {(int)g.M, (int)kend}, tid, {(int)m0, (int)kbeg});
  typename Mma::IteratorB itB(pB, const_cast<double*>(g.B), {(int)kend, (int)g.N}, tid, {(int)kbeg, (int)n0});
  Mma mma(ss, tid, warp, lane);
  typename Mma::FragmentC accum;
  accum.clear();
  if (kend > kbeg) mma((int)((kend - kbeg + 15) / 16), accum, itA, itB, accum);

  // CUTLASS warp tile (mma_tensor_op.h, accumulators column-major over the
  // 8x8 instruction tiles): tile (i, j) -> accum[2 (i + j TM) + h] holds
  // C[wm WTM + 8 i + gq][wn WTN + 8 j + 2 t4 + h]; warps are m-fastest.
  double acc[TM][TN][2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) acc[i][j][h] = accum[2 * (i + j * TM) + h];
  const int wm = warp % WM, wn = warp / WM;
  gemm_epilogue<BM, BN, WM, WN, PARTIALS>(g, acc, g.C, g.Cin, m0, n0, tid, wm, wn, lane >> 2, lane & 3, red_sq,
                                          red_dot);
  if (g.gv_y && blockIdx.x == gridDim.x - 1) {
    // fused GEMV rows of this row block: one warp per row, 16-byte loads, lane-strided sums
    const bool v2 = (g.K % 2 == 0) && (g.sa_r % 2 == 0) && ((((uintptr_t)g.A) | ((uintptr_t)g.gv_x)) & 15) == 0;
    for (int r = warp; r < BM; r += CM::THREADS / 32) {
      const int64_t row = m0 + r;
      if (row >= g.M) break;
      const double* a = g.A + row * g.sa_r;
      double s = 0.0;
      if (v2) {
        const double2* a2 = reinterpret_cast<const double2*>(a);
        const double2* x2 = reinterpret_cast<const double2*>(g.gv_x);
        for (int64_t c = lane; c < g.K / 2; c += 32) {
          const double2 av = a2[c], xv = __ldg(x2 + c);
          s = fma(av.x, xv.x, s);
          s = fma(av.y, xv.y, s);
        }
      } else {
        for (int64_t c = lane; c < g.K; c += 32) s = fma(a[c], g.gv_x[c], s);
      }
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) g.gv_y[row] = s;
    }
  }
}

template <int BM, int BN, int WTM, int WTN, int STAGES, bool P>
int launch_cutlass(const GemmArgs& g, cudaStream_t st) {
  using CM = CutlassMain<BM, BN, WTM, WTN, STAGES>;
  using Mma = typename CM::Mma;
  constexpr size_t smem = sizeof(typename Mma::SharedStorage);
  auto kern = dgemm_cutlass_kernel<BM, BN, WTM, WTN, STAGES, P>;
  static bool configured = false;
  if (!configured) {
    HIKF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  typename Mma::IteratorA::Params pA(cutlass::layout::RowMajor((int)g.sa_r));
  typename Mma::IteratorB::Params pB(cutlass::layout::RowMajor((int)g.sb_r));
  dim3 grid((unsigned)ceil_div(g.N, BN), (unsigned)ceil_div(g.M, BM), 1u);
  kern<<<grid, CM::THREADS, smem, st>>>(g, pA, pB);
  HIKF_CHECK_LAUNCH();
  return HIKF_OK;
}

int g_variant = -1;

}  // namespace

int dgemm_variant() {
  if (g_variant < 0) {
    const char* e = getenv("HIKF_DGEMM_VARIANT");
    g_variant = e ? atoi(e) : 30;  // default: CUTLASS mainloop 64x128x16, 4 warps of 32x64, 3 stages (profiles/r01_gemm_sweep_cutlass.log)
  }
  return g_variant;
}

void set_dgemm_variant(int v) { g_variant = v; }

int update_variant_c(int64_t n) {
  if (getenv("HIKF_DGEMM_VARIANT")) return dgemm_variant();
  // 128-column tiles (variant 30) unless 64-column tiles (variant 32) pad n less
  // (e.g. n = 64, cfg1: one full 64-wide tile instead of half a 128-wide one)
  const int64_t w128 = ceil_div(n, 128) * 128 - n, w64 = ceil_div(n, 64) * 64 - n;
  return w64 < w128 ? 32 : 30;
}

int dgemm(const GemmArgs& g, int batch, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0 || batch <= 0) return HIKF_OK;
  int variant = g.variant >= 0 ? g.variant : dgemm_variant();
  auto al16 = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  bool vec = g.sa_c == 1 && g.sb_c == 1 && (g.sa_r % 2 == 0) && (g.sb_r % 2 == 0) && al16(g.A) && al16(g.B) &&
             (batch == 1 || (g.bsA % 2 == 0 && g.bsB % 2 == 0));
  bool part = g.psq != nullptr;
  // CUTLASS-mainloop variants: row-major operands (any kmode), one batch
  const bool cutlass_ok = g.sa_c == 1 && g.sb_c == 1 && batch == 1 && g.M < (1ll << 31) &&
                          g.K < (1ll << 31) && g.N < (1ll << 31);
  if (variant == 30 && cutlass_ok)  // 64x128x16, 4 warps of 32x64, 3 stages
    return part ? launch_cutlass<64, 128, 32, 64, 3, true>(g, st) : launch_cutlass<64, 128, 32, 64, 3, false>(g, st);
  if (variant == 31 && cutlass_ok)  // 64x128x16, 4 warps of 32x64, 4 stages
    return part ? launch_cutlass<64, 128, 32, 64, 4, true>(g, st) : launch_cutlass<64, 128, 32, 64, 4, false>(g, st);
  if (variant == 32 && cutlass_ok)  // 128x64x16, 4 warps of 64x32, 3 stages (64-column tiles: finer triangles)
    return part ? launch_cutlass<128, 64, 64, 32, 3, true>(g, st) : launch_cutlass<128, 64, 64, 32, 3, false>(g, st);
  if (g.gv_y) {
    set_error("dgemm: the fused GEMV (gv_x / gv_y) needs a CUTLASS variant (30-32) and row-major operands");
    return HIKF_BAD_ARGUMENT;
  }
  if (variant >= 30) variant = 7;
  switch (variant) {
    case 1:  // 128x128x32, 8 warps of 64x32, 3 stages
      return launch_variant<128, 128, 32, 2, 4, 3, 1>(g, batch, vec, part, st);
    case 2:  // 128x128x16, 16 warps of 32x32, 5 stages
      return launch_variant<128, 128, 16, 4, 4, 5, 1>(g, batch, vec, part, st);
    case 3:  // 128x128x32, 16 warps of 32x32, 3 stages
      return launch_variant<128, 128, 32, 4, 4, 3, 1>(g, batch, vec, part, st);
    case 4:  // 64x128x16, 8 warps of 32x32, 4 stages, 2 CTAs / SM
      return launch_variant<64, 128, 16, 2, 4, 4, 2>(g, batch, vec, part, st);
    case 5:  // 128x64x16, 8 warps of 32x32, 4 stages, 2 CTAs / SM
      return launch_variant<128, 64, 16, 4, 2, 4, 2>(g, batch, vec, part, st);
    case 6:  // 64x128x32, 8 warps of 32x32, 2 stages, 2 CTAs / SM
      return launch_variant<64, 128, 32, 2, 4, 2, 2>(g, batch, vec, part, st);
    case 7:  // 64x128x16, 8 warps of 32x32, 3 stages, 2 CTAs / SM
      return launch_variant<64, 128, 16, 2, 4, 3, 2>(g, batch, vec, part, st);
    case 8:  // 64x64x16, 4 warps of 32x32, 4 stages, 3 CTAs / SM (smem-bound)
      return launch_variant<64, 64, 16, 2, 2, 4, 4>(g, batch, vec, part, st);
    case 9:  // 64x64x32, 4 warps of 32x32, 2 stages, 3 CTAs / SM
      return launch_variant<64, 64, 32, 2, 2, 2, 3>(g, batch, vec, part, st);
    case 10:  // 64x64x16, 4 warps of 32x32, 2 stages, 5 CTAs / SM
      return launch_variant<64, 64, 16, 2, 2, 2, 4>(g, batch, vec, part, st);
    case 11:  // 64x128x16, 4 warps of 32x64, 3 stages, 2 CTAs / SM
      return launch_variant<64, 128, 16, 2, 2, 3, 2>(g, batch, vec, part, st);
    case 12:  // 64x128x16, 4 warps of 32x64, 4 stages, 2 CTAs / SM
      return launch_variant<64, 128, 16, 2, 2, 4, 2>(g, batch, vec, part, st);
    case 13:  // 128x64x16, 4 warps of 64x32, 3 stages, 2 CTAs / SM
      return launch_variant<128, 64, 16, 2, 2, 3, 2>(g, batch, vec, part, st);
    case 15:  // 64x128x32, 4 warps of 32x64, 2 stages, 2 CTAs / SM
      return launch_variant<64, 128, 32, 2, 2, 2, 2>(g, batch, vec, part, st);
    case 21:  // LDS.128 kernel: 64x128x16, 4 warps of 32x64, 3 stages, 2 CTAs / SM
      return launch_variant3<64, 128, 2, 2, 3, 2>(g, batch, vec, part, st);
    case 22:  // LDS.128 kernel: 128x64x16, 4 warps of 32x64 stacked along rows, 3 stages
      return launch_variant3<128, 64, 4, 1, 3, 2>(g, batch, vec, part, st);
    case 28:  // LDS.128 kernel: 128x64x16, 4 warps of 64x32 (cuBLAS's warp shape), 3 stages, 2 CTAs / SM
      return launch_variant3<128, 64, 2, 2, 3, 2>(g, batch, vec, part, st);
    case 29:  // LDS.128 kernel: 128x64x16, 4 warps of 64x32, 4 stages, 2 CTAs / SM
      return launch_variant3<128, 64, 2, 2, 4, 2>(g, batch, vec, part, st);
    case 27:  // LDS.128 kernel: 64x128x16, 4 warps of 32x64, 2 stages, 2 CTAs / SM
      return launch_variant3<64, 128, 2, 2, 2, 2>(g, batch, vec, part, st);
    default:  // 128x128x16, 8 warps of 64x32, 5 stages
      return launch_variant<128, 128, 16, 2, 4, 5, 1>(g, batch, vec, part, st);
  }
}

}  // namespace hikf

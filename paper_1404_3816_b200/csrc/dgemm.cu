// FP64 DMMA GEMM (see dgemm.cuh), hand-written for sm_100a (no library
// mainloop).  Two kernels share one fused epilogue:
//   * dgemm_rm_kernel -- row-major operands (every large GEMM of the update and
//     of the factored path): register-double-buffered fragments, a cp.async
//     ring whose copies are spread over the k-groups, one barrier per k-tile
//     placed before the last k-group so the next tile's first fragments load
//     under the last DMMAs, serpentine DMMA order, 1D tile raster with the
//     column tiles of a row block adjacent (the A row panel is reused from L2);
//   * dgemm_kernel -- any strides (the transposed-B GEMMs of the recursive
//     Cholesky on n x n blocks).
#include <algorithm>
#include <cstdlib>

#include "dgemm.cuh"

namespace hikf {

namespace {

// Shared epilogue: alpha/beta, fused row partials (written to column slot
// `ctile` of psq / pdot), the chained-predict second output, stores.
// Accumulator acc[i][j][h] holds C[row = i*8 + gq][col = j*8 + 2 t4 + h] of the
// warp tile (8 x 8 DMMA tiles).
template <int BM, int BN, int WM, int WN, bool PARTIALS>
__device__ __forceinline__ void gemm_epilogue(const GemmArgs& g, double (&acc)[BM / WM / 8][BN / WN / 8][2], double* C,
                                              const double* Cin, int64_t m0, int64_t n0, int tid, int wm, int wn,
                                              int gq, int t4, double (*red_sq)[PARTIALS ? BM : 1],
                                              double (*red_dot)[PARTIALS ? BM : 1], int64_t ctile) {
  constexpr int THREADS = WM * WN * 32;
  constexpr int TM = BM / WM / 8;
  constexpr int TN = BN / WN / 8;
  const int64_t cw = n0 + wn * TN * 8;
  auto colh = [&](int j, int h) -> int64_t { return cw + j * 8 + 2 * t4 + h; };
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
    if (g.chain_out) {
      // also emit chain_out = C + chain_add (the next step's predict, fused);
      // columns 2 t4 and 2 t4 + 1 are adjacent: 16-byte accesses when aligned
      const bool v16 = row < g.M && cw + BN / WN <= g.N && (g.ldc | g.ldch) % 2 == 0 &&
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
    } else if (row < g.M && cw + BN / WN <= g.N && g.ldc % 2 == 0 && ((uintptr_t)C & 15) == 0) {
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
        g.psq[row * g.ldp + ctile] = s;
        if (g.pdot) g.pdot[row * g.ldp + ctile] = d;
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

  gemm_epilogue<BM, BN, WM, WN, PARTIALS>(g, acc, C, Cin, m0, n0, tid, wm, wn, gq, t4, red_sq, red_dot, blockIdx.x);
}

// ---------------------------------------------------------------------------
// Row-major mainloop.  CTA tile BM x BN x 16, warps of WTM x WTN (TM x TN
// DMMA 8x8 tiles, 2 TM TN accumulator doubles per thread), STAGES-deep cp.async
// ring.  Shared-memory rows are padded to 4 (mod 16) doubles: the 32 fragment
// addresses of a warp (A[8 rows][4 k] or B[4 k][8 cols]) then cover every
// 8-byte bank pair exactly twice, the minimum of two wavefronts per LDS.64.
//
// Per k-tile and warp: 4 k-groups of TM + TN fragment loads and TM TN DMMAs.
// The fragments of k-group q+1 are loaded into the other register buffer
// before the DMMAs of q are issued; the 16-byte copies of tile t+STAGES-1 are
// spread over the first three k-groups; the one barrier per tile sits before
// the last k-group, so the first fragments of the next tile load while the
// last DMMAs of this one run.
template <int BM, int BN, int WTM, int WTN>
struct RmCfg {
  static constexpr int BK = 16, WM = BM / WTM, WN = BN / WTN, THREADS = WM * WN * 32;
  static constexpr int TM = WTM / 8, TN = WTN / 8;
  static constexpr int AS = BK + 4, BS = BN + 4;
  static constexpr int STAGE = BM * AS + BK * BS;
  static constexpr int A_CH = BM * BK / 2 / THREADS, B_CH = BK * BN / 2 / THREADS;
  static constexpr int A_RPI = THREADS / (BK / 2);  // A rows covered per copy iteration
  static constexpr int B_CPR = BN / 2;              // 16-byte chunks per B row
  static constexpr int B_RPI = THREADS / B_CPR;     // B rows covered per copy iteration
  static_assert(A_CH * THREADS * 2 == BM * BK && B_CH * THREADS * 2 == BK * BN, "copy split");
  static_assert(THREADS % B_CPR == 0, "B copy rows");
  static_assert(AS % 16 == 4 && BS % 16 == 4, "conflict-free fragment padding");
};

__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp16z(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(bytes));
}

template <int BM, int BN, int WTM, int WTN, int STAGES, bool PARTIALS>
__global__ void __launch_bounds__(RmCfg<BM, BN, WTM, WTN>::THREADS, 2) dgemm_rm_kernel(GemmArgs g, int64_t ntn) {
  using Cf = RmCfg<BM, BN, WTM, WTN>;
  constexpr int BK = Cf::BK, TM = Cf::TM, TN = Cf::TN, WM = Cf::WM, WN = Cf::WN;
  constexpr int AS = Cf::AS, BS = Cf::BS, STAGE = Cf::STAGE;
  constexpr int A_CH = Cf::A_CH, NCH = Cf::A_CH + Cf::B_CH;
  extern __shared__ __align__(16) double smem[];
  __shared__ double red_sq[PARTIALS ? WN : 1][PARTIALS ? BM : 1];
  __shared__ double red_dot[PARTIALS ? WN : 1][PARTIALS ? BM : 1];

  // 1D raster: the ntn column tiles of a row block are consecutive CTAs, so the
  // A row panel they all stream is read from HBM once and from L2 after that
  const int64_t ctile = (int64_t)blockIdx.x % ntn;
  const int64_t n0 = ctile * BN;
  const int64_t m0 = ((int64_t)blockIdx.x / ntn) * BM;
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int wm = warp % WM, wn = warp / WM, gq = lane >> 2, t4 = lane & 3;

  // triangular B: only the k-range that can hold nonzeros
  int64_t kbeg = 0, kend = g.K;
  if (g.kmode == KB_UPPER) kend = min(g.K, n0 + BN);
  if (g.kmode == KB_LOWER) kbeg = (n0 / BK) * BK;
  const int ntiles = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;

  const int ar = tid / (BK / 2), ak = (tid % (BK / 2)) * 2;
  const int br = tid / Cf::B_CPR, bc = (tid % Cf::B_CPR) * 2;
  const double* gA = g.A + (m0 + ar) * g.sa_r + kbeg + ak;
  const double* gB = g.B + (kbeg + br) * g.sb_r + n0 + bc;
  const int64_t stepA = (int64_t)Cf::A_RPI * g.sa_r, stepB = (int64_t)Cf::B_RPI * g.sb_r;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t sA = sbase + (uint32_t)(ar * AS + ak) * 8u;
  const uint32_t sB = sbase + (uint32_t)(BM * AS + br * BS + bc) * 8u;
  // per-thread copy bounds, fixed for the CTA: A row validity (bit q) and the
  // B column bytes (16, 8 at an odd last column, 0 past N)
  uint32_t arow_ok = 0;
#pragma unroll
  for (int q = 0; q < A_CH; ++q) arow_ok |= (m0 + ar + q * Cf::A_RPI < g.M ? 1u : 0u) << q;
  const int bcol_bytes = n0 + bc < g.N ? (g.N - (n0 + bc) >= 2 ? 16 : 8) : 0;
  const int64_t kspan = kend - kbeg;  // k offsets below are relative to kbeg

  // 16-byte copy q (0 .. NCH-1) of k-tile `tile` into ring slot `slot`.  No
  // branches: out-of-range chunks (rows >= M, columns >= N, k >= kend, tiles
  // past the last) copy 0 source bytes (zero fill), so the copies interleave
  // freely with the DMMAs of the k-group they are issued in.
  auto copy_chunk = [&](int q, int tile, int slot) {
    const int64_t k0 = (int64_t)tile * BK;
    const uint32_t so = (uint32_t)(slot * STAGE) * 8u;
    if (q < A_CH) {
      const int64_t kr = kspan - (k0 + ak);  // valid k columns left at this chunk
      const int bytes = ((arow_ok >> q) & 1u) ? (kr >= 2 ? 16 : (kr == 1 ? 8 : 0)) : 0;
      const double* src = gA + q * stepA + k0;
      cp16z(sA + so + (uint32_t)(q * Cf::A_RPI * AS) * 8u, bytes ? src : g.A, bytes);
    } else {
      const int it = q - A_CH;
      const int64_t kk = k0 + it * Cf::B_RPI;  // gB already points at row br
      const int bytes = kk + br < kspan ? bcol_bytes : 0;
      const double* src = gB + kk * g.sb_r;
      cp16z(sB + so + (uint32_t)(it * Cf::B_RPI * BS) * 8u, bytes ? src : g.B, bytes);
    }
  };

  double acc[TM][TN][2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
#pragma unroll
    for (int q = 0; q < NCH; ++q) copy_chunk(q, s, s);
    cp_async_commit();
  }
  cp_async_wait<STAGES - 2>();
  __syncthreads();

  double af[2][TM], bf[2][TN];
  const double* fa = smem + (wm * WTM + gq) * AS + t4;
  const double* fb = smem + BM * AS + t4 * BS + wn * WTN + gq;
  auto load_frags = [&](int buf, int slot, int kg) {
    const double* a = fa + slot * STAGE + kg * 4;
    const double* b = fb + slot * STAGE + kg * 4 * BS;
#pragma unroll
    for (int i = 0; i < TM; ++i) af[buf][i] = a[i * 8 * AS];
#pragma unroll
    for (int j = 0; j < TN; ++j) bf[buf][j] = b[j * 8];
  };
  load_frags(0, 0, 0);
  int rs = 0, wsl = STAGES - 1;
  for (int tile = 0; tile < ntiles; ++tile) {
#pragma unroll
    for (int kg = 0; kg < 4; ++kg) {
      if (kg == 3) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        rs = rs + 1 == STAGES ? 0 : rs + 1;
      }
      load_frags((kg + 1) & 1, rs, (kg + 1) & 3);
      if (kg < 3) {
#pragma unroll
        for (int q = kg * NCH / 3; q < (kg + 1) * NCH / 3; ++q) copy_chunk(q, tile + STAGES - 1, wsl);
        if (kg == 2) {
          cp_async_commit();
          wsl = wsl + 1 == STAGES ? 0 : wsl + 1;
        }
      }
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int ii = 0; ii < TM; ++ii) {
          const int i = (j & 1) ? TM - 1 - ii : ii;  // serpentine: consecutive DMMAs share an operand
          dmma884(acc[i][j][0], acc[i][j][1], af[kg & 1][i], bf[kg & 1][j]);
        }
    }
  }
  cp_async_wait<0>();

  gemm_epilogue<BM, BN, WM, WN, PARTIALS>(g, acc, g.C, g.Cin, m0, n0, tid, wm, wn, gq, t4, red_sq, red_dot, ctile);
  if (g.gv_y && ctile == ntn - 1) {
    // fused GEMV rows of this row block: one warp per row, 16-byte loads, lane-strided sums
    const bool v2 = (g.K % 2 == 0) && (g.sa_r % 2 == 0) && ((((uintptr_t)g.A) | ((uintptr_t)g.gv_x)) & 15) == 0;
    for (int r = warp; r < BM; r += Cf::THREADS / 32) {
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
int launch_rm(const GemmArgs& g, cudaStream_t st) {
  using Cf = RmCfg<BM, BN, WTM, WTN>;
  constexpr size_t smem = (size_t)STAGES * Cf::STAGE * sizeof(double);
  auto kern = dgemm_rm_kernel<BM, BN, WTM, WTN, STAGES, P>;
  static bool configured = false;
  if (!configured) {
    HIKF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  const int64_t ntn = ceil_div(g.N, BN), ntm = (g.M + BM - 1) / BM;
  if (ntm * ntn > 0x7fffffffll) {
    set_error("dgemm: %lld x %lld tiles exceed the grid limit", (long long)ntm, (long long)ntn);
    return HIKF_BAD_ARGUMENT;
  }
  kern<<<(unsigned)(ntm * ntn), Cf::THREADS, smem, st>>>(g, ntn);
  HIKF_CHECK_LAUNCH();
  return HIKF_OK;
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int MINB, bool VEC, bool P>
int launch_gen(const GemmArgs& g, int batch, cudaStream_t st) {
  constexpr size_t smem = (size_t)STAGES * (BM * (BK + 4) + BK * (BN + 4)) * sizeof(double);
  auto kern = dgemm_kernel<BM, BN, BK, WM, WN, STAGES, MINB, VEC, P>;
  static bool configured = false;
  if (!configured) {
    HIKF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  if ((g.M + BM - 1) / BM > 65535 || batch > 65535) {
    set_error("dgemm: strided operands with M = %lld exceed the generic kernel's grid", (long long)g.M);
    return HIKF_BAD_ARGUMENT;
  }
  dim3 grid((unsigned)ceil_div(g.N, BN), (unsigned)ceil_div(g.M, BM), (unsigned)batch);
  kern<<<grid, WM * WN * 32, smem, st>>>(g);
  HIKF_CHECK_LAUNCH();
  return HIKF_OK;
}

// y[i] = sum_k A[i][k] x[k] (row-major A, any stride): one warp per row, k in order per lane
__global__ void gemv_rows_kernel(int64_t M, int64_t K, const double* __restrict__ A, int64_t lda,
                                 const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  for (int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < M;
       row += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const double* a = A + row * lda;
    double s = 0.0;
    for (int64_t c = lane; c < K; c += 32) s = fma(a[c], x[c], s);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) y[row] = s;
  }
}

int g_variant = -1;

}  // namespace

int dgemm_variant() {
  if (g_variant < 0) {
    const char* e = getenv("HIKF_DGEMM_VARIANT");
    g_variant = e ? atoi(e) : 30;
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
  const int variant = g.variant >= 0 ? g.variant : dgemm_variant();
  auto al16 = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  const bool part = g.psq != nullptr;
  // row-major mainloop: unit column strides, 16-byte aligned rows, one batch
  const bool rm = g.sa_c == 1 && g.sb_c == 1 && batch == 1 && g.sa_r % 2 == 0 && g.sb_r % 2 == 0 && al16(g.A) &&
                  al16(g.B);
  if (rm && variant != 7) {
    switch (variant) {
      case 32:  // 128 x 64, warps 64 x 32, 3 stages (64-column tiles: finer triangles, n = 64)
        return part ? launch_rm<128, 64, 64, 32, 3, true>(g, st) : launch_rm<128, 64, 64, 32, 3, false>(g, st);
      default:  // 30: 64 x 128, warps 32 x 64, 3 stages
        return part ? launch_rm<64, 128, 32, 64, 3, true>(g, st) : launch_rm<64, 128, 32, 64, 3, false>(g, st);
    }
  }
  if (g.gv_y) {
    // unaligned or odd-stride rows (e.g. an odd ray count): the GEMM on the generic kernel,
    // then the GEMV over A as its own pass
    if (g.sa_c != 1 || batch != 1) {
      set_error("dgemm: the GEMV over A (gv_x / gv_y) needs row-major A and one batch");
      return HIKF_BAD_ARGUMENT;
    }
    GemmArgs h = g;
    h.gv_x = nullptr;
    h.gv_y = nullptr;
    HIKF_TRY(dgemm(h, 1, st));
    const int64_t blocks = std::min<int64_t>((g.M + 7) / 8, (int64_t)num_sms() * 16);
    gemv_rows_kernel<<<(unsigned)blocks, 256, 0, st>>>(g.M, g.K, g.A, g.sa_r, g.gv_x, g.gv_y);
    HIKF_CHECK_LAUNCH();
    return HIKF_OK;
  }
  const bool vec = g.sa_c == 1 && g.sb_c == 1 && (g.sa_r % 2 == 0) && (g.sb_r % 2 == 0) && al16(g.A) && al16(g.B) &&
                   (batch == 1 || (g.bsA % 2 == 0 && g.bsB % 2 == 0));
  // generic strides: 64 x 128 x 16, 8 warps of 32 x 32, 3 stages.  The row partials
  // land in column-tile slots, so a caller sized for a 64-column variant (its
  // dgemm_col_tiles) gets 64-column tiles here too (64 x 64, 4 warps of 32 x 32)
  if (part && variant == 32)
    return vec ? launch_gen<64, 64, 16, 2, 2, 3, 2, true, true>(g, batch, st)
               : launch_gen<64, 64, 16, 2, 2, 3, 2, false, true>(g, batch, st);
  if (vec)
    return part ? launch_gen<64, 128, 16, 2, 4, 3, 2, true, true>(g, batch, st)
                : launch_gen<64, 128, 16, 2, 4, 3, 2, true, false>(g, batch, st);
  return part ? launch_gen<64, 128, 16, 2, 4, 3, 2, false, true>(g, batch, st)
              : launch_gen<64, 128, 16, 2, 4, 3, 2, false, false>(g, batch, st);
}

}  // namespace hikf

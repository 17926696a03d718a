// FP64 DMMA GEMM (see dgemm.cuh).  One templated kernel; the tile shape is
// a compile-time variant (dgemm_variant() picks it; HIKF_DGEMM_VARIANT
// overrides for tuning sweeps).
#include <algorithm>
#include <cstdlib>

#include "dgemm.cuh"

namespace hikf {

namespace {

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

  auto issue = [&](int tile, int stage) {
    double* As = smem + stage * STAGE;
    double* Bs = As + BM * AS;
    const int64_t k0 = kbeg + (int64_t)tile * BK;
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
  for (int tile = 0; tile < ntiles; ++tile) {
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
  }
  cp_async_wait<0>();

  // ---- epilogue ----
  // beta * Cin is read for the whole warp tile before any store: C may alias
  // Cin (in-place C_new = C' - Y P), and separating the phases lets the loads
  // overlap instead of serialising load -> store round trips.
  if (Cin) {
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int64_t row = m0 + wm * TM * 8 + i * 8 + gq;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int64_t col = n0 + wn * TN * 8 + j * 8 + 2 * t4;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double c = 0.0;
          if (row < g.M && col + h < g.N) c = Cin[row * g.ldcin + col + h];
          acc[i][j][h] = g.alpha * acc[i][j][h] + g.beta * c;
        }
      }
    }
  }
  // row partials first (they read w / px), then the stores: keeping the
  // loads ahead of the stores avoids load-after-store serialisation on
  // possibly aliasing pointers
  if (PARTIALS) {
    const double sc = g.px ? 1.0 : (Cin ? 1.0 : g.alpha);
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int rl = wm * TM * 8 + i * 8 + gq;
      const int64_t row = m0 + rl;
      double ssq = 0.0, sdot = 0.0;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int64_t col = n0 + wn * TN * 8 + j * 8 + 2 * t4;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (row < g.M && col + h < g.N) {
            const double v = sc * acc[i][j][h];
            ssq += v * (g.px ? g.px[row * g.ldx + col + h] : v);
            sdot += v * g.w[col + h];
          }
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
  for (int i = 0; i < TM; ++i) {
    const int64_t row = m0 + wm * TM * 8 + i * 8 + gq;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t col = n0 + wn * TN * 8 + j * 8 + 2 * t4;
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (row < g.M && col + h < g.N) C[row * g.ldc + col + h] = Cin ? acc[i][j][h] : g.alpha * acc[i][j][h];
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
        g.pdot[row * g.ldp + blockIdx.x] = d;
      }
    }
  }
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

int g_variant = -1;

}  // namespace

int dgemm_variant() {
  if (g_variant < 0) {
    const char* e = getenv("HIKF_DGEMM_VARIANT");
    g_variant = e ? atoi(e) : 7;  // default: 64x128x16, 3 stages, 2 CTAs per SM (profiles/r01_gemm_sweep*.log)
  }
  return g_variant;
}

void set_dgemm_variant(int v) { g_variant = v; }

int update_variant_y() { return getenv("HIKF_DGEMM_VARIANT") ? dgemm_variant() : 10; }
int update_variant_c() { return getenv("HIKF_DGEMM_VARIANT") ? dgemm_variant() : 7; }

int dgemm(const GemmArgs& g, int batch, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0 || batch <= 0) return HIKF_OK;
  const int variant = g.variant >= 0 ? g.variant : dgemm_variant();
  auto al16 = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  bool vec = g.sa_c == 1 && g.sb_c == 1 && (g.sa_r % 2 == 0) && (g.sb_r % 2 == 0) && al16(g.A) && al16(g.B) &&
             (batch == 1 || (g.bsA % 2 == 0 && g.bsB % 2 == 0));
  bool part = g.psq != nullptr;
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
    default:  // 128x128x16, 8 warps of 64x32, 5 stages
      return launch_variant<128, 128, 16, 2, 4, 5, 1>(g, batch, vec, part, st);
  }
}

}  // namespace hikf

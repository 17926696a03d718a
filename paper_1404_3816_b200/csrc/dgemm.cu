// FP64 DMMA GEMM (see dgemm.cuh).
#include "dgemm.cuh"

namespace hikf {

namespace {

template <bool VEC, bool PARTIALS>
__global__ void __launch_bounds__(DG_THREADS, 1) dgemm_kernel(GemmArgs g) {
  extern __shared__ double smem[];
  __shared__ double red_sq[4][DG_BM];
  __shared__ double red_dot[4][DG_BM];

  const int64_t n0 = (int64_t)blockIdx.x * DG_BN;
  const int64_t m0 = (int64_t)blockIdx.y * DG_BM;
  const int z = blockIdx.z;
  const double* A = g.A + z * g.bsA;
  const double* B = g.B + z * g.bsB;
  double* C = g.C + z * g.bsC;
  const double* Cin = g.Cin ? g.Cin + z * g.bsCin : nullptr;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  const int gq = lane >> 2, t4 = lane & 3;

  int64_t kbeg = 0, kend = g.K;
  if (g.kmode == KB_UPPER) kend = min(g.K, n0 + DG_BN);
  if (g.kmode == KB_LOWER) kbeg = (n0 / DG_BK) * DG_BK;
  const int ntiles = kend > kbeg ? (int)((kend - kbeg + DG_BK - 1) / DG_BK) : 0;

  auto issue = [&](int tile, int stage) {
    double* As = smem + stage * DG_STAGE;
    double* Bs = As + DG_BM * DG_AS;
    const int64_t k0 = kbeg + (int64_t)tile * DG_BK;
    if (VEC) {
#pragma unroll
      for (int it = 0; it < (DG_BM * DG_BK / 2) / DG_THREADS; ++it) {
        int e = tid + it * DG_THREADS;
        int r = e / (DG_BK / 2), kc = (e % (DG_BK / 2)) * 2;
        int64_t row = m0 + r, kk = k0 + kc;
        int bytes = 0;
        const double* src = A;
        if (row < g.M && kk < kend) {
          bytes = (int)(kend - kk) >= 2 ? 16 : 8;
          src = A + row * g.sa_r + kk;
        }
        cp_async16(As + r * DG_AS + kc, src, bytes);
      }
#pragma unroll
      for (int it = 0; it < (DG_BK * DG_BN / 2) / DG_THREADS; ++it) {
        int e = tid + it * DG_THREADS;
        int kr = e / (DG_BN / 2), c = (e % (DG_BN / 2)) * 2;
        int64_t kk = k0 + kr, col = n0 + c;
        int bytes = 0;
        const double* src = B;
        if (kk < kend && col < g.N) {
          bytes = (int)(g.N - col) >= 2 ? 16 : 8;
          src = B + kk * g.sb_r + col;
        }
        cp_async16(Bs + kr * DG_BS + c, src, bytes);
      }
    } else {
#pragma unroll
      for (int it = 0; it < (DG_BM * DG_BK) / DG_THREADS; ++it) {
        int e = tid + it * DG_THREADS;
        int r = e / DG_BK, kc = e % DG_BK;
        int64_t row = m0 + r, kk = k0 + kc;
        bool ok = row < g.M && kk < kend;
        cp_async8(As + r * DG_AS + kc, ok ? A + row * g.sa_r + kk * g.sa_c : A, ok);
      }
#pragma unroll
      for (int it = 0; it < (DG_BK * DG_BN) / DG_THREADS; ++it) {
        int e = tid + it * DG_THREADS;
        int kr = e / DG_BN, c = e % DG_BN;
        int64_t kk = k0 + kr, col = n0 + c;
        bool ok = kk < kend && col < g.N;
        cp_async8(Bs + kr * DG_BS + c, ok ? B + kk * g.sb_r + col * g.sb_c : B, ok);
      }
    }
  };

  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < DG_STAGES - 1; ++s) {
    if (s < ntiles) issue(s, s);
    cp_async_commit();
  }
  for (int tile = 0; tile < ntiles; ++tile) {
    cp_async_wait<DG_STAGES - 2>();
    __syncthreads();
    int nt = tile + DG_STAGES - 1;
    if (nt < ntiles) issue(nt, nt % DG_STAGES);
    cp_async_commit();
    const double* As = smem + (tile % DG_STAGES) * DG_STAGE + (wm * 64) * DG_AS;
    const double* Bs = smem + (tile % DG_STAGES) * DG_STAGE + DG_BM * DG_AS + wn * 32;
#pragma unroll
    for (int kb = 0; kb < DG_BK; kb += 4) {
      double af[8], bf[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) af[i] = As[(i * 8 + gq) * DG_AS + kb + t4];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs[(kb + t4) * DG_BS + j * 8 + gq];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // ---- epilogue ----
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int rl = wm * 64 + i * 8 + gq;
    const int64_t row = m0 + rl;
    double ssq = 0.0, sdot = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t col = n0 + wn * 32 + j * 8 + 2 * t4;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (row < g.M && col + h < g.N) {
          double v = g.alpha * acc[i][j][h];
          if (PARTIALS) {
            ssq += v * v;
            sdot += v * g.w[col + h];
          }
          if (Cin) v += g.beta * Cin[row * g.ldcin + col + h];
          C[row * g.ldc + col + h] = v;
        }
      }
    }
    if (PARTIALS) {
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
  if (PARTIALS) {
    __syncthreads();
    for (int rl = tid; rl < DG_BM; rl += DG_THREADS) {
      int64_t row = m0 + rl;
      if (row < g.M) {
        g.psq[row * g.ldp + blockIdx.x] = ((red_sq[0][rl] + red_sq[1][rl]) + red_sq[2][rl]) + red_sq[3][rl];
        g.pdot[row * g.ldp + blockIdx.x] = ((red_dot[0][rl] + red_dot[1][rl]) + red_dot[2][rl]) + red_dot[3][rl];
      }
    }
  }
}

template <bool VEC, bool P>
int launch_dgemm(const GemmArgs& g, int batch, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    HIKF_CHECK_CUDA(
        cudaFuncSetAttribute(dgemm_kernel<VEC, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DG_SMEM));
    configured = true;
  }
  dim3 grid((unsigned)ceil_div(g.N, DG_BN), (unsigned)ceil_div(g.M, DG_BM), (unsigned)batch);
  dgemm_kernel<VEC, P><<<grid, DG_THREADS, DG_SMEM, st>>>(g);
  HIKF_CHECK_LAUNCH();
  return HIKF_OK;
}

}  // namespace

int dgemm(const GemmArgs& g, int batch, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0 || batch <= 0) return HIKF_OK;
  auto al16 = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  bool vec = g.sa_c == 1 && g.sb_c == 1 && (g.sa_r % 2 == 0) && (g.sb_r % 2 == 0) && al16(g.A) && al16(g.B) &&
             (batch == 1 || (g.bsA % 2 == 0 && g.bsB % 2 == 0));
  bool part = g.psq != nullptr;
  if (vec) return part ? launch_dgemm<true, true>(g, batch, st) : launch_dgemm<true, false>(g, batch, st);
  return part ? launch_dgemm<false, true>(g, batch, st) : launch_dgemm<false, false>(g, batch, st);
}

}  // namespace hikf

// Dense Kalman filter on the GPU (filters.py:45-74) and the dense Gram
// (kernels.py:97-117): the reference's exact-algebra oracle path, used to
// check HiKF == KF on the device at sizes where the m x m covariance fits in
// HBM (cfg2: 34 GB).
//
//   kf_update: C = H P, S = sym(H C^T + r I), K^T = S^-1 C (spd_solve: two
//   triangular applications), mean += K (z - H mean), P = sym(P - K C).
#include <algorithm>

#include "dgemm.cuh"
#include "kf.h"
#include "update.h"

namespace hikf {

namespace {

constexpr int KT = 256;

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

int grid_kf(int64_t n) {
  int64_t b = (n + KT - 1) / KT;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)num_sms() * 32));
}

// G[i][j] = K(|x_i - x_j|), r = 0 -> value_at_zero (log family: 0); symmetric by construction
__global__ void gram_kernel(const double* __restrict__ xy, int64_t m, KParams kp, double* __restrict__ G) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * m; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / m, j = e % m;
    G[e] = kernel_of_r(kp, dist2d(xy[2 * i], xy[2 * i + 1], xy[2 * j], xy[2 * j + 1]));
  }
}

// X (nrows x ncols, ld ncols) = H B, H CSR nrows x (rows of B), B row-major with ld ncols
__global__ void spmm_rect(int64_t ncols, const int32_t* __restrict__ ip, const int32_t* __restrict__ ix,
                          const double* __restrict__ val, const double* __restrict__ B, double* __restrict__ X) {
  const int64_t r = blockIdx.x;
  const int32_t b = ip[r], e1 = ip[r + 1];
  for (int64_t j = threadIdx.x; j < ncols; j += blockDim.x) {
    double s = 0.0;
    for (int32_t e = b; e < e1; ++e) s += val[e] * B[(int64_t)ix[e] * ncols + j];
    X[r * ncols + j] = s;
  }
}

// Y (cols x rows) = X^T, X rows x cols; 32 x 32 tiles through shared memory
__global__ void transpose_rect(const double* __restrict__ X, int64_t rows, int64_t cols, double* __restrict__ Y) {
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = X[r * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) Y[c * rows + r] = tile[threadIdx.x][i];
  }
}

// S = 0.5 ((X + r I) + (X + r I)^T)  (filters.py:67-68)
__global__ void sym_plus_r(const double* __restrict__ X, int64_t n, double r, double* __restrict__ S) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e % n;
    const double a = X[e] + (i == j ? r : 0.0), b = X[j * n + i] + (i == j ? r : 0.0);
    S[e] = 0.5 * (a + b);
  }
}

__global__ void kf_innov(int64_t n, const int32_t* __restrict__ ip, const int32_t* __restrict__ ix,
                         const double* __restrict__ val, const double* __restrict__ mean, const double* __restrict__ z,
                         double* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int32_t e = ip[r]; e < ip[r + 1]; ++e) s += val[e] * mean[ix[e]];
    out[r] = z[r] - s;
  }
}

// mean_out[i] = mean[i] + sum_r K^T[r][i] innov[r]
__global__ void kf_mean(int64_t m, int64_t n, const double* __restrict__ Kt, const double* __restrict__ innov,
                        const double* __restrict__ mean, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t r = 0; r < n; ++r) s += Kt[r * m + i] * innov[r];
    out[i] = mean[i] + s;
  }
}

// P = 0.5 (P + P^T) in place (filters.py:73)
__global__ void sym_inplace(double* __restrict__ P, int64_t m) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * m; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / m, j = e % m;
    if (j <= i) continue;
    const double v = 0.5 * (P[e] + P[j * m + i]);
    P[e] = v;
    P[j * m + i] = v;
  }
}

__global__ void add_rect(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ c,
                         int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    c[e] = a[e] + b[e];
}

}  // namespace

int dense_gram(const double* xy_dev, int64_t m, const KParams& kp, double* G, cudaStream_t st) {
  if (m <= 0) return HIKF_OK;
  gram_kernel<<<grid_kf(m * m), KT, 0, st>>>(xy_dev, m, kp, G);
  HIKF_CHECK_LAUNCH();
  return HIKF_OK;
}

int kf_predict(int64_t m, const double* P, const double* Q, double* P_out, cudaStream_t st) {
  add_rect<<<grid_kf(m * m), KT, 0, st>>>(P, Q, P_out, m * m);
  HIKF_CHECK_LAUNCH();
  return HIKF_OK;
}

size_t kf_workspace_bytes(int64_t m, int64_t n) {
  return align_up(8 * n * m) * 3 + align_up(8 * n * n) * 2 + align_up(8 * std::max<int64_t>(n, 1)) +
         spd_workspace_bytes(n, m);
}

int kf_update(int64_t m, int64_t n, const double* mean, const double* P, const int32_t* ip, const int32_t* ix,
              const double* val, double r, const double* z, double* mean_out, double* P_out, void* ws,
              size_t ws_bytes, cudaStream_t st) {
  if (ws_bytes < kf_workspace_bytes(m, n)) {
    set_error("kf_update workspace too small");
    return HIKF_BAD_ARGUMENT;
  }
  if (n == 0) {  // filters.py:64-65: the state is returned unchanged
    HIKF_CHECK_CUDA(cudaMemcpyAsync(mean_out, mean, sizeof(double) * m, cudaMemcpyDeviceToDevice, st));
    HIKF_CHECK_CUDA(cudaMemcpyAsync(P_out, P, sizeof(double) * m * m, cudaMemcpyDeviceToDevice, st));
    return HIKF_OK;
  }
  char* p = (char*)ws;
  auto take = [&](size_t bytes) {
    char* q = p;
    p += align_up(bytes);
    return q;
  };
  double* C = (double*)take(8 * n * m);   // H P          (n x m)
  double* Ct = (double*)take(8 * n * m);  // C^T, then K  (m x n)
  double* Kt = (double*)take(8 * n * m);  // S^-1 C       (n x m)
  double* X = (double*)take(8 * n * n);
  double* S = (double*)take(8 * n * n);
  double* innov = (double*)take(8 * n);
  void* sws = take(spd_workspace_bytes(n, m));
  spmm_rect<<<(unsigned)n, KT, 0, st>>>(m, ip, ix, val, P, C);
  HIKF_CHECK_LAUNCH();
  const dim3 tb(32, 8);
  transpose_rect<<<dim3((unsigned)((m + 31) / 32), (unsigned)((n + 31) / 32)), tb, 0, st>>>(C, n, m, Ct);
  HIKF_CHECK_LAUNCH();
  spmm_rect<<<(unsigned)n, KT, 0, st>>>(n, ip, ix, val, Ct, X);  // H C^T
  HIKF_CHECK_LAUNCH();
  sym_plus_r<<<grid_kf(n * n), KT, 0, st>>>(X, n, r, S);
  HIKF_CHECK_LAUNCH();
  int64_t info = 0;
  HIKF_TRY(spd_solve(n, m, S, C, Kt, sws, spd_workspace_bytes(n, m), &info, st));
  kf_innov<<<grid_kf(n), KT, 0, st>>>(n, ip, ix, val, mean, z, innov);
  HIKF_CHECK_LAUNCH();
  kf_mean<<<grid_kf(m), KT, 0, st>>>(m, n, Kt, innov, mean, mean_out);
  HIKF_CHECK_LAUNCH();
  transpose_rect<<<dim3((unsigned)((m + 31) / 32), (unsigned)((n + 31) / 32)), tb, 0, st>>>(Kt, n, m, Ct);  // K
  HIKF_CHECK_LAUNCH();
  GemmArgs g;  // P_out = P - K C
  g.M = m; g.N = m; g.K = n;
  g.A = Ct; g.sa_r = n;
  g.B = C; g.sb_r = m;
  g.C = P_out; g.ldc = m;
  g.Cin = P; g.ldcin = m;
  g.alpha = -1.0; g.beta = 1.0;
  HIKF_TRY(dgemm(g, 1, st));
  sym_inplace<<<grid_kf(m * m), KT, 0, st>>>(P_out, m);
  HIKF_CHECK_LAUNCH();
  return HIKF_OK;
}

}  // namespace hikf

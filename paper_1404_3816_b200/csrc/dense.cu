// Direct-sum Q H^T for hikf_precompute_dense (filters.py:108-115, kernels.py:97-117).
//
// The reference forms the dense Gram Q (m x m) and multiplies it by the
// densified H^T.  Here Q is never stored: C_Q[i, ray] = sum over the ray's
// cells c of K(|x_i - x_c|) * len_c, i.e. Q @ H^T restricted to the nonzeros
// of H^T (every skipped term is an exact zero).  K uses the same device
// evaluation as the FMM (kernel_of_r on the no-FMA distance), with K(0) =
// value_at_zero for the log family.
//
// One CTA = 128 targets x 8 rays; each ray's (x, y, len) entries are staged in
// shared memory in chunks, each thread accumulates its target's 8 ray sums in
// CSR order and writes 8 contiguous doubles of its C_Q row.
#include "dense.h"

namespace hikf {

namespace {

constexpr int DT = 128;     // targets per CTA (one per thread)
constexpr int DR = 8;       // rays per CTA
constexpr int DCHUNK = 512;  // staged entries per chunk

__global__ void __launch_bounds__(DT) direct_cq(int64_t m, int64_t n, const double* __restrict__ xy,
                                                const int32_t* __restrict__ ip, const int32_t* __restrict__ ix,
                                                const double* __restrict__ val, KParams kp, double* __restrict__ CQ) {
  __shared__ double sx[DCHUNK], sy[DCHUNK], sh[DCHUNK];
  const int64_t i = blockIdx.x * (int64_t)DT + threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * DR;
  const double xi = i < m ? xy[2 * i] : 0.0, yi = i < m ? xy[2 * i + 1] : 0.0;
  double acc[DR];
#pragma unroll
  for (int q = 0; q < DR; ++q) acc[q] = 0.0;
#pragma unroll
  for (int q = 0; q < DR; ++q) {
    const int64_t r = r0 + q;
    if (r >= n) break;
    const int32_t b = ip[r], e = ip[r + 1];
    for (int32_t c0 = b; c0 < e; c0 += DCHUNK) {
      const int cn = min(DCHUNK, e - c0);
      __syncthreads();
      for (int t = threadIdx.x; t < cn; t += DT) {
        const int32_t col = ix[c0 + t];
        sx[t] = xy[2 * (int64_t)col];
        sy[t] = xy[2 * (int64_t)col + 1];
        sh[t] = val[c0 + t];
      }
      __syncthreads();
      double s = acc[q];
      for (int t = 0; t < cn; ++t) s += kernel_of_r(kp, dist2d(xi, yi, sx[t], sy[t])) * sh[t];
      acc[q] = s;
    }
  }
  if (i >= m) return;
#pragma unroll
  for (int q = 0; q < DR; ++q)
    if (r0 + q < n) CQ[i * n + r0 + q] = acc[q];
}

}  // namespace

int dense_cq(int64_t m, int64_t n, const double* xy_dev, const int32_t* ip, const int32_t* ix, const double* val,
             const KParams& kp, double* CQ, cudaStream_t st) {
  if (m <= 0 || n <= 0) return HIKF_OK;
  dim3 grid((unsigned)ceil_div(m, DT), (unsigned)ceil_div(n, DR));
  direct_cq<<<grid, DT, 0, st>>>(m, n, xy_dev, ip, ix, val, kp, CQ);
  HIKF_CHECK_LAUNCH();
  return HIKF_OK;
}

}  // namespace hikf

// Cholesky + inverse of one <= 64 x 64 diagonal block (device function shared by
// the recursive multi-launch factorisation in update.cu and the fused n x n
// chain programs in nnchain.cu, so both produce bit-identical factors).
// Called by all 256 threads of a CTA; base_smem: 2 x 64 x 65 doubles.
#pragma once

#include "common.cuh"

namespace hikf {

constexpr int CHOL_NB = 64;
constexpr size_t CHOL_SMEM = 2 * CHOL_NB * (CHOL_NB + 1) * sizeof(double);

// Cholesky + inverse of one <= CHOL_NB x CHOL_NB diagonal block held in shared memory.
// L (lower, ld), Li (lower, ld) written; upper triangles left untouched (zeroed
// by the caller).  status[0] = global 1-based pivot of the first failure.
// Right-looking factorisation: every thread recomputes the pivot (no extra
// barrier), warp w updates rows i = w (mod 8) of the trailing triangle.
__device__ __forceinline__ void chol_inv_block(const double* __restrict__ S, int64_t ld, int nb, int64_t offset,
                                               double* __restrict__ L, double* __restrict__ Li, int* status,
                                               double* base_smem) {
  double(*a)[CHOL_NB + 1] = reinterpret_cast<double(*)[CHOL_NB + 1]>(base_smem);
  double(*x)[CHOL_NB + 1] = reinterpret_cast<double(*)[CHOL_NB + 1]>(base_smem + CHOL_NB * (CHOL_NB + 1));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < nb * nb; e += blockDim.x) {
    int i = e / nb, k = e - i * nb;
    a[i][k] = S[(int64_t)i * ld + k];
  }
  __syncthreads();
  // Right-looking Cholesky with the lower triangle in registers: thread t owns
  // the elements e = t, t + 256, ... of the packed triangle (i >= k).  Per column
  // j the owner of (j, j) publishes it, the owners of column j scale their
  // entries and publish them, and every owner applies a[i][k] -= a[i][j] a[k][j]
  // (k > j) in registers -- the same operations in the same order as updating
  // a shared-memory copy, with two barriers per column (double-buffered).
  constexpr int EPT = (CHOL_NB * (CHOL_NB + 1) / 2 + 255) / 256;  // elements per thread
  __shared__ double colb[2][CHOL_NB];
  __shared__ double diagb[2];
  const int ne = nb * (nb + 1) / 2;
  double el[EPT];
  int ei[EPT], ek[EPT];
#pragma unroll
  for (int q = 0; q < EPT; ++q) {
    const int e = tid + q * 256;
    int i = 0, k = 0;
    if (e < ne) {
      i = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while ((i + 1) * (i + 2) / 2 <= e) ++i;
      while (i * (i + 1) / 2 > e) --i;
      k = e - i * (i + 1) / 2;
      el[q] = a[i][k];
    } else {
      i = k = -1;
      el[q] = 0.0;
    }
    ei[q] = i;
    ek[q] = k;
  }
  int bad = 0;
  for (int j = 0; j < nb; ++j) {
    const int b = j & 1;
#pragma unroll
    for (int q = 0; q < EPT; ++q)
      if (ei[q] == j && ek[q] == j) diagb[b] = el[q];
    __syncthreads();
    double d = diagb[b];
    if (!(d > 0.0)) {
      if (!bad) bad = j + 1;
      d = 1.0;  // keep going; the result is discarded by the caller
    }
    const double piv = sqrt(d);
    const double inv = 1.0 / piv;
#pragma unroll
    for (int q = 0; q < EPT; ++q) {
      if (ek[q] == j && ei[q] > j) {  // column j below the diagonal
        el[q] *= inv;
        colb[b][ei[q]] = el[q];
      } else if (ek[q] == j && ei[q] == j) {
        el[q] = piv;
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < EPT; ++q)
      if (ek[q] > j) el[q] = fma(-colb[b][ei[q]], colb[b][ek[q]], el[q]);
  }
#pragma unroll
  for (int q = 0; q < EPT; ++q)
    if (ei[q] >= 0) a[ei[q]][ek[q]] = el[q];
  __syncthreads();
  // inverse, right-looking over k (row k of x final after step k, then every
  // row i > k takes its next fma): each element's fma chain in k order, the
  // 64 columns' chains advancing together
  __shared__ double rdiag[CHOL_NB];
  __shared__ double xrow[2][CHOL_NB];
  for (int i = tid; i < nb; i += blockDim.x) rdiag[i] = 1.0 / a[i][i];
  __syncthreads();
  double xs[EPT];
#pragma unroll
  for (int q = 0; q < EPT; ++q) xs[q] = 0.0;
  for (int k = 0; k < nb; ++k) {
    const int b = k & 1;
    const double rk = rdiag[k];
#pragma unroll
    for (int q = 0; q < EPT; ++q)
      if (ei[q] == k) {
        xs[q] = ek[q] == k ? rk : -xs[q] * rk;
        xrow[b][ek[q]] = xs[q];
      }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < EPT; ++q)
      if (ei[q] > k && ek[q] <= k) xs[q] = fma(a[ei[q]][k], xrow[b][ek[q]], xs[q]);
  }
#pragma unroll
  for (int q = 0; q < EPT; ++q)
    if (ei[q] >= 0) x[ei[q]][ek[q]] = xs[q];
  __syncthreads();
  for (int e = tid; e < nb * nb; e += blockDim.x) {
    int i = e / nb, k = e - i * nb;
    if (k <= i) {
      L[(int64_t)i * ld + k] = a[i][k];
      Li[(int64_t)i * ld + k] = x[i][k];
    }
  }
  if (tid == 0 && bad && status[0] == 0) status[0] = (int)(offset + bad);
}


}  // namespace hikf

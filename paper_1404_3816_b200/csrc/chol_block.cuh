// Cholesky + inverse of one <= 64 x 64 diagonal block (device function shared by
// the recursive multi-launch factorisation in update.cu and the fused n x n
// chain programs in nnchain.cu, so both produce bit-identical factors).
// Called by all 256 threads of a CTA; base_smem: 2 x 64 x 65 doubles.
#pragma once

#include "common.cuh"

namespace hikf {

constexpr int CHOL_NB = 64;
constexpr size_t CHOL_SMEM = 2 * CHOL_NB * (CHOL_NB + 1) * sizeof(double);

#ifdef CHOL_BENCH_CLOCK
#define CHOL_STAMP(slot) \
  if (threadIdx.x == 0) CHOL_BENCH_CLOCK[slot] = clock64()
#else
#define CHOL_STAMP(slot)
#endif

__device__ __forceinline__ int chol_ld_acquire(unsigned addr) {
  int v;
  asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void chol_st_release(unsigned addr, int v) {
  asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// Cholesky + inverse of one <= CHOL_NB x CHOL_NB diagonal block.
// L (lower, ld), Li (lower, ld) written; upper triangles left untouched (zeroed
// by the caller).  status[0] = global 1-based pivot of the first failure.
//
// The arithmetic (fixed: the multi-launch and fused chains share it, and it is
// what the factor's bits depend on):
//   Cholesky  a_ik <- fma(-L_ij, L_kj, a_ik) for j = 0 .. k-1 in order, then
//             L_kk = sqrt(a_kk), inv_k = 1 / L_kk, L_ik = a_ik * inv_k (i > k);
//   inverse   x_cc = inv_c, x_ic = (-(fma chain over k = c .. i-1 of L_ik x_kc)) * inv_i.
// The schedule is warp-level (the block is latency-bound, ~2 x 64 dependent
// steps): warp w owns the columns w, w + 8, ... and lane l the rows l, l + 32.
//   Cholesky, left-looking: a warp accumulates its column's fma chain as soon
//     as each earlier column is published (a shared-memory counter with
//     release / acquire, no CTA barrier), so only the last fma, the pivot
//     broadcast (shuffle), sqrt and reciprocal sit on the column-to-column path.
//   Inverse: the 64 columns are independent forward substitutions; a warp runs
//     its 8 columns over k together, x_kc broadcast by shuffle from the row's
//     owner -- no barrier at all.
// Called by all 256 threads of a CTA; base_smem: 2 x 64 x 65 doubles.
__device__ __forceinline__ void chol_inv_block(const double* __restrict__ S, int64_t ld, int nb, int64_t offset,
                                               double* __restrict__ L, double* __restrict__ Li, int* status,
                                               double* base_smem) {
  double(*a)[CHOL_NB + 1] = reinterpret_cast<double(*)[CHOL_NB + 1]>(base_smem);
  double(*x)[CHOL_NB + 1] = reinterpret_cast<double(*)[CHOL_NB + 1]>(base_smem + CHOL_NB * (CHOL_NB + 1));
  __shared__ double rdiag[CHOL_NB];
  __shared__ int ncols, sbad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr unsigned full = 0xffffffffu;
  for (int e = tid; e < nb * nb; e += blockDim.x) {
    int i = e / nb, k = e - i * nb;
    if (k <= i) a[i][k] = S[(int64_t)i * ld + k];
  }
  if (tid == 0) {
    ncols = 0;
    sbad = 0x7fffffff;
  }
  __syncthreads();
  CHOL_STAMP(4);
  const int r0 = lane, r1 = lane + 32;
  const unsigned ncols_addr = (unsigned)__cvta_generic_to_shared(&ncols);
  int avail = 0;
  for (int k = warp; k < nb; k += 8) {
    double acc0 = a[r0][k], acc1 = a[r1][k];  // rows < k or >= nb: unused
    for (int j = 0; j < k; ++j) {
      if (j >= avail) {
        do {
          avail = chol_ld_acquire(ncols_addr);  // columns < avail are published
        } while (avail <= j);
      }
      const double lkj = a[k][j];
      acc0 = fma(-a[r0][j], lkj, acc0);
      acc1 = fma(-a[r1][j], lkj, acc1);
    }
    double d = __shfl_sync(full, k < 32 ? acc0 : acc1, k & 31);
    if (!(d > 0.0)) {
      if (lane == 0) atomicMin(&sbad, k + 1);
      d = 1.0;  // keep going; the result is discarded by the caller
    }
    const double piv = sqrt(d);
    const double inv = 1.0 / piv;
    if (r0 > k && r0 < nb) a[r0][k] = acc0 * inv;
    if (r1 > k && r1 < nb) a[r1][k] = acc1 * inv;
    if (lane == (k & 31)) {
      a[k][k] = piv;
      rdiag[k] = inv;
    }
    __syncwarp();
    if (lane == 0) chol_st_release(ncols_addr, k + 1);
  }
  CHOL_STAMP(12);
  __syncthreads();
  CHOL_STAMP(13);
  for (int e = tid; e < nb * nb; e += blockDim.x) {
    int i = e / nb, k = e - i * nb;
    if (k <= i) L[(int64_t)i * ld + k] = a[i][k];
  }
  // acc[cc][h]: the fma chain of x(row r_h = lane + 32 h, column c = warp + 8 cc),
  // complete for row k after step k - 1, when x_kc = -acc * inv_k.  The chain of
  // the diagonal element starts at -1 (so x_cc = -(-1) * inv_c = inv_c exactly,
  // without a select) and every other at +0; every step then updates every
  // column and row unpredicated: a column c > k receives fma(l, -0, acc) and
  // a finished row r <= k fma(0, x, acc), both adding a zero, which leaves a
  // chain value (nonzero, or +0) bit-unchanged.
  double acc[8][2];
#pragma unroll
  for (int cc = 0; cc < 8; ++cc) {
    acc[cc][0] = r0 == warp + 8 * cc ? -1.0 : 0.0;
    acc[cc][1] = r1 == warp + 8 * cc ? -1.0 : 0.0;
  }
  const int kmid = nb < 32 ? nb : 32;
  for (int k = warp; k < kmid; ++k) {  // rows k < 32 broadcast from the first halves
    const double rk = rdiag[k];
    const double l0 = r0 > k ? a[r0][k] : 0.0, l1 = a[r1][k];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      const double fin = -__shfl_sync(full, acc[cc][0], k) * rk;  // x_kc
      acc[cc][0] = fma(l0, fin, acc[cc][0]);
      acc[cc][1] = fma(l1, fin, acc[cc][1]);
    }
  }
  for (int k = warp > 32 ? warp : 32; k < nb; ++k) {  // rows k >= 32: only the second halves move
    const double rk = rdiag[k];
    const double l1 = r1 > k ? a[r1][k] : 0.0;
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      const double fin = -__shfl_sync(full, acc[cc][1], k - 32) * rk;
      acc[cc][1] = fma(l1, fin, acc[cc][1]);
    }
  }
#pragma unroll
  for (int cc = 0; cc < 8; ++cc) {
    const int c = warp + 8 * cc;
    if (r0 >= c && r0 < nb) x[r0][c] = -acc[cc][0] * rdiag[r0];
    if (r1 >= c && r1 < nb) x[r1][c] = -acc[cc][1] * rdiag[r1];
  }
  CHOL_STAMP(14);
  __syncthreads();
  for (int e = tid; e < nb * nb; e += blockDim.x) {
    int i = e / nb, k = e - i * nb;
    if (k <= i) Li[(int64_t)i * ld + k] = x[i][k];
  }
  if (tid == 0 && sbad != 0x7fffffff && status[0] == 0) status[0] = (int)(offset + sbad);
  __syncthreads();
}

}  // namespace hikf

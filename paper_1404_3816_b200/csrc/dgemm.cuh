// FP64 GEMM on the DMMA tensor path (mma.sync m8n8k4 -> SASS DMMA.8x8x4).
//
// sm_100a has no tcgen05 f64 kind, so FP64 matrix work runs on the warp-level
// DMMA pipe (measured 37.0 TFLOP/s on this B200, same as DFMA).  dgemm() is the
// workhorse of the per-step update: hand-written mainloops (dgemm.cu) with
// triangular K-range skipping for triangular B and fused epilogues (alpha/beta,
// per-row sum of squares / dot with a vector, the chained predict output, a
// GEMV over A, a sparse-row addend).
#pragma once

#include "common.cuh"

namespace hikf {

enum { KFULL = 0, KB_UPPER = 1, KB_LOWER = 2 };

struct GemmArgs {
  int64_t M = 0, N = 0, K = 0;
  const double* A = nullptr;  // A[i][k] = A[i * sa_r + k * sa_c]
  int64_t sa_r = 0, sa_c = 1;
  const double* B = nullptr;  // B[k][j] = B[k * sb_r + j * sb_c]
  int64_t sb_r = 0, sb_c = 1;
  double* C = nullptr;        // C[i][j] = C[i * ldc + j]
  int64_t ldc = 0;
  const double* Cin = nullptr;  // beta term source (may alias C)
  int64_t ldcin = 0;
  double alpha = 1.0, beta = 0.0;
  int kmode = KFULL;
  int64_t bsA = 0, bsB = 0, bsC = 0, bsCin = 0;  // batch strides (blockIdx.z)
  // fused row partials over the CTA's column tile:
  //   px == null: psq[i * ldp + tile] = sum_j (alpha acc)^2, pdot[...] = sum_j (alpha acc) w[j]
  //   px != null: psq[i * ldp + tile] = sum_j acc px[i * ldx + j], pdot[...] = sum_j acc w[j]
  double* psq = nullptr;
  double* pdot = nullptr;
  const double* w = nullptr;
  int64_t ldp = 0;
  const double* px = nullptr;
  int64_t ldx = 0;
  // optional second output: chain_out = C (as stored) + chain_add, same indexing with ldch
  const double* chain_add = nullptr;
  double* chain_out = nullptr;
  int64_t ldch = 0;
  // optional fused GEMV over A (row-major variants 30-34): gv_y[i] = sum_k A[i][k] gv_x[k] for all M rows,
  // done by the CTAs of the last column tile (the shortest k-range under KB_LOWER) from the A
  // panel their row block just streamed through L2
  const double* gv_x = nullptr;
  double* gv_y = nullptr;
  // optional sparse-row addend before the partials (PARTIALS, px == null): the value of
  // element (i, j) becomes alpha (acc + sp_alpha sum_{e in row i of the CSR sp} sp_val[e] sp_Y[sp_ix[e]][j])
  // (the factored update with C_0 = alpha H^T: sp = H^T, sp_Y = Y)
  const int32_t *sp_ip = nullptr, *sp_ix = nullptr;
  const double* sp_val = nullptr;
  const double* sp_Y = nullptr;
  int64_t sp_ldy = 0;
  double sp_alpha = 0.0;
  int variant = -1;  // tile-shape variant (-1: dgemm_variant())
};

// C = alpha * A B + beta * Cin (+ partials); launches on `stream`.
int dgemm(const GemmArgs& g, int batch, cudaStream_t stream);
// tile-shape variant in use (0 = default); HIKF_DGEMM_VARIANT overrides
int dgemm_variant();
void set_dgemm_variant(int v);
// number of column tiles (= partial sums per row) the current variant uses for N columns
inline int dgemm_col_tiles(int64_t N, int variant = -1) {
  int v = variant >= 0 ? variant : dgemm_variant();
  return ceil_div(N, v == 32 ? 64 : 128);
}
// variant used by the update's K GEMM (tools/gemm_sweep.py, profiles/r01_gemm_sweep*.log);
// HIKF_DGEMM_VARIANT overrides it
int update_variant_c(int64_t n);
constexpr int DG_MIN_BN = 64;  // smallest column tile of any variant (partials workspace sizing)

}  // namespace hikf

// Fused n x n chain of the per-step update for small n (nnchain.cu).
#pragma once

#include <vector>

#include "common.cuh"

namespace hikf {

// Operand table of a chain program: programs name buffers by id, every launch
// binds the ids to this call's pointers.
enum NnBuf {
  NB_HC = 0, NB_HCQ, NB_HCP, NB_S, NB_L, NB_LI, NB_LIT, NB_SINV, NB_TMP, NB_P, NB_R, NB_HCOUT,
  NB_LA_HC, NB_LA_HCQ, NB_LA_HCP, NB_LA_LI, NB_LA_LIT, NB_LA_SINV, NB_COUNT
};
enum NnIBuf { NI_STATUS = 0, NI_LA_STATUS, NI_FLAG, NI_COUNT };

struct NnPtrs {
  double* d[NB_COUNT] = {};
  int* i[NI_COUNT] = {};
  double r = 0.0;
  int64_t n = 0;
  int force_miss = 1;  // 1: the look-ahead is not usable (host-side checks failed): factorise
  // innovation (z - H mean, or z - Hmean for a row-sharded state) into innov
  const int32_t *ip = nullptr, *ix = nullptr;
  const double *val = nullptr, *mean = nullptr, *z = nullptr, *Hmean = nullptr;
  double* innov = nullptr;
};

// largest n the fused programs take (bigger n: the multi-launch chain, hidden under the GEMM;
// at n = 480 the cooperative post-GEMM program slowed the concurrent K-GEMM by 20 %)
constexpr int64_t NN_FUSED_MAX = 256;
bool nn_fused_enabled(int64_t n);
int nn_set_fused(int on);  // returns the previous setting

// The pre-GEMM program: HC' = HC + HC_Q, the innovation, the device-side
// look-ahead probe (HC, HC_Q bitwise equal to the look-ahead's inputs) and then
// either the copy of the look-ahead's factor (hit) or the factorisation of
// S = sym(HC') + r I (miss): Li, Li^T, S^-1 and the pivot status.
int nn_pre(const NnPtrs& p, bool probe, cudaStream_t st);
// The post-GEMM program (concurrent with the K GEMM): HC_out = HC' - (HC' Li^T)(Li HC')
// and, with lookahead, the factorisation of the next step's S = sym(HC_out + HC_Q) + r I
// into the look-ahead buffers (their inputs saved for the next probe).
int nn_post(const NnPtrs& p, bool lookahead, cudaStream_t st);

}  // namespace hikf

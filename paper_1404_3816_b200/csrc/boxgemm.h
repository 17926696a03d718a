// Box-streaming DMMA GEMM for the L2L / L2P transfers (see boxgemm.cu).
#pragma once

#include "common.cuh"
#include "tree.h"

namespace hikf {

// L_l[child][a][j] = S[tmap[child n + j]][a] (0 without a slot) + sum_b C_child[a][b] L_{l-1}[parent][b][j] for every
// child of an occupied parent (l > 2); S is the pair-major M2L scratch of level l
// (parents outside the box-column range [pxlo, pxhi] of level l-1 are skipped)
int l2l_boxes(const hikf_tree* t, int l, const double* S, const int32_t* tmap, const double* Lp, int64_t n,
              double* L, cudaStream_t st, int64_t pxlo = 0, int64_t pxhi = INT64_MAX);
// whether the warp-streaming kernel handles R rows x K inner (K <= 64, A fits in smem)
bool box_supported(int rows, int K);
// L2L of a level child-major (one CTA per occupied child box, 1) or parent-major (0); tuning key 4
int l2l_set_child_major(int on);
// U[order[p]][j] = sum_a W2[p][a] L_leaf[a][j] (store)
// U = W2 L_leaf; with a row window only original rows r0 <= row < r1 are written, to U + (row - r0) ldu
int l2p_boxes(const hikf_tree* t, const double* Lleaf, int64_t n, double* U, int64_t ldu, cudaStream_t st,
              int64_t r0 = 0, int64_t r1 = -1, const LeafWindow* lw = nullptr);

// Fused leaf-level L2L + L2P (the leaf locals stay on chip): U rows of every leaf
// = W2 (S_D[leaf] + C_ci L_{D-1}[parent]); bit-identical to l2l_boxes + l2p_boxes.
// Needs depth >= 3, <= 64 points per leaf and (leaf order, parent order) in
// {(o, o), (o, o + 1)}, 2 <= o <= 8 (leaf_down_supported).
bool leaf_down_supported(const hikf_tree* t);
bool leaf_fused_enabled();
int leaf_set_fused(int on);  // returns the previous setting
// With Pnear (the near-field sums p2p_sparse parked per (leaf, ray) item, item-major), items and
// item_start, the leaf step also adds them: U = far + near, the same single add as
// sparse_p2p_scatter, without its scattered read-modify-write pass (n <= 16384 rays).
bool leaf_down_adds_near(int64_t n);
int leaf_down(const hikf_tree* t, const double* S, const int32_t* tmap, const double* Lp, int64_t n, double* U,
              int64_t ldu, cudaStream_t st, int64_t r0 = 0, int64_t r1 = -1, const LeafWindow* lw = nullptr,
              const double* Pnear = nullptr, const int64_t* items = nullptr, const int32_t* item_start = nullptr);

}  // namespace hikf

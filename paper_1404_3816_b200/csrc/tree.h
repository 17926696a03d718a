// Internal layout of an FMM tree handle (the opaque hikf_tree of the C ABI).
//
// HBM layout (all device arrays owned by the handle):
//   xy        m x 2   point coordinates, original order
//   xy_s      m x 2   coordinates in leaf (sorted-key) order
//   order     m       sorted position -> original point index (= FmmTree._order)
//   leaf_*    L       occupied leaves in ascending box key (x-major bx*G+by):
//                     box id, first sorted position, point count
//   box2leaf  G*G     leaf rank of a box or -1
//   occ[l]    per level 2..depth: ids of boxes with >= 1 point below them,
//             occ_flag[l] the same as a dense G_l*G_l byte map
//   W2s       m x q   leaf interpolation weights S_ix(xi) S_iy(eta), sorted order
//   m2l[l]    40 x q_l x q_l   M2L operators in the reference's offset order
//   shift[l]  4 x q_{l+1} x q_l  kron(Bx, By) child->parent operators (l < depth)
#pragma once

#include <stdint.h>

#include <vector>

#include "common.cuh"
#include "host_ops.h"

struct hikf_tree {
  int64_t m = 0;
  hikf_kernel spec{};
  hikf::KParams kp{};
  int n_cheb = 0;
  int64_t max_leaf = 0;
  double lo[2] = {0, 0};
  double size = 0;
  int depth = 0;
  int64_t G = 1;
  int orders[hikf::kMaxDepth + 1] = {0};

  double* xy = nullptr;
  double* xy_s = nullptr;
  int64_t* order = nullptr;
  int32_t* inv_order = nullptr;  // point -> sorted position
  int32_t* leaf_of = nullptr;    // sorted position -> leaf rank
  int32_t* leaf_box = nullptr;
  int32_t* leaf_start = nullptr;
  int32_t* leaf_count = nullptr;
  int32_t* box2leaf = nullptr;
  int64_t n_leaves = 0;
  int64_t max_count = 0;
  int32_t* occ[hikf::kMaxDepth + 1] = {nullptr};
  uint8_t* occ_flag[hikf::kMaxDepth + 1] = {nullptr};
  int64_t n_occ[hikf::kMaxDepth + 1] = {0};

  double* W2s = nullptr;
  // near-field kernel blocks (fmm.py:166-201 builds `near` at tree construction too):
  // near[((T * 9 + s) * 64 + c) * 64 + t] = K(x_t, x_c) for target leaf T, its neighbour
  // slot s (ox outer, oy inner), local source point c and local target point t; null when
  // a leaf holds more than 64 points or the blocks would not fit (P2P then evaluates K)
  double* near = nullptr;
  double* m2l[hikf::kMaxDepth + 1] = {nullptr};
  uint64_t m2l_present[hikf::kMaxDepth + 1] = {0};  // bit s: offset s has pairs at this level
  double* shift[hikf::kMaxDepth + 1] = {nullptr};

  // host copies (parity export, near-pair enumeration)
  std::vector<int64_t> h_leaf_box, h_leaf_start, h_leaf_count;
};

namespace hikf {

// The 40 M2L offsets, dx outer / dy inner (fmm.py:280-284).
struct M2LOffsets {
  int dx[40], dy[40];
  M2LOffsets() {
    int s = 0;
    for (int x = -3; x <= 3; ++x)
      for (int y = -3; y <= 3; ++y)
        if ((x < 0 ? -x : x) >= 2 || (y < 0 ? -y : y) >= 2) {
          dx[s] = x;
          dy[s] = y;
          ++s;
        }
  }
};

int tree_build(const double* xy_host, int64_t m, const hikf_kernel& k, int n_cheb, int64_t max_leaf,
               cudaStream_t stream, hikf_tree** out);
void tree_free(hikf_tree* t);
int tree_export_m2l_pairs(const hikf_tree* t, int lev, int dx, int dy, std::vector<int64_t>& tgt,
                          std::vector<int64_t>& src);

// U = tree @ V (dense V, m x k), fmm.py:325-367
int fmm_matmat(hikf_tree* t, const double* V, int64_t ldv, int64_t k, double* U, int64_t ldu, cudaStream_t stream);
// U (m x n) = tree @ H^T for a device CSR H (n x m), H^T kept sparse
// U = Q H^T; with a row window only original rows r0 <= row < r1 are produced, at U + (row - r0) n
// Leaf-aligned shard (hikf_precompute_leaves): only the points of leaves [leaf0, leaf1),
// rows in leaf order (sorted positions s0 .. s1-1 -> U rows 0 .. s1-s0-1); x0 / x1 = the
// leaf-level box-column range of those leaves (their ancestors' columns are x >> (D - l)).
struct LeafWindow {
  int64_t leaf0 = 0, leaf1 = 0, s0 = 0, s1 = 0, x0 = 0, x1 = 0;
};
int leaf_window(const hikf_tree* t, int64_t leaf0, int64_t leaf1, LeafWindow* w);
int fmm_matmat_csrT(hikf_tree* t, int64_t n, const int32_t* ip, const int32_t* ix, const double* val, double* U,
                    cudaStream_t stream, int64_t r0 = 0, int64_t r1 = -1, const LeafWindow* lw = nullptr);

}  // namespace hikf

// H^T in leaf-grouped sparse form for the Q H^T precompute (see sparse.cu).
#pragma once

#include "common.cuh"
#include "host_ops.h"

struct hikf_tree;

namespace hikf {
struct LeafWindow;
}

namespace hikf {

struct SparseHt {
  int64_t n = 0, nnz = 0, ngroups = 0, nitems = 0, ngr = 0;
  bool build_masks = false;    // per-level 8-ray activity masks (masked dense M2L path)
  int32_t* e_sp = nullptr;     // entry: sorted position of the cell
  int32_t* e_j = nullptr;      // entry: ray
  double* e_v = nullptr;       // entry: intersection length
  int32_t* g_j = nullptr;      // group (leaf, ray): ray
  int32_t* g_start = nullptr;  // group -> first entry, [ngroups + 1]
  int32_t* leaf_g = nullptr;   // leaf -> first group, [n_leaves + 1]
  int32_t* g_leaf = nullptr;   // group (leaf, ray): leaf rank
  int64_t* items = nullptr;    // P2P work items: target_leaf * n + ray (ascending)
  int32_t* item_start = nullptr;  // target leaf -> first item, [n_leaves + 1]
  uint8_t* mask[21] = {nullptr};  // per level: (G_l^2, ngr) activity of 8-ray groups (optional)
};

// Active multipoles of one level in compact form: (box, ray) pairs with a
// nonzero multipole, sorted by key = box * n + ray, and their q coefficients.
struct PairLevel {
  int64_t np = 0;             // pairs, or (deferred mode) the allocated bound with the count in np_dev
  int32_t* np_dev = nullptr;  // deferred mode: the number of pairs, on the device
  int64_t* key = nullptr;
  double* W = nullptr;  // np x q
};

int sparse_build(const hikf_tree* t, int64_t n, const int32_t* ip, const int32_t* ix, const double* val, SparseHt* s,
                 cudaStream_t st);
void sparse_free(SparseHt* s, cudaStream_t st);
int sparse_p2m(const hikf_tree* t, const SparseHt& s, double* W, int64_t kcols, int64_t c0, cudaStream_t st);
// near field of the (target leaf, ray) items: U += near sum, or, with Pnear
// (nitems x max_count, item-major), the sums are parked there and added by the fused leaf
// step (leaf_down) or by sparse_p2p_scatter
// (row window as l2p_boxes: only original rows r0 <= row < r1, at U + (row - r0) ldu)
// (lw: leaf-aligned shard -- items of other target leaves are skipped, U rows are sorted
//  positions - lw->s0)
int sparse_p2p(const hikf_tree* t, const SparseHt& s, double* U, int64_t ldu, cudaStream_t st,
               double* Pnear = nullptr, int64_t r0 = 0, int64_t r1 = -1, const LeafWindow* lw = nullptr);
// use the tree's near-field kernel blocks in P2P (1) or evaluate the kernel (0); tuning key 2
int p2p_set_near_blocks(int on);
// near-field sums added inside the fused leaf step (1) or by sparse_p2p_scatter (0); tuning key 3 (fmm.cu)
int near_set_fold(int on);
int sparse_p2p_scatter(const hikf_tree* t, const SparseHt& s, const double* Pnear, double* U, int64_t ldu,
                       cudaStream_t st, int64_t r0 = 0, int64_t r1 = -1, const LeafWindow* lw = nullptr);

// leaf multipoles of the active (leaf, ray) pairs (sparse P2M); keys_ready is recorded once the
// keys exist (before the coefficients)
int pairs_leaf(const hikf_tree* t, const SparseHt& s, PairLevel* out, cudaStream_t st,
               cudaEvent_t keys_ready = nullptr);
// The active pairs of level l (keys only) from those of a finer level lc: sort + unique of the
// ancestors' keys.  The levels' key lists do not depend on the multipole values, so they (and
// the M2L targets built from them) can be formed for all levels at once, beside the M2M chain.
// (deferred: no host read-back of the pair count -- out->np is a bound, out->np_dev the count;
//  m2l_targets, m2l_products and pairs_m2m accept such levels)
int pairs_keys(const hikf_tree* t, int l, int lc, const PairLevel& child, int64_t n, PairLevel* out, cudaStream_t st,
               bool deferred = false);
// parent multipoles (sparse M2M) of level l's pairs (keys from pairs_keys) from level l + 1
int pairs_m2m(const hikf_tree* t, int l, const PairLevel& child, int64_t n, PairLevel* out, cudaStream_t st);
void pairs_free(PairLevel* p, cudaStream_t st);
// Compact M2L targets of level l: the (box, ray) pairs that receive at least one
// M2L term (an admissible, occupied T = S - d of an active source pair (S, j),
// inside the box-column range [xlo, xhi]).  tmap (G_l^2 x n int32) maps T * n + j
// to its slot in the compact scratch (q coefficients per slot) or -1; *count_dev
// receives the number of slots.  Replaces a dense G_l^2 x n x q scratch that is
// mostly zeros (cfg4 leaf level: 4.8 GB dense, ~0.3 GB compact).
// The per-offset work lists of the level: ent = (source pair, target slot) of every
// admissible (offset, pair), offset-major; off[d] .. off[d+1] = offset d's entries.
struct M2LPlan {
  int2* ent = nullptr;
  int64_t* off = nullptr;  // 41 (device)
};
// count_dev[0] = target slots, count_dev[1] = entries (2 ints)
int m2l_targets(const hikf_tree* t, int l, const PairLevel& src, int64_t n, int32_t* tmap, int32_t* count_dev,
                M2LPlan* plan, cudaStream_t st, int64_t xlo = 0, int64_t xhi = INT64_MAX);
void m2l_plan_free(M2LPlan* plan, cudaStream_t st);
// every order the tree can select (q <= 256) has a product M2L: instantiated kernels for orders
// 2..8, a generic one above
bool m2l_list_supported(const hikf_tree* t, int l);
// Every M2L term of level l at once: the products M_d W_p of all
// entries in one launch, then S[slot] = the slot's products added in the reference's offset
// order -- the per-offset passes' sums bit for bit, without their 40 dependent launches.
// hoff: host copy of plan.off (41); nslots: target slots; S is written, not accumulated into.
int m2l_products(const hikf_tree* t, int l, const PairLevel& src, const M2LPlan& plan, const int64_t* hoff,
                 int64_t nslots, double* S, cudaStream_t st);
// L[T][a][j] = S[tmap[T n + j]][a] (0 without a slot) for the occupied boxes of level l
int pair_to_box(const hikf_tree* t, int l, const double* S, const int32_t* tmap, int64_t n, double* L,
                cudaStream_t st);

}  // namespace hikf

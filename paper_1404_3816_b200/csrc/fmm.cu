// FmmTree.matmat on the GPU (fmm.py:325-367): near-field P2P, then the
// upward pass (P2M, M2M) and the downward pass (M2L fused with L2L, L2P),
// each stage a seg_gemm_kernel launch over boxes x column tiles.
#include <algorithm>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <utility>
#include <chrono>
#include <string>
#include <vector>

#include "boxgemm.h"
#include "fmm_device.cuh"
#include "prof.h"
#include "sparse.h"
#include "tree.h"

namespace hikf {

namespace {

// Near field (fmm.py:166-201, :330): U rows of target leaf = sum over the
// occupied 3x3-adjacent leaves (ox outer, oy inner) of K(x_t, x_s) V_s.
struct P2PProv : ProvBase {
  static constexpr int kStage = ST_P2P;
  static constexpr bool kAccumulate = false;
  const int32_t *leaf_box, *leaf_start, *leaf_count, *box2leaf;
  const double* xy_s;
  const int64_t* order;
  int64_t G;
  const double* V;
  int64_t ldv;
  double* U;
  int64_t ldu;
  __device__ int rows(int task) const { return leaf_count[task]; }
  __device__ int nsegs(int) const { return 9; }
  __device__ bool seg(int task, int s, Seg& d) const {
    int64_t box = leaf_box[task], bx = box / G, by = box % G;
    int64_t nx = bx + (s / 3 - 1), ny = by + (s % 3 - 1);
    if (nx < 0 || nx >= G || ny < 0 || ny >= G) return false;
    int32_t src = box2leaf[nx * G + ny];
    if (src < 0) return false;
    int32_t s0 = leaf_start[src];
    d.K = leaf_count[src];
    d.gen = true;
    d.a = nullptr;
    d.a_rs = d.a_cs = 0;
    d.txy = xy_s + 2 * (int64_t)leaf_start[task];
    d.sxy = xy_s + 2 * (int64_t)s0;
    d.b = V;
    d.ldb = ldv;
    d.b_rows = order + s0;
    d.bmask = nullptr;
    return true;
  }
  __device__ double* out_row(int task, int r) const { return U + order[leaf_start[task] + r] * ldu; }
};

// P2M (fmm.py:338): W_leaf[a][:] = sum_p W2[p][a] V[p][:]
struct P2MProv : ProvBase {
  static constexpr int kStage = ST_P2M;
  static constexpr int kStages = 2;
  static constexpr int kMinBlocks = 2;
  static constexpr bool kAccumulate = false;
  const int32_t *leaf_box, *leaf_start, *leaf_count;
  const double* W2s;
  int q;
  const int64_t* order;
  const double* V;
  int64_t ldv;
  double* W;  // leaf level, (G^2, q, kcols)
  __device__ int rows(int) const { return q; }
  __device__ int nsegs(int) const { return 1; }
  __device__ bool seg(int task, int, Seg& d) const {
    int32_t s0 = leaf_start[task];
    d.K = leaf_count[task];
    d.gen = false;
    d.a = W2s + (int64_t)s0 * q;  // A[r = a][kk = p] = W2s[(s0 + p) q + a]
    d.a_rs = 1;
    d.a_cs = q;
    d.b = V;
    d.ldb = ldv;
    d.b_rows = order + s0;
    d.bmask = nullptr;
    return true;
  }
  __device__ double* out_row(int task, int r) const { return W + ((int64_t)leaf_box[task] * q + r) * kcols; }
};

// M2M (fmm.py:339-345): W_p[b] = sum_{children c} sum_a C_c[a][b] W_c[a]
struct M2MProv : ProvBase {
  static constexpr int kStage = ST_M2M;
  static constexpr int kStages = 2;
  static constexpr int kMinBlocks = 2;
  static constexpr bool kAccumulate = false;
  const int32_t* occ;            // occupied parents at level l
  const uint8_t* child_flag;     // occupancy at level l+1
  const double* shift;           // 4 x (qc x qp)
  int qp, qc;
  int64_t Gp;
  const double* Wc;              // level l+1
  double* Wp;                    // level l
  const uint8_t* cmask;          // child activity masks (sparse charges) or null
  __device__ int rows(int) const { return qp; }
  __device__ int nsegs(int) const { return 4; }
  __device__ bool seg(int task, int s, Seg& d) const {
    int64_t box = occ[task], X = box / Gp, Y = box % Gp;
    int cx = s >> 1, cy = s & 1;
    int64_t child = (2 * X + cx) * (2 * Gp) + (2 * Y + cy);
    if (!child_flag[child]) return false;
    d.K = qc;
    d.gen = false;
    d.a = shift + (int64_t)s * qc * qp;  // A[r = b][kk = a] = C[a][b]
    d.a_rs = 1;
    d.a_cs = qp;
    d.b = Wc + child * qc * kcols;
    d.ldb = kcols;
    d.b_rows = nullptr;
    d.bmask = cmask ? cmask + child * ngroups : nullptr;
    return true;
  }
  __device__ double* out_row(int task, int r) const { return Wp + ((int64_t)occ[task] * qp + r) * kcols; }
};

// M2L over the interaction list (fmm.py:349-359) with the parent-to-child
// shift (fmm.py:361-363) fused as a 41st segment.
struct M2LProv : ProvBase {
  static constexpr int kStage = ST_M2L;
  static constexpr bool kAccumulate = false;
  const int32_t* occ;         // occupied targets at level l
  const uint8_t* flag;        // occupancy at level l
  const double* ops;          // 40 x q x q
  uint64_t present;
  M2LOffsets offs;
  int q;
  int64_t G;
  const double* W;            // multipoles, level l
  double* L;                  // locals, level l
  const uint8_t* smask;       // source activity masks (sparse charges) or null
  // L2L from the parent level (null at level 2)
  const double* Lp;
  const double* shift;        // shift ops between l-1 and l: 4 x (q x qp)
  int qp;
  __device__ int rows(int) const { return q; }
  __device__ int nsegs(int) const { return Lp ? 41 : 40; }
  __device__ bool seg(int task, int s, Seg& d) const {
    int64_t t = occ[task], tx = t / G, ty = t % G;
    d.gen = false;
    d.b_rows = nullptr;
    d.ldb = kcols;
    d.bmask = nullptr;
    if (s < 40) {
      if (!((present >> s) & 1)) return false;
      int64_t src;
      if (!m2l_source(tx, ty, offs.dx[s], offs.dy[s], G, src)) return false;
      if (!flag[src]) return false;  // empty source: zero multipole
      d.K = q;
      d.a = ops + (int64_t)s * q * q;
      d.a_rs = q;
      d.a_cs = 1;
      d.b = W + src * q * kcols;
      d.bmask = smask ? smask + src * ngroups : nullptr;
      return true;
    }
    int c = (int)((tx & 1) * 2 + (ty & 1));
    int64_t parent = (tx >> 1) * (G >> 1) + (ty >> 1);
    d.K = qp;
    d.a = shift + (int64_t)c * q * qp;  // A[r = a][kk = b] = C[a][b]
    d.a_rs = qp;
    d.a_cs = 1;
    d.b = Lp + parent * qp * kcols;
    return true;
  }
  __device__ double* out_row(int task, int r) const { return L + ((int64_t)occ[task] * q + r) * kcols; }
};

// L2L only (fmm.py:361-363), accumulated after the per-offset sparse M2L passes
struct L2LProv : ProvBase {
  static constexpr int kStage = ST_L2L;
  static constexpr int kStages = 2;
  static constexpr int kMinBlocks = 2;
  static constexpr bool kAccumulate = true;
  const int32_t* occ;
  int q, qp;
  int64_t G;
  const double* Lp;
  const double* shift;  // 4 x (q x qp)
  double* L;
  __device__ int rows(int) const { return q; }
  __device__ int nsegs(int) const { return 1; }
  __device__ bool seg(int task, int, Seg& d) const {
    int64_t t = occ[task], tx = t / G, ty = t % G;
    int c = (int)((tx & 1) * 2 + (ty & 1));
    d.K = qp;
    d.gen = false;
    d.a = shift + (int64_t)c * q * qp;
    d.a_rs = qp;
    d.a_cs = 1;
    d.b = Lp + ((tx >> 1) * (G >> 1) + (ty >> 1)) * qp * kcols;
    d.ldb = kcols;
    d.b_rows = nullptr;
    d.bmask = nullptr;
    return true;
  }
  __device__ double* out_row(int task, int r) const { return L + ((int64_t)occ[task] * q + r) * kcols; }
};

// L2L grouped by parent (fmm.py:361-363): the four children of a parent share
// B = L_parent, A = the four stacked shift operators (4 q x qp); accumulates
// into the children's locals (which already hold the M2L sum).
struct L2LParentProv : ProvBase {
  static constexpr int kStage = ST_L2L;
  static constexpr int kStages = 2;
  static constexpr int kMinBlocks = 2;
  static constexpr bool kAccumulate = true;
  const int32_t* occp;  // occupied parents at level l-1
  int q, qp;
  int64_t Gp;
  const double* Lp;
  const double* shift;  // 4 x (q x qp), stacked
  double* L;
  __device__ int rows(int) const { return 4 * q; }
  __device__ int nsegs(int) const { return 1; }
  __device__ bool seg(int task, int, Seg& d) const {
    d.K = qp;
    d.gen = false;
    d.a = shift;
    d.a_rs = qp;
    d.a_cs = 1;
    d.b = Lp + (int64_t)occp[task] * qp * kcols;
    d.ldb = kcols;
    d.b_rows = nullptr;
    d.bmask = nullptr;
    return true;
  }
  __device__ double* out_row(int task, int r) const {
    int64_t P = occp[task], X = P / Gp, Y = P % Gp;
    int c = r / q;
    int64_t child = (2 * X + (c >> 1)) * (2 * Gp) + (2 * Y + (c & 1));
    return L + (child * q + (r % q)) * kcols;
  }
};

// L2P (fmm.py:366): U[p][:] += sum_a W2[p][a] L_leaf[a][:]  (kAdd = false:
// store, for the sparse path where the near field is added afterwards)
template <bool kAdd>
struct L2PProv : ProvBase {
  static constexpr int kStage = ST_L2P;
  static constexpr int kStages = 2;
  static constexpr int kMinBlocks = 2;
  static constexpr bool kAccumulate = kAdd;
  const int32_t *leaf_box, *leaf_start, *leaf_count;
  const double* W2s;
  int q;
  const int64_t* order;
  const double* L;
  double* U;
  int64_t ldu;
  __device__ int rows(int task) const { return leaf_count[task]; }
  __device__ int nsegs(int) const { return 1; }
  __device__ bool seg(int task, int, Seg& d) const {
    d.K = q;
    d.gen = false;
    d.a = W2s + (int64_t)leaf_start[task] * q;
    d.a_rs = q;
    d.a_cs = 1;
    d.b = L + (int64_t)leaf_box[task] * q * kcols;
    d.ldb = kcols;
    d.b_rows = nullptr;
    d.bmask = nullptr;
    return true;
  }
  __device__ double* out_row(int task, int r) const { return U + order[leaf_start[task] + r] * ldu; }
};

template <class Prov>
int launch(const Prov& p, int64_t tasks, int64_t max_rows, int64_t kcols, cudaStream_t st) {
  if (tasks <= 0 || max_rows <= 0 || kcols <= 0) return HIKF_OK;
  static bool configured = false;
  if (!configured) {
    HIKF_CHECK_CUDA(cudaFuncSetAttribute(seg_gemm_kernel<Prov>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sg_smem<Prov>()));
    configured = true;
  }
  // blockIdx.x = (task * row_tiles + row_tile) * col_tiles + col_tile
  const int64_t rt = ceil_div(max_rows, SG_R), ct = ceil_div(kcols, SG_BN);
  dim3 grid((unsigned)(tasks * rt * ct), 1, 1);
  Prov q = p;
  q.row_tiles = (int)rt;
  if (!q.flops) q.flops = prof_flops_ptr(Prov::kStage);
  seg_gemm_kernel<Prov><<<grid, SG_THREADS, sg_smem<Prov>(), st>>>(q);
  HIKF_CHECK_LAUNCH();
  return HIKF_OK;
}

}  // namespace

namespace {

bool aligned16(const void* p, int64_t ld) { return (((uintptr_t)p & 15) == 0) && (ld % 2 == 0); }

// bytes per column of the expansion workspace: all W levels + two L levels
int64_t expansion_bytes_per_col(const hikf_tree* t) {
  const int D = t->depth;
  if (D < 2) return 0;
  int64_t per_col = 0;
  for (int l = 2; l <= D; ++l) per_col += (int64_t)8 * ((int64_t)1 << (2 * l)) * t->orders[l] * t->orders[l];
  per_col += (int64_t)8 * ((int64_t)1 << (2 * D)) * t->orders[D] * t->orders[D];
  if (D > 2) per_col += (int64_t)8 * ((int64_t)1 << (2 * (D - 1))) * t->orders[D - 1] * t->orders[D - 1];
  return per_col;
}

template <class P>
void set_base(P& p, const hikf_tree* t, int64_t kc, int64_t gofs, int64_t ngroups, bool vecB) {
  p.kcols = kc;
  p.gofs = gofs;
  p.ngroups = ngroups;
  p.vecB = vecB;
  p.kp = t->kp;
}

// M2M, M2L (+L2L) and L2P for one column pass whose leaf multipoles are in
// Wl[D].  masks[l] (sparse charges) lets the DMMA stages skip zero groups.
template <bool kL2PAdd>
int far_field(hikf_tree* t, double* const* Wl, double* const* Lbuf, int64_t kc, int64_t gofs, int64_t ngroups,
              uint8_t* const* masks, double* Uc, int64_t ldu, cudaStream_t st) {
  const int D = t->depth;
  const int qD = t->orders[D] * t->orders[D];
  for (int l = D - 1; l >= 2; --l) {
    M2MProv mm;
    set_base(mm, t, kc, gofs, ngroups, aligned16(Wl[l + 1], kc));
    mm.occ = t->occ[l];
    mm.child_flag = t->occ_flag[l + 1];
    mm.shift = t->shift[l];
    mm.qp = t->orders[l] * t->orders[l];
    mm.qc = t->orders[l + 1] * t->orders[l + 1];
    mm.Gp = (int64_t)1 << l;
    mm.Wc = Wl[l + 1];
    mm.Wp = Wl[l];
    mm.cmask = masks ? masks[l + 1] : nullptr;
    ProfScope ps(ST_M2M, st);
    HIKF_TRY(launch(mm, t->n_occ[l], mm.qp, kc, st));
  }
  const double* Lprev = nullptr;
  double* Lcur = nullptr;
  for (int l = 2; l <= D; ++l) {
    Lcur = Lbuf[(D - l) & 1];
    M2LProv ml;
    set_base(ml, t, kc, gofs, ngroups, aligned16(Wl[l], kc) && aligned16(Lbuf[0], kc) && aligned16(Lbuf[1], kc));
    ml.occ = t->occ[l];
    ml.flag = t->occ_flag[l];
    ml.ops = t->m2l[l];
    ml.present = t->m2l_present[l];
    ml.q = t->orders[l] * t->orders[l];
    ml.G = (int64_t)1 << l;
    ml.W = Wl[l];
    ml.L = Lcur;
    ml.smask = masks ? masks[l] : nullptr;
    ml.Lp = Lprev;
    ml.shift = l > 2 ? t->shift[l - 1] : nullptr;
    ml.qp = l > 2 ? t->orders[l - 1] * t->orders[l - 1] : 0;
    {
      ProfScope ps(ST_M2L, st);
      HIKF_TRY(launch(ml, t->n_occ[l], ml.q, kc, st));
    }
    Lprev = Lcur;
  }
  L2PProv<kL2PAdd> lp;
  set_base(lp, t, kc, gofs, ngroups, aligned16(Lcur, kc));
  lp.leaf_box = t->leaf_box;
  lp.leaf_start = t->leaf_start;
  lp.leaf_count = t->leaf_count;
  lp.W2s = t->W2s;
  lp.q = qD;
  lp.order = t->order;
  lp.L = Lcur;
  lp.U = Uc;
  lp.ldu = ldu;
  ProfScope ps(ST_L2P, st);
  return launch(lp, t->n_leaves, t->max_count, kc, st);
}

void carve(const hikf_tree* t, double* ws, int64_t kc, double** Wl, double** Lbuf) {
  const int D = t->depth;
  double* cur = ws;
  for (int l = 2; l <= D; ++l) {
    Wl[l] = cur;
    cur += ((int64_t)1 << (2 * l)) * t->orders[l] * t->orders[l] * kc;
  }
  Lbuf[0] = cur;  // holds the levels with the parity of D
  cur += ((int64_t)1 << (2 * D)) * t->orders[D] * t->orders[D] * kc;
  Lbuf[1] = cur;
}

}  // namespace

int fmm_matmat(hikf_tree* t, const double* V, int64_t ldv, int64_t k, double* U, int64_t ldu, cudaStream_t st) {
  if (k <= 0) return HIKF_OK;
  const int D = t->depth;
  // column pass width: keep the expansion workspace within ~24 GiB
  const int64_t per_col = expansion_bytes_per_col(t);
  const int64_t budget = (int64_t)24 << 30;
  int64_t kpass = k;
  if (per_col > 0 && per_col * kpass > budget) kpass = std::max<int64_t>(SG_BN, (budget / per_col) / SG_BN * SG_BN);

  double* ws = nullptr;
  if (D >= 2) HIKF_CHECK_CUDA(cudaMallocAsync((void**)&ws, (size_t)per_col * std::min(kpass, k), st));

  for (int64_t c0 = 0; c0 < k; c0 += kpass) {
    const int64_t kc = std::min(kpass, k - c0);
    const double* Vc = V + c0;
    double* Uc = U + c0;
    const bool vecV = aligned16(Vc, ldv);
    // ---- near field: U = near @ V ----
    P2PProv pp;
    set_base(pp, t, kc, 0, 0, vecV);
    pp.leaf_box = t->leaf_box;
    pp.leaf_start = t->leaf_start;
    pp.leaf_count = t->leaf_count;
    pp.box2leaf = t->box2leaf;
    pp.xy_s = t->xy_s;
    pp.order = t->order;
    pp.G = t->G;
    pp.V = Vc;
    pp.ldv = ldv;
    pp.U = Uc;
    pp.ldu = ldu;
    {
      ProfScope ps(ST_P2P, st);
      HIKF_TRY(launch(pp, t->n_leaves, t->max_count, kc, st));
    }
    if (D < 2) continue;
    double* Wl[kMaxDepth + 1] = {nullptr};
    double* Lbuf[2];
    carve(t, ws, kc, Wl, Lbuf);
    // ---- upward pass: P2M ----
    const int qD = t->orders[D] * t->orders[D];
    P2MProv pm;
    set_base(pm, t, kc, 0, 0, vecV);
    pm.leaf_box = t->leaf_box;
    pm.leaf_start = t->leaf_start;
    pm.leaf_count = t->leaf_count;
    pm.W2s = t->W2s;
    pm.q = qD;
    pm.order = t->order;
    pm.V = Vc;
    pm.ldv = ldv;
    pm.W = Wl[D];
    {
      ProfScope ps(ST_P2M, st);
      HIKF_TRY(launch(pm, t->n_leaves, qD, kc, st));
    }
    // ---- M2M, M2L + L2L, L2P: U += interp @ local ----
    HIKF_TRY(far_field<true>(t, Wl, Lbuf, kc, 0, 0, nullptr, Uc, ldu, st));
  }
  if (ws) HIKF_CHECK_CUDA(cudaFreeAsync(ws, st));
  return HIKF_OK;
}

// Side streams for the concurrent parts of the sparse Q H^T: the near field
// (compute-bound P2P) and the per-level M2L chains (latency-bound launches)
// are independent of each other and of the other levels.
namespace {
// s[0]: the near field, at the lowest priority, so that it fills the gaps of the
// latency-bound upward pass; w (the precompute's own main stream) and s[1..7] (the
// M2L level groups) at the highest priority: they carry the critical path
struct QhtStreams {
  cudaStream_t s[8] = {};
  cudaStream_t w = nullptr;
  cudaEvent_t e[kMaxDepth + 4] = {};
  cudaEvent_t e_keys[kMaxDepth + 1] = {}, e_pairs[kMaxDepth + 1] = {}, e_tgt[kMaxDepth + 1] = {};  // level's pair keys / multipoles / M2L targets ready
  cudaEvent_t e_in = nullptr, e_out = nullptr;
  cudaEvent_t e_join[8] = {};           // side streams joined into w before the workspace is freed
  int32_t* hcount = nullptr;            // pinned: M2L slot / entry counts per level
  int64_t (*hoff)[41] = nullptr;        // pinned: first entry of every offset per level
};
int qht_streams(QhtStreams** out) {
  static QhtStreams p;
  static bool init = false;
  if (!init) {
    int lo = 0, hi = 0;
    HIKF_CHECK_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    for (int i = 0; i < 8; ++i)
      HIKF_CHECK_CUDA(cudaStreamCreateWithPriority(&p.s[i], cudaStreamNonBlocking, i == 0 ? lo : hi));
    HIKF_CHECK_CUDA(cudaStreamCreateWithPriority(&p.w, cudaStreamNonBlocking, hi));
    for (auto& x : p.e) HIKF_CHECK_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    for (auto& x : p.e_pairs) HIKF_CHECK_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    for (auto& x : p.e_keys) HIKF_CHECK_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    for (auto& x : p.e_join) HIKF_CHECK_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    for (auto& x : p.e_tgt) HIKF_CHECK_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    HIKF_CHECK_CUDA(cudaMallocHost((void**)&p.hcount, sizeof(int32_t) * 2 * (kMaxDepth + 1)));
    HIKF_CHECK_CUDA(cudaMallocHost((void**)&p.hoff, sizeof(int64_t) * 41 * (kMaxDepth + 1)));
    HIKF_CHECK_CUDA(cudaEventCreateWithFlags(&p.e_in, cudaEventDisableTiming));
    HIKF_CHECK_CUDA(cudaEventCreateWithFlags(&p.e_out, cudaEventDisableTiming));
    init = true;
  }
  *out = &p;
  return HIKF_OK;
}
}  // namespace

int leaf_window(const hikf_tree* t, int64_t leaf0, int64_t leaf1, LeafWindow* w) {
  if (leaf0 < 0 || leaf1 < leaf0 || leaf1 > t->n_leaves) {
    set_error("leaf range [%lld, %lld) outside [0, %lld]", (long long)leaf0, (long long)leaf1, (long long)t->n_leaves);
    return HIKF_BAD_ARGUMENT;
  }
  const int64_t G = (int64_t)1 << t->depth;
  w->leaf0 = leaf0;
  w->leaf1 = leaf1;
  w->s0 = leaf0 < t->n_leaves ? t->h_leaf_start[leaf0] : t->m;
  w->s1 = leaf1 > leaf0 ? t->h_leaf_start[leaf1 - 1] + t->h_leaf_count[leaf1 - 1] : w->s0;
  w->x0 = leaf1 > leaf0 ? t->h_leaf_box[leaf0] / G : 0;
  w->x1 = leaf1 > leaf0 ? t->h_leaf_box[leaf1 - 1] / G : -1;
  return HIKF_OK;
}

// HIKF_QHT_TIMELINE=1: event timestamps of the Q H^T stages (ms from the start) to stderr
namespace {
struct Timeline {
  bool on = false;
  std::vector<std::pair<const char*, cudaEvent_t>> ev;
  cudaEvent_t t0 = nullptr;
  void start(cudaStream_t s) {
    static const bool env = getenv("HIKF_QHT_TIMELINE") != nullptr;
    on = env;
    if (!on) return;
    cudaEventCreate(&t0);
    cudaEventRecord(t0, s);
    h0 = std::chrono::steady_clock::now();
  }
  std::vector<std::pair<std::string, double>> hv;  // host-side enqueue times
  std::chrono::steady_clock::time_point h0;
  void mark(const char* name, cudaStream_t s, int level = -1) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    static char names[64][48];
    static int nn = 0;
    char* nm = names[nn++ % 64];
    if (level >= 0) snprintf(nm, 48, "%s %d", name, level); else snprintf(nm, 48, "%s", name);
    ev.emplace_back(nm, e);
    hv.emplace_back(nm, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count());
  }
  void report() {
    if (!on) return;
    cudaDeviceSynchronize();
    for (size_t i = 0; i < ev.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, t0, ev[i].second);
      fprintf(stderr, "qht %-22s %8.3f ms   (enqueued by the host at %8.3f ms)\n", ev[i].first, ms, hv[i].second);
      cudaEventDestroy(ev[i].second);
    }
    cudaEventDestroy(t0);
  }
};
}  // namespace

// the near-field sums are added inside the fused leaf step (1, default) or by the separate
// scatter pass (0: HIKF_NEAR_FOLD=0 or tuning key 3) -- the same single add either way
static int g_near_fold = -1;
static bool near_fold_enabled() {
  if (g_near_fold < 0) {
    const char* e = getenv("HIKF_NEAR_FOLD");
    g_near_fold = (e && e[0] == '0') ? 0 : 1;
  }
  return g_near_fold != 0;
}
int near_set_fold(int on) {
  const int prev = near_fold_enabled() ? 1 : 0;
  g_near_fold = on ? 1 : 0;
  return prev;
}

int fmm_matmat_csrT(hikf_tree* t, int64_t n, const int32_t* ip, const int32_t* ix, const double* val, double* U,
                    cudaStream_t st, int64_t r0, int64_t r1, const LeafWindow* lw) {
  Timeline tl;
  tl.start(st);
  if (n <= 0) return HIKF_OK;
  const bool window = r0 != 0 || (r1 >= 0 && r1 != t->m);
  if (r1 < 0) r1 = t->m;
  if (lw) {
    r0 = 0;
    r1 = lw->s1 - lw->s0;
    if (lw->leaf1 <= lw->leaf0) return HIKF_OK;
  }
  const int D = t->depth;
  // box-column range of level l that holds ancestors of the shard's leaves
  auto xlo = [&](int l) { return lw ? (lw->x0 >> (D - l)) : (int64_t)0; };
  auto xhi = [&](int l) { return lw ? (lw->x1 >> (D - l)) : INT64_MAX; };
  QhtStreams* qs = nullptr;
  HIKF_TRY(qht_streams(&qs));
  // the precompute runs on its own high-priority stream qs->w, forked from and
  // joined back into the caller's stream
  struct Join {
    QhtStreams* qs;
    cudaStream_t caller;
    ~Join() {
      cudaEventRecord(qs->e_out, qs->w);
      cudaStreamWaitEvent(caller, qs->e_out, 0);
    }
  };
  HIKF_CHECK_CUDA(cudaEventRecord(qs->e_in, st));
  HIKF_CHECK_CUDA(cudaStreamWaitEvent(qs->w, qs->e_in, 0));
  Join join{qs, st};
  st = qs->w;
  SparseHt sp;
  // the call's workspace; freed (after every side stream has been joined into the main stream)
  // when the function leaves, on the error paths too
  PairLevel pl[kMaxDepth + 1];
  double* scratch[kMaxDepth + 1] = {};
  int32_t* tmap[kMaxDepth + 1] = {};
  int32_t* tcount = nullptr;
  M2LPlan plan[kMaxDepth + 1];
  double* Lbuf[2] = {nullptr, nullptr};
  double* Pnear = nullptr;
  struct Workspace {
    QhtStreams* qs;
    SparseHt& sp;
    PairLevel* pl;
    double** scratch;
    int32_t** tmap;
    int32_t*& tcount;
    M2LPlan* plan;
    double** Lbuf;
    double*& Pnear;
    ~Workspace() {
      cudaStream_t w = qs->w;
      for (int i = 0; i < 8; ++i) {
        cudaEventRecord(qs->e_join[i], qs->s[i]);
        cudaStreamWaitEvent(w, qs->e_join[i], 0);
      }
      for (int l = 0; l <= kMaxDepth; ++l) {
        pairs_free(&pl[l], w);
        if (scratch[l]) cudaFreeAsync(scratch[l], w);
        if (tmap[l]) cudaFreeAsync(tmap[l], w);
        m2l_plan_free(&plan[l], w);
      }
      if (tcount) cudaFreeAsync(tcount, w);
      if (Lbuf[0]) cudaFreeAsync(Lbuf[0], w);
      if (Lbuf[1]) cudaFreeAsync(Lbuf[1], w);
      if (Pnear) cudaFreeAsync(Pnear, w);
      sparse_free(&sp, w);
    }
  } workspace{qs, sp, pl, scratch, tmap, tcount, plan, Lbuf, Pnear};
  {
    ProfScope ps(ST_DENSIFY, st);  // the regrouping of H^T replaces the densify step
    HIKF_TRY(sparse_build(t, n, ip, ix, val, &sp, st));
  }
  tl.mark("regroup", st);
  if (D < 2) {
    HIKF_CHECK_CUDA(cudaMemsetAsync(U, 0, sizeof(double) * (r1 - r0) * n, st));
    int status;
    {
      ProfScope ps(ST_P2P, st);
      status = sparse_p2p(t, sp, U, n, st, nullptr, r0, r1, lw);
    }
    return status;
  }
  cudaEvent_t ev_base = qs->e[0], ev_p2p = qs->e[1];

  // ---- near field, concurrently: sums parked in Pnear, added after L2P.  Launched
  // first, on the lowest-priority stream: it fills the machine while the upward pass
  // and the M2L target maps (latency-bound, on the critical path) run ahead of it ----
  HIKF_CHECK_CUDA(cudaMallocAsync((void**)&Pnear, sizeof(double) * std::max<int64_t>(1, sp.nitems * t->max_count), st));
  int status = HIKF_OK;
  auto launch_p2p = [&]() -> int {
    HIKF_CHECK_CUDA(cudaEventRecord(ev_base, st));
    HIKF_CHECK_CUDA(cudaStreamWaitEvent(qs->s[0], ev_base, 0));
    int s2;
    {
      ProfScope ps(ST_P2P, qs->s[0]);
      s2 = sparse_p2p(t, sp, U, n, qs->s[0], Pnear, 0, -1, lw);
    }
    HIKF_CHECK_CUDA(cudaEventRecord(ev_p2p, qs->s[0]));
    tl.mark("p2p end", qs->s[0]);
    return s2;
  };
  status = launch_p2p();

  // ---- upward pass on the active (box, ray) pairs only (main stream), and beside it,
  // per level, the M2L targets: a (box, ray) -> slot map and the per-offset entry lists,
  // built on the level group's stream as soon as the level's pairs exist.  A group's 40
  // M2L passes are enqueued one upward step later (its slot / entry counts have arrived in
  // pinned memory by then), so the leaf level's M2L runs beside the M2M chain instead of
  // after it ----
  int32_t* hcount = qs->hcount;          // [2 l]: target slots, [2 l + 1]: entries of level l
  int64_t (*hoff)[41] = qs->hoff;        // first entry of every offset of level l
  // fused leaf step (leaf_down): the leaf-level locals are never stored
  const bool fused_leaf = leaf_fused_enabled() && leaf_down_supported(t);
  int64_t lsz[2] = {1, 1};  // ping-pong local buffers: level l lives in Lbuf[(D - l) & 1]
  for (int l = 2; l <= D - (fused_leaf ? 1 : 0); ++l)
    lsz[(D - l) & 1] = std::max(lsz[(D - l) & 1], ((int64_t)1 << (2 * l)) * t->orders[l] * t->orders[l] * n);
  int groups[kMaxDepth + 1][kMaxDepth + 1], gsize[kMaxDepth + 1] = {0}, ng = 0, glevel[kMaxDepth + 1] = {0};
  for (int l = D; l >= 2; --l) {  // one group (stream) per level: the levels' M2L sums are independent
    groups[ng][gsize[ng]++] = l;
    glevel[l] = ng++;
  }
  auto gstream = [&](int gi) { return qs->s[1 + gi % 7]; };
  if (status == HIKF_OK) {
    HIKF_CHECK_CUDA(cudaMallocAsync((void**)&Lbuf[0], sizeof(double) * lsz[0], st));
    HIKF_CHECK_CUDA(cudaMallocAsync((void**)&Lbuf[1], sizeof(double) * lsz[1], st));
    HIKF_CHECK_CUDA(cudaMallocAsync((void**)&tcount, sizeof(int32_t) * 2 * (kMaxDepth + 1), st));
    for (int l = 2; l <= D; ++l)
      HIKF_CHECK_CUDA(cudaMallocAsync((void**)&tmap[l], sizeof(int32_t) * ((int64_t)1 << (2 * l)) * n, st));
  }
  // deferred pair counts (no host read-back inside the upward pass) when every level has the
  // entry-list M2L; everything is enqueued before the host waits for a count
  bool deferred = true;
  for (int l = 2; l <= D; ++l) deferred = deferred && m2l_list_supported(t, l);
  // level l's pair keys (from the leaf level's: they do not depend on the multipole values)
  // and its M2L targets, on the level's stream
  auto enqueue_targets = [&](int l) -> int {
    cudaStream_t sl = gstream(glevel[l]);
    HIKF_CHECK_CUDA(cudaStreamWaitEvent(sl, qs->e_keys[D], 0));
    if (l < D) {
      ProfScope ps(ST_M2M, sl);
      HIKF_TRY(pairs_keys(t, l, D, pl[D], n, &pl[l], sl, deferred));
      HIKF_CHECK_CUDA(cudaEventRecord(qs->e_keys[l], sl));
    }
    ProfScope ps(ST_M2L, sl);
    HIKF_TRY(m2l_targets(t, l, pl[l], n, tmap[l], tcount + 2 * l, &plan[l], sl, xlo(l), xhi(l)));
    HIKF_CHECK_CUDA(cudaMemcpyAsync(hcount + 2 * l, tcount + 2 * l, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, sl));
    HIKF_CHECK_CUDA(cudaMemcpyAsync(hoff[l], plan[l].off, 41 * sizeof(int64_t), cudaMemcpyDeviceToHost, sl));
    HIKF_CHECK_CUDA(cudaEventRecord(qs->e_tgt[l], sl));
    tl.mark("targets", sl, l);
    return HIKF_OK;
  };
  // the M2L sums of a group whose targets have all been enqueued: every term of the level in
  // one launch plus the ordered per-target sums (m2l_products)
  auto launch_group = [&](int gi) -> int {
    cudaStream_t sl = gstream(gi);
    const int l0 = groups[gi][0];
    const bool lists = m2l_list_supported(t, l0);
    for (int k = 0; k < gsize[gi]; ++k) {
      const int l = groups[gi][k];
      HIKF_CHECK_CUDA(cudaEventSynchronize(qs->e_tgt[l]));
      HIKF_CHECK_CUDA(cudaStreamWaitEvent(sl, qs->e_pairs[l], 0));  // the level's multipoles
      const int64_t words = (int64_t)hcount[2 * l] * t->orders[l] * t->orders[l];
      HIKF_CHECK_CUDA(cudaMallocAsync((void**)&scratch[l], sizeof(double) * std::max<int64_t>(1, words), sl));
      if (!lists) HIKF_CHECK_CUDA(cudaMemsetAsync(scratch[l], 0, sizeof(double) * words, sl));
    }
    ProfScope ps(ST_M2L, sl);
    int s2 = HIKF_OK;
    if (lists) {
      for (int k = 0; k < gsize[gi] && s2 == HIKF_OK; ++k) {
        const int l = groups[gi][k];
        s2 = m2l_products(t, l, pl[l], plan[l], hoff[l], hcount[2 * l], scratch[l], sl);
      }
    } else {
      set_error("M2L: order %d of level %d has no product kernel", t->orders[l0], l0);
      s2 = HIKF_BAD_ARGUMENT;
    }
    for (int k = 0; k < gsize[gi]; ++k) HIKF_CHECK_CUDA(cudaEventRecord(qs->e[3 + groups[gi][k]], sl));
    tl.mark("m2l sums", sl, l0);
    return s2;
  };
  {
    ProfScope ps(ST_P2M, st);
    if (status == HIKF_OK) status = pairs_leaf(t, sp, &pl[D], st, qs->e_keys[D]);
    if (status == HIKF_OK) HIKF_CHECK_CUDA(cudaEventRecord(qs->e_pairs[D], st));
  }
  tl.mark("pairs", st, D);
  for (int l = D; l >= 2 && status == HIKF_OK; --l) status = enqueue_targets(l);
  for (int l = D - 1; l >= 2 && status == HIKF_OK; --l) {  // the M2M chain (main stream)
    ProfScope ps(ST_M2M, st);
    HIKF_CHECK_CUDA(cudaStreamWaitEvent(st, qs->e_keys[l], 0));
    status = pairs_m2m(t, l, pl[l + 1], n, &pl[l], st);
    if (status == HIKF_OK) HIKF_CHECK_CUDA(cudaEventRecord(qs->e_pairs[l], st));
    tl.mark("pairs", st, l);
  }
  for (int gi = 0; gi < ng && status == HIKF_OK; ++gi) status = launch_group(gi);
  // ---- downward pass (main stream): L = scratch^T + shift L_parent, then L2P ----
  const bool vec = (n % 2) == 0;
  const double* Lprev = nullptr;
  double* Lcur = nullptr;
  cudaStream_t dn = st;  // the L2L chain (main stream)
  for (int l = 2; l <= D && status == HIKF_OK; ++l) {
    if (l == D && fused_leaf) {  // the leaf L2L runs inside the fused L2P below
      HIKF_CHECK_CUDA(cudaStreamWaitEvent(st, qs->e[3 + l], 0));
      break;
    }
    Lcur = Lbuf[(D - l) & 1];
    const int q = t->orders[l] * t->orders[l];
    HIKF_CHECK_CUDA(cudaStreamWaitEvent(dn, qs->e[3 + l], 0));
    if (l > 2 && box_supported(4 * q, t->orders[l - 1] * t->orders[l - 1])) {
      ProfScope ps(ST_L2L, dn);
      status = l2l_boxes(t, l, scratch[l], tmap[l], Lprev, n, Lcur, dn, xlo(l - 1), xhi(l - 1));
    } else {
      ProfScope ps(ST_L2L, dn);
      status = pair_to_box(t, l, scratch[l], tmap[l], n, Lcur, dn);
      if (status == HIKF_OK && l > 2) {
        L2LParentProv ll;
        set_base(ll, t, n, 0, 0, vec);
        ll.occp = t->occ[l - 1];
        ll.q = q;
        ll.qp = t->orders[l - 1] * t->orders[l - 1];
        ll.Gp = (int64_t)1 << (l - 1);
        ll.Lp = Lprev;
        ll.shift = t->shift[l - 1];
        ll.L = Lcur;
        status = launch(ll, t->n_occ[l - 1], 4 * q, n, dn);
      }
    }
    Lprev = Lcur;
    tl.mark("l2l", dn, l);
  }
  // the fused leaf step also adds the near-field sums (it waits for P2P; no scatter pass then)
  const bool near_in_leaf = fused_leaf && leaf_down_adds_near(n) && near_fold_enabled();
  if (status == HIKF_OK && fused_leaf) {
    if (near_in_leaf) HIKF_CHECK_CUDA(cudaStreamWaitEvent(st, ev_p2p, 0));
    ProfScope ps(ST_L2P, st);
    status = leaf_down(t, scratch[D], tmap[D], Lprev, n, U, n, st, r0, r1, lw, near_in_leaf ? Pnear : nullptr,
                       sp.items, sp.item_start);
  } else if (status == HIKF_OK && box_supported(64, t->orders[D] * t->orders[D])) {
    ProfScope ps(ST_L2P, st);
    status = l2p_boxes(t, Lcur, n, U, n, st, r0, r1, lw);
  } else if (status == HIKF_OK && lw) {
    set_error("a leaf-aligned Q H^T shard needs the box-streaming L2P (leaf order <= 8)");
    status = HIKF_BAD_ARGUMENT;
  } else if (status == HIKF_OK && window) {
    set_error("row-windowed Q H^T needs the box-streaming L2P (leaf order <= 8)");
    status = HIKF_BAD_ARGUMENT;
  } else if (status == HIKF_OK) {
    L2PProv<false> lp;
    set_base(lp, t, n, 0, 0, vec);
    lp.leaf_box = t->leaf_box;
    lp.leaf_start = t->leaf_start;
    lp.leaf_count = t->leaf_count;
    lp.W2s = t->W2s;
    lp.q = t->orders[D] * t->orders[D];
    lp.order = t->order;
    lp.L = Lcur;
    lp.U = U;
    lp.ldu = n;
    ProfScope ps(ST_L2P, st);
    status = launch(lp, t->n_leaves, t->max_count, n, st);
  }
  tl.mark("leaf step", st);
  // ---- join: every side stream's work is ordered before the frees below ----
  for (int l = 2; l <= D; ++l) HIKF_CHECK_CUDA(cudaStreamWaitEvent(st, qs->e[3 + l], 0));
  HIKF_CHECK_CUDA(cudaStreamWaitEvent(st, ev_p2p, 0));
  if (status == HIKF_OK && !near_in_leaf) {
    ProfScope ps(ST_P2P, st);
    status = sparse_p2p_scatter(t, sp, Pnear, U, n, st, r0, r1, lw);
  }
  tl.mark("leaf + scatter end", st);
  tl.report();
  return status;
}

}  // namespace hikf

// Device building blocks of the FMM stages.
//
// Every stage of FmmTree.matmat (fmm.py:325-367) is one "segmented GEMM":
// an output block O (rows x k) of one box/leaf is a sum over a short list of
// segments, each a small dense product A_s (rows x K_s) * B_s (K_s x k):
//   P2P  : rows = target-leaf points, segments = the <= 9 adjacent leaves,
//          A = K(x_t, x_s) generated on the fly, B = V rows of the source leaf
//   P2M  : rows = q_leaf, one segment, A = W2^T of the leaf, B = V rows
//   M2M  : rows = q_l, segments = 4 children, A = shift^T, B = child W
//   M2L  : rows = q_l, segments = <= 27 interaction-list sources (+ the
//          parent's local for L2L), A = M2L op / shift op, B = source W / L
//   L2P  : rows = leaf points, one segment, A = W2 rows, B = leaf local
// seg_gemm_kernel streams (A, B) K-chunks through a 4-stage cp.async ring in
// shared memory and accumulates with FP64 DMMA (mma.sync m8n8k4) into
// registers; CTA tile = 64 rows x 128 columns, 8 warps, each warp owns 16
// columns x all 8 row tiles.
//
// Sparse charges (V = H^T): a segment may carry an activity mask (one byte
// per 8-column group of its B block).  Inactive groups are exact zeros, so
// their loads and DMMAs are skipped -- the sums are the same numbers (a skipped
// product is +-0), only the work shrinks.
#pragma once

#include "common.cuh"

namespace hikf {

constexpr int kMaxLeafOrder = 12;  // n_cheb <= 12 (fmm.py:51)

// M2L source of target (tx, ty) at offset (dx, dy): in range and parents
// adjacent per dimension (fmm.py:301-302).  Source flat index x-major.
__device__ __forceinline__ bool m2l_source(int64_t tx, int64_t ty, int dx, int dy, int64_t G, int64_t& s) {
  int64_t sx = tx + dx, sy = ty + dy;
  if (sx < 0 || sx >= G || sy < 0 || sy >= G) return false;
  int64_t px = (sx >> 1) - (tx >> 1), py = (sy >> 1) - (ty >> 1);
  if (px < -1 || px > 1 || py < -1 || py > 1) return false;
  s = sx * G + sy;
  return true;
}

constexpr int SG_R = 64;
constexpr int SG_BN = 128;
constexpr int SG_KC = 32;
constexpr int SG_STAGES = 4;
constexpr int SG_THREADS = 256;
constexpr int SG_AS = SG_KC + 4;  // smem row strides (doubles), == 4 mod 16: conflict-free DMMA fragments
constexpr int SG_BS = SG_BN + 4;
constexpr int SG_STAGE_DOUBLES = SG_R * SG_AS + SG_KC * SG_BS;
constexpr size_t SG_SMEM = (size_t)SG_STAGES * SG_STAGE_DOUBLES * sizeof(double) + 64;
// shared memory of a provider's pipeline depth
template <class Prov>
constexpr size_t sg_smem() { return (size_t)Prov::kStages * SG_STAGE_DOUBLES * sizeof(double) + 64; }

// One segment of an output block.
struct Seg {
  int K;                      // inner length; <= 0 means "skip"
  bool gen;                   // A generated from coordinates (P2P)
  const double* a;            // A[r][kk] = a[r * a_rs + kk * a_cs]
  int64_t a_rs, a_cs;
  const double* txy;          // gen: target coords (row r at txy + 2 r), source coords sxy + 2 kk
  const double* sxy;
  const double* b;            // B[kk][c] = b[(b_rows ? b_rows[kk] : kk) * ldb + c]
  int64_t ldb;
  const int64_t* b_rows;
  const uint8_t* bmask;       // per 8-column group activity of B (absolute groups), null = dense
};

// Base of every provider: columns of this pass and the kernel parameters.
struct ProvBase {
  static constexpr int kStages = SG_STAGES;  // cp.async ring depth (long K: interaction lists)
  static constexpr int kMinBlocks = 1;       // CTAs per SM the register budget must allow
  unsigned long long* flops = nullptr;       // useful-flop counter (profiling) or null
  int64_t kcols = 0;   // columns of this pass
  int64_t gofs = 0;    // absolute 8-column group of column 0 of the pass (masks)
  int64_t ngroups = 0; // groups per mask row
  bool vecB = false;   // B rows 16-byte aligned with an even leading dimension
  int row_tiles = 1;   // 64-row tiles per task (set by the launcher)
  KParams kp;
  __device__ int64_t ncols() const { return kcols; }
  __device__ double kernel(double r) const { return kernel_of_r(kp, r); }
};

template <class Prov>
__global__ void __launch_bounds__(SG_THREADS, Prov::kMinBlocks) seg_gemm_kernel(Prov prov) {
  constexpr int STAGES = Prov::kStages;
  extern __shared__ double smem_raw[];
  double* smem = smem_raw;
  __shared__ int stage_k[STAGES];
  __shared__ unsigned stage_am[STAGES];
  unsigned long long useful = 0;  // thread 0: 2 * rows * k * active columns

  // flattened grid, column tiles fastest: consecutive CTAs share the task's A
  // block (W2 rows, M2L operators) in L2
  const int64_t ncols = prov.ncols();
  const int nct = (int)((ncols + SG_BN - 1) / SG_BN);
  const int64_t bid = blockIdx.x;
  const int col0 = (int)(bid % nct) * SG_BN;
  const int64_t rest = bid / nct;
  const int task = (int)(rest / prov.row_tiles);
  const int row0 = (int)(rest % prov.row_tiles) * SG_R;
  const int nrows = prov.rows(task);
  if (row0 >= nrows) return;
  const int nsegs = prov.nsegs(task);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int rows_here = min(SG_R, nrows - row0);
  const int nrt = (rows_here + 7) >> 3;  // active 8-row tiles
  const int arows = nrt * 8;
  // groups of this column tile that exist at all
  const int ncol_here = (int)(ncols - col0 < SG_BN ? ncols - col0 : SG_BN);
  const unsigned all_groups = ncol_here >= SG_BN ? 0xffffu : ((1u << ((ncol_here + 7) >> 3)) - 1u);
  const int64_t g0 = prov.gofs + col0 / 8;

  auto activity = [&](const Seg& s) -> unsigned {
    if (!s.bmask) return all_groups;
    unsigned am = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q)
      if (g0 + q < prov.ngroups && s.bmask[g0 + q]) am |= 1u << q;
    return am & all_groups;
  };

  // producer cursor
  int cur_seg = 0, cur_k = 0;
  unsigned cur_am = 0;
  Seg sd;
  sd.K = 0;
  auto next_valid = [&](int s) {
    while (s < nsegs) {
      if (prov.seg(task, s, sd) && sd.K > 0) {
        cur_am = activity(sd);
        if (cur_am) return s;
      }
      ++s;
    }
    return s;
  };
  cur_seg = next_valid(0);

  auto issue = [&](int stage) {
    double* As = smem + stage * SG_STAGE_DOUBLES;
    double* Bs = As + SG_R * SG_AS;
    if (cur_seg >= nsegs) {
      if (tid == 0) stage_k[stage] = 0;
      return;
    }
    const int kc = min(SG_KC, sd.K - cur_k);
    const int kc4 = (kc + 3) & ~3;  // zero-fill up to the DMMA k granularity
    // A tile: arows x kc4 (rows beyond rows_here only feed unstored accumulators)
    for (int e = tid; e < arows * SG_KC; e += SG_THREADS) {
      int r = e / SG_KC, kk = e % SG_KC;
      if (kk >= kc4) continue;
      bool ok = r < rows_here && kk < kc;
      double* dst = As + r * SG_AS + kk;
      if (sd.gen) {
        double v = 0.0;
        if (ok) {
          const double* tp = sd.txy + 2 * (int64_t)(row0 + r);
          const double* sp = sd.sxy + 2 * (int64_t)(cur_k + kk);
          v = prov.kernel(dist2d(tp[0], tp[1], sp[0], sp[1]));
        }
        *dst = v;
      } else {
        const double* src = ok ? sd.a + (int64_t)(row0 + r) * sd.a_rs + (int64_t)(cur_k + kk) * sd.a_cs : sd.a;
        cp_async8(dst, src, ok);
      }
    }
    // B tile: kc4 x SG_BN, only the active 8-column groups
    if (prov.vecB) {
      for (int e = tid; e < SG_KC * (SG_BN / 2); e += SG_THREADS) {
        int kk = e / (SG_BN / 2), c = (e % (SG_BN / 2)) * 2;
        if (kk >= kc4 || !((cur_am >> (c >> 3)) & 1)) continue;
        int bytes = 0;
        const double* src = sd.b;
        if (kk < kc && col0 + c < ncols) {
          int64_t row = sd.b_rows ? sd.b_rows[cur_k + kk] : (int64_t)(cur_k + kk);
          src = sd.b + row * sd.ldb + col0 + c;
          bytes = col0 + c + 1 < ncols ? 16 : 8;
        }
        cp_async16(Bs + kk * SG_BS + c, src, bytes);
      }
    } else {
      for (int e = tid; e < SG_KC * SG_BN; e += SG_THREADS) {
        int kk = e / SG_BN, c = e % SG_BN;
        if (kk >= kc4 || !((cur_am >> (c >> 3)) & 1)) continue;
        bool ok = kk < kc && col0 + c < ncols;
        const double* src = sd.b;
        if (ok) {
          int64_t row = sd.b_rows ? sd.b_rows[cur_k + kk] : (int64_t)(cur_k + kk);
          src = sd.b + row * sd.ldb + col0 + c;
        }
        cp_async8(Bs + kk * SG_BS + c, src, ok);
      }
    }
    if (tid == 0) {
      stage_k[stage] = kc;
      stage_am[stage] = cur_am;
      useful += 2ull * rows_here * kc * (8ull * __popc(cur_am));
    }
    // advance the cursor
    cur_k += SG_KC;
    if (cur_k >= sd.K) {
      cur_k = 0;
      cur_seg = next_valid(cur_seg + 1);
    }
  };

  double acc[8][2][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    issue(s);
    cp_async_commit();
  }
  for (int it = 0;; ++it) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int stage = it % STAGES;
    const int kc = stage_k[stage];
    if (kc == 0) break;
    const unsigned am = stage_am[stage];
    // refill the slot consumed in the previous iteration
    issue((it + STAGES - 1) % STAGES);
    cp_async_commit();

    const bool on0 = (am >> (2 * warp)) & 1, on1 = (am >> (2 * warp + 1)) & 1;
    if (!(on0 || on1)) continue;
    const double* As = smem + stage * SG_STAGE_DOUBLES;
    const double* Bs = As + SG_R * SG_AS;
    const int nk4 = (kc + 3) >> 2;
    for (int k4 = 0; k4 < nk4; ++k4) {
      const int kb = k4 * 4;
      double bf0 = Bs[(kb + t4) * SG_BS + warp * 16 + g];
      double bf1 = Bs[(kb + t4) * SG_BS + warp * 16 + 8 + g];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (i < nrt) {
          double af = As[(i * 8 + g) * SG_AS + kb + t4];
          if (on0) dmma884(acc[i][0][0], acc[i][0][1], af, bf0);
          if (on1) dmma884(acc[i][1][0], acc[i][1][1], af, bf1);
        }
      }
    }
  }
  cp_async_wait<0>();
  if (prov.flops && tid == 0 && useful) atomicAdd(prov.flops, useful);

  // epilogue: store or accumulate into the output rows (accumulate: all the
  // reads first, so they overlap instead of serialising behind the stores)
  double* orows[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = i * 8 + g;
    orows[i] = (i < nrt && r < rows_here) ? prov.out_row(task, row0 + r) : nullptr;
  }
  if (Prov::kAccumulate) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (!orows[i]) continue;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int64_t c = col0 + warp * 16 + j * 8 + 2 * t4;
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (c + h < ncols) acc[i][j][h] += orows[i][c + h];
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (!orows[i]) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int64_t c = col0 + warp * 16 + j * 8 + 2 * t4;
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (c + h < ncols) orows[i][c + h] = acc[i][j][h];
    }
  }
}

}  // namespace hikf

/*
 * hikf_b200.h -- C ABI of the B200-native HiKF hot path (libhikf_b200.so).
 *
 * The reference (`hikf`, pure Python; /root/reference/pkg/src/hikf) has no FFI:
 * its boundary is the Python function surface re-exported from
 * hikf/__init__.py:10-26.  Each entry point below replaces one reference
 * function (cited file:line); the Python mirror in paper_1404_3816_b200/
 * binds them with ctypes.
 *
 * Conventions
 *   - Plain pointers and sizes only.  "dev" pointers are CUDA device memory
 *     (any allocator), "host" pointers are CPU memory.  Dense matrices are
 *     row-major float64 with an explicit leading dimension, exactly the
 *     C-order numpy layout the reference uses (state (m, n), V (m, k)).
 *   - Sparse H is CSR (n_rows x m): int32 indptr[n+1], int32 indices[nnz],
 *     float64 data[nnz] -- scipy's canonical csr_matrix arrays.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *     stream-ordered; the ones that must report a numerical status
 *     synchronise the stream before returning (as the reference raises
 *     synchronously).
 *   - Every function returns an hikf_status; hikf_last_error() gives the
 *     message of the most recent failure on the calling thread.
 *   - Calls on distinct handles are re-entrant; a single tree handle may be
 *     used for concurrent read-only matmat calls on distinct streams only if
 *     each call passes its own workspace (matmat allocates its own).
 */
#ifndef HIKF_B200_H
#define HIKF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HIKF_OK = 0,
  HIKF_BAD_ARGUMENT = 1,      /* -> ValueError (fmm.py:50-54, :328-329; filters.py:31-37) */
  HIKF_NOT_PD = 2,            /* -> DecompositionError (linalg.py:33-36) */
  HIKF_NEGATIVE_VARIANCE = 3, /* -> NumericalConsistencyError (filters.py:149-153) */
  HIKF_CUDA_ERROR = 4,
  HIKF_ASYMMETRIC = 5,        /* -> ValueError("A is not symmetric") (linalg.py:30-32) */
  HIKF_NO_DEVICE = 6
} hikf_status;

/* Kernel family codes (kernels.py:22 _FAMILIES). */
enum { HIKF_GAUSSIAN = 0, HIKF_EXPONENTIAL = 1, HIKF_LOGARITHM = 2 };

/* KernelSpec (kernels.py:25-69).  `power` is the effective power
 * (2 gaussian / 1 exponential unless overridden); ignored for logarithm. */
typedef struct {
  int32_t family;
  double variance;
  double length_scale;
  double power;
  double log_amplitude;
} hikf_kernel;

typedef struct hikf_tree hikf_tree; /* opaque, immutable after create */

/* 3D kernel (no reference counterpart; oracle/hikf_oracle3d.py Kern3):
 * variance exp(-r'^p), r' = |(dx/lx, dy/ly, dz/lz)|, family gaussian (p = 2)
 * or exponential (p = 1).  Anisotropic when lx, ly, lz differ. */
typedef struct {
  int32_t family;
  double variance;
  double lx, ly, lz;
} hikf_kernel3;

typedef struct hikf_tree3 hikf_tree3; /* 3D octree bbFMM, opaque */

int hikf_abi_version(void);
/* Copy the last error message of this thread into buf (NUL-terminated). */
int hikf_last_error(char* buf, size_t len);

/* ---- FMM tree: replaces build_tree / FmmTree.__init__ (fmm.py:95-135, 370-374) ----
 * xy_host: (m, 2) row-major cell/point coordinates.  n_cheb in [2, 12],
 * max_leaf >= 1 (FmmConfig, fmm.py:38-54).  All construction kernels run on
 * `stream`; the call returns after the tree is complete. */
int hikf_tree_create(const double* xy_host, int64_t m, const hikf_kernel* kernel, int32_t n_cheb,
                     int64_t max_leaf, void* stream, hikf_tree** out);
int hikf_tree_destroy(hikf_tree* tree);
/* Return the library's cached stream-ordered workspace (FMM expansions,
 * H^T regrouping) to the driver; it is otherwise kept between calls. */
int hikf_release_cached_memory(void);

/* Scalars of the tree: depth, per-level orders (orders[lev] for lev 2..depth,
 * 0 elsewhere; array of 21), root_lo[2], root_size, #occupied leaves,
 * #near leaf pairs. */
int hikf_tree_info(const hikf_tree* tree, int64_t* m, int32_t* depth, int32_t* orders21, double* root_lo2,
                   double* root_size, int64_t* n_leaves, int64_t* n_near_pairs);

/* Parity export of the integer tree data (fmm.py:116-128, 166-190), host
 * buffers sized from hikf_tree_info: order[m] (= FmmTree._order),
 * leaf_ids/leaf_starts/leaf_counts[n_leaves], near_t/near_s[n_near_pairs]
 * (leaf ranks of each adjacent pair, in the reference's offset-major order). */
int hikf_tree_export(const hikf_tree* tree, int64_t* order, int64_t* leaf_ids, int64_t* leaf_starts,
                     int64_t* leaf_counts, int64_t* near_t, int64_t* near_s);

/* Parity export of the operators at one level (fmm.py:246-312):
 *   which = 0: M2L op for offset (dx, dy) -> out[q*q] (q = orders[lev]^2); returns
 *              HIKF_BAD_ARGUMENT if the offset has no pairs at that level.
 *   which = 1: shift op kron(Bx, By) for child parity (dx, dy) = (cx, cy) between
 *              lev and lev+1 -> out[q_child * q_parent].
 *   which = 2: interpolation weights W2 of every point in ORIGINAL point order,
 *              out[m * q_leaf] (lev, dx, dy ignored). */
int hikf_tree_export_op(const hikf_tree* tree, int32_t which, int32_t lev, int32_t dx, int32_t dy, double* out_host);

/* Parity export of the M2L interaction list of one (level, offset) over the
 * full G x G lattice (fmm.py:299-312 _m2l_pairs), evaluated by the device rule
 * the M2L kernel uses.  Call with tgt == NULL to get *count, then with
 * buffers of *count entries. */
int hikf_tree_m2l_pairs(const hikf_tree* tree, int32_t lev, int32_t dx, int32_t dy, int64_t* tgt, int64_t* src,
                        int64_t* count);

/* ---- FmmTree.matmat (fmm.py:325-367) ----
 * U (m x k, ldu) = approx Gram(points) @ V (m x k, ldv), both device. */
int hikf_tree_matmat(hikf_tree* tree, const double* V_dev, int64_t ldv, int64_t k, double* U_dev, int64_t ldu,
                     void* stream);

/* Same product with V = H^T for a CSR H (n x m) on the device, without
 * densifying H^T (filters.py:101-102).  U is (m x n) row-major. */
int hikf_tree_matmat_csrT(hikf_tree* tree, int64_t n, const int32_t* indptr_dev, const int32_t* indices_dev,
                          const double* data_dev, double* U_dev, void* stream);

/* ---- hikf_precompute_fmm (filters.py:99-105) ----
 * C_Q (m x n) = tree @ H^T; HC_Q (n x n) = sym(H C_Q); diag_Q (m) = K(0). */
int hikf_precompute(hikf_tree* tree, int64_t n, const int32_t* indptr_dev, const int32_t* indices_dev,
                    const double* data_dev, double* C_Q_dev, double* HC_Q_dev, double* diag_Q_dev, void* stream);

/* ---- row-sharded precompute: the rows r0 <= i < r1 of C_Q
 * (the upward pass and M2L are replicated; L2P / P2P produce only these
 * rows), the partial H[:, r0:r1] C_Q_rows (n x n; the caller sums the
 * partials over ranks and symmetrises: HC_Q = sym(sum)), and diag_Q rows. */
int hikf_precompute_rows(hikf_tree* tree, int64_t n, const int32_t* indptr_dev, const int32_t* indices_dev,
                         const double* data_dev, int64_t r0, int64_t r1, double* C_Q_rows_dev,
                         double* HC_Q_partial_dev, double* diag_Q_rows_dev, void* stream);
/* Leaf-aligned shard of the precompute: the rows of the points of
 * leaves [leaf0, leaf1) in the tree's leaf order (sorted positions s0 .. s1-1,
 * s0 = leaf_start[leaf0]; C_Q_rows row i <-> sorted position s0 + i <-> original
 * row order[s0 + i]).  P2P and the fused leaf L2L + L2P run for these leaves
 * only, M2L and L2L only for their ancestors (the x-major leaf range is a strip
 * of box columns); the upward pass is replicated.  HC_Q_partial = H[:, rows]
 * C_Q_rows as hikf_precompute_rows.  hikf_leaf_partition: the balanced
 * contiguous leaf range of a rank (equal point counts), out4 = {leaf0, leaf1,
 * s0, s1}. */
int hikf_leaf_partition(const hikf_tree* tree, int32_t world, int32_t rank, int64_t* out4);
int hikf_precompute_leaves(hikf_tree* tree, int64_t n, const int32_t* indptr_dev, const int32_t* indices_dev,
                           const double* data_dev, int64_t leaf0, int64_t leaf1, double* C_Q_rows_dev,
                           double* HC_Q_partial_dev, double* diag_Q_rows_dev, void* stream);

/* ---- hikf_precompute_dense (filters.py:108-115; Gram as kernels.py:97-117) ----
 * The reference's exact-algebra oracle path: C_Q = Q H^T with the dense Gram
 * Q[i][j] = K(|x_i - x_j|), here as a direct sum over the nonzeros of H^T (Q is
 * never stored); HC_Q = sym(H C_Q); diag_Q = diag(Q).  xy_host: m x 2 cell
 * coordinates (original order); H CSR on the device. */
int hikf_precompute_dense(const double* xy_host, int64_t m, const hikf_kernel* kernel, int64_t n,
                          const int32_t* indptr_dev, const int32_t* indices_dev, const double* data_dev,
                          double* C_Q_dev, double* HC_Q_dev, double* diag_Q_dev, void* stream);

/* ---- hikf_init (filters.py:118-126): C = alpha H^T, var = alpha, HC = alpha H H^T ----
 * (the mean is the caller's initial_mean copy). */
int hikf_init_state(int64_t m, int64_t n, const int32_t* indptr_dev, const int32_t* indices_dev,
                    const double* data_dev, double alpha, double* C_out, double* var_out, double* HC_out,
                    void* stream);

/* ---- hikf_predict (filters.py:129-135): out = in + pre, elementwise ----
 * Any output may alias its input. */
int hikf_predict(int64_t m, int64_t n, const double* C_dev, const double* var_dev, const double* HC_dev,
                 const double* C_Q_dev, const double* diag_Q_dev, const double* HC_Q_dev, double* C_out,
                 double* var_out, double* HC_out, void* stream);

/* ---- hikf_update (filters.py:138-157) + the optional fused predict ----
 * Inputs: state (mean m, C m x n, var m, HC n x n), CSR H, r, z (device, n).
 * If C_Q_dev != NULL the predict step (filters.py:129-135) is fused in front:
 * the update then acts on (C + C_Q, var + diag_Q, HC + HC_Q).
 * Outputs are written to the *_out buffers (may not alias the inputs).
 * workspace: device buffer of hikf_update_workspace_bytes(m, n) bytes.
 * Returns HIKF_NOT_PD / HIKF_NEGATIVE_VARIANCE like the reference raises;
 * the stream is synchronised before returning. */
size_t hikf_update_workspace_bytes(int64_t m, int64_t n);
int hikf_update(int64_t m, int64_t n, const double* mean_dev, const double* C_dev, const double* var_dev,
                const double* HC_dev, const double* C_Q_dev, const double* diag_Q_dev, const double* HC_Q_dev,
                const int32_t* indptr_dev, const int32_t* indices_dev, const double* data_dev, double r_variance,
                const double* z_dev, double* mean_out, double* C_out, double* var_out, double* HC_out,
                void* workspace, size_t workspace_bytes, double* min_var_out, void* stream);

/* ---- hikf_update with a chained predict ----
 * Same contract as hikf_update, plus two flags in chain:
 *   bit 0 (produce): the GEMM epilogue also writes the next call's predicted
 *          C' = C_out + C_Q (bit-identical to the predict add) into the
 *          workspace;
 *   bit 1 (consume): this call's C is the previous call's C_out, unmodified,
 *          with the same C_Q and workspace -- use the C' that call produced and
 *          skip the C + C_Q pass.  Pointers, sizes and success of the previous
 *          call are checked; any mismatch falls back to the full predict.
 *   bit 2 (deferred status): the call does not synchronise; min_var_out must be
 *          pinned host memory of 4 doubles that receives, on the stream,
 *          [Cholesky pivot (0 = ok), negative-variance flag, min posterior var,
 *          max prior var].  The caller synchronises the stream (or an event
 *          recorded after the call) before reading it and raises HIKF_NOT_PD /
 *          HIKF_NEGATIVE_VARIANCE itself; a failed step's outputs are undefined.
 * Setting bit 1 while C_out was modified in between gives wrong results.
 * mean_host (optional, pinned host memory, m doubles): mean_out is also
 * copied there, inside the call (the read-back overlaps the update's tail). */
int hikf_update_chained(int64_t m, int64_t n, const double* mean_dev, const double* C_dev, const double* var_dev,
                        const double* HC_dev, const double* C_Q_dev, const double* diag_Q_dev, const double* HC_Q_dev,
                        const int32_t* indptr_dev, const int32_t* indices_dev, const double* data_dev,
                        double r_variance, const double* z_dev, double* mean_out, double* C_out, double* var_out,
                        double* HC_out, void* workspace, size_t workspace_bytes, double* min_var_out, int32_t chain,
                        double* mean_host, void* stream);

/* ---- factored cross covariance (C = C_Q N, N n x n) ----
 * Replaces filters.py:129-157 for a state whose cross covariance is C_Q N
 * (every state of a filter started from C_0 = 0, i.e. alpha = 0): with
 * predict = 1 the prior is predicted first (C' = C_Q (N + I), var + diag_Q,
 * HC + HC_Q).  Outputs mean_out, var_out and HC_out as hikf_update (same
 * consistency check and status codes) and N_out with C_new = C_Q N_out.
 * Per step: the n x n recursion, one m x n GEMV (C_Q u) and one triangular
 * m x n x n GEMM (var -= rowsum((C_Q L_G)^2), G = M S^-1 M^T), no m x n
 * output.  HIKF_NOT_PD also when G loses definiteness.  mean_host as in
 * hikf_update_chained. */
size_t hikf_update_factored_workspace_bytes(int64_t m, int64_t n);
int hikf_update_factored(int64_t m, int64_t n, const double* mean_dev, const double* N_dev, const double* var_dev,
                         const double* HC_dev, const double* C_Q_dev, const double* diag_Q_dev, const double* HC_Q_dev,
                         int32_t predict, const int32_t* indptr_dev, const int32_t* indices_dev,
                         const double* data_dev, double r_variance, const double* z_dev, double* mean_out,
                         double* N_out, double* var_out, double* HC_out, void* workspace, size_t workspace_bytes,
                         double* min_var_out, double* mean_host, double alpha0, const double* A_dev, double* A_out,
                         const int32_t* ht_indptr_dev, const int32_t* ht_indices_dev, const double* ht_data_dev,
                         void* stream);
/* (alpha0 != 0: a state started from C_0 = alpha0 H^T (filters.py:118-126) keeps
 * C = alpha0 H^T A + C_Q N with a second n x n factor A (A_dev -> A_out); H^T is passed
 * as a CSR with m rows.  alpha0 = 0 ignores A and H^T.) */
/* Y (rows x k) += alpha * S X for a CSR S (rows x cols) and X (cols x k), row-major: the
 * sparse term alpha0 H^T A of a factored cross covariance on materialisation. */
int hikf_csr_spmm_add(int64_t rows, int64_t k, const int32_t* indptr_dev, const int32_t* indices_dev,
                      const double* data_dev, const double* X_dev, double alpha, double* Y_dev, void* stream);

/* ---- row-sharded update: the same update on rows [r0, r1) of a
 * state sharded across ranks.  Hmean_dev = the all-reduced H mean (the
 * caller sums the per-rank hikf_csr_spmv partials); the n x n quantities are
 * replicated and identical on every rank.  The negative-variance check is
 * global, so it is not applied here: minmax_out[0] = min over the local rows
 * of the posterior variance, minmax_out[1] = max of the prior variance, for
 * the caller's all-reduce.  Returns HIKF_NOT_PD like hikf_update. */
int hikf_update_rows(int64_t m_local, int64_t n, const double* mean_dev, const double* C_dev, const double* var_dev,
                     const double* HC_dev, const double* C_Q_dev, const double* diag_Q_dev, const double* HC_Q_dev,
                     const double* Hmean_dev, double r_variance, const double* z_dev, double* mean_out,
                     double* C_out, double* var_out, double* HC_out, void* workspace, size_t workspace_bytes,
                     double* minmax_out, int32_t chain, void* stream);
/* (chain: the produce / consume flags of hikf_update_chained, for this rank's rows;
 *  bit 2 (deferred): minmax_out is a DEVICE array of 3 doubles that receives
 *  [min posterior var, max prior var, Cholesky pivot status] on the stream, and
 *  the call neither synchronises nor raises -- the caller all-reduces the array
 *  on the device and checks it at its next host touch.) */
/* y (n) = H x for a CSR H (n x cols) on the device. */
int hikf_csr_spmv(int64_t n, const int32_t* indptr_dev, const int32_t* indices_dev, const double* data_dev,
                  const double* x_dev, double* y_dev, void* stream);

/* ---- spd_solve (linalg.py:18-37): X (n x k) = A^{-1} B, A SPD n x n ----
 * Symmetry check |A - A^T|max <= 1e-10 |A|max (HIKF_ASYMMETRIC), Cholesky
 * (HIKF_NOT_PD with the failing pivot in *info), two triangular solves. */
size_t hikf_spd_solve_workspace_bytes(int64_t n, int64_t k);
int hikf_spd_solve(int64_t n, int64_t k, const double* A_dev, const double* B_dev, double* X_dev, void* workspace,
                   size_t workspace_bytes, int64_t* info, void* stream);

/* ---- build_ray_operator (tomography.py:76-133), host input producer ----
 * Straight rays src[i] -> rcv[i] (n rays, (n, 2) row-major) over the nx x ny
 * cell grid at origin (x0, y0) with spacing (dx, dy).  Two-call protocol:
 * with indices == NULL returns nnz in *nnz_out; then call again with
 * indptr[n+1] / indices[nnz] / data[nnz] host buffers. */
int hikf_ray_operator(int64_t nx, int64_t ny, double dx, double dy, double x0, double y0, int64_t n,
                      const double* src, const double* rcv, int32_t* indptr, int32_t* indices, double* data,
                      int64_t* nnz_out);

/* ---- build_ray_operator on the device (tomography.py:76-133) ----
 * Same result as hikf_ray_operator (bit-identical pattern and lengths) with
 * the per-ray tracing on the GPU: one CTA per ray.  src/rcv are HOST arrays
 * (the ray lengths are taken with the host's hypot so they round like
 * numpy's); indptr_dev[n+1] / indices_dev / data_dev are device buffers.
 * With indices_dev == NULL only indptr_dev and *nnz_out are produced; else
 * capacity (entries) must be >= nnz.  Requires nx + ny <= 4096. */
int hikf_ray_operator_device(int64_t nx, int64_t ny, double dx, double dy, double x0, double y0, int64_t n,
                             const double* src, const double* rcv, int32_t* indptr_dev, int32_t* indices_dev,
                             double* data_dev, int64_t capacity, int64_t* nnz_out, void* stream);

/* ---- 3D path (BASELINE cfg3 / cfg5) -- PARITY UNPINNED:
 * the reference is 2D only; these follow oracle/hikf_oracle3d.py. ----
 * 3D ray operator: cells x fastest (then y, z); n3/d3/o3 = cells/spacing/origin
 * per axis; src/rcv (n, 3) row-major.  Host two-call protocol as
 * hikf_ray_operator; the _device variant as hikf_ray_operator_device. */
int hikf_ray_operator_3d(const int64_t* n3, const double* d3, const double* o3, int64_t n, const double* src,
                         const double* rcv, int32_t* indptr, int32_t* indices, double* data, int64_t* nnz_out);
int hikf_ray_operator_3d_device(const int64_t* n3, const double* d3, const double* o3, int64_t n,
                                const double* src, const double* rcv, int32_t* indptr_dev, int32_t* indices_dev,
                                double* data_dev, int64_t capacity, int64_t* nnz_out, void* stream);
/* octree: xyz_host (m, 3); 2 <= n_cheb <= 5 (one order at every level);
 * 1 <= max_leaf <= 128. */
int hikf_tree3_create(const double* xyz_host, int64_t m, const hikf_kernel3* kernel, int32_t n_cheb,
                      int64_t max_leaf, void* stream, hikf_tree3** out);
int hikf_tree3_destroy(hikf_tree3* tree);
int hikf_tree3_info(const hikf_tree3* tree, int64_t* m, int32_t* depth, int32_t* n_cheb, int64_t* n_leaves,
                    double* lo3, double* size);
/* order[m] (sorted position -> point), leaf keys ((bx G + by) G + bz), starts, counts */
int hikf_tree3_export(const hikf_tree3* tree, int64_t* order, int64_t* leaf_keys, int64_t* leaf_starts,
                      int64_t* leaf_counts);
/* U (m x k) = Q V, device, row-major, original point order */
int hikf_tree3_matmat(const hikf_tree3* tree, const double* V_dev, int64_t k, double* U_dev, void* stream);
/* C_Q = Q H^T (m x n) from CSR H; HC_Q = sym(H C_Q); diag_Q = K(0) */
int hikf_precompute3(hikf_tree3* tree, int64_t n, const int32_t* indptr_dev, const int32_t* indices_dev,
                     const double* data_dev, double* C_Q_dev, double* HC_Q_dev, double* diag_Q_dev, void* stream);

/* ---- dense Kalman filter (filters.py:45-74) and dense Gram (kernels.py:97-117) ----
 * The reference's exact-algebra oracle path, on the device: G (m x m) =
 * K(|x_i - x_j|) (r = 0 -> value_at_zero); kf_predict P_out = P + Q;
 * kf_update: C = H P, S = sym(H C^T + r I), K^T = S^-1 C, mean += K (z - H mean),
 * P = sym(P - K C).  All arrays device, row-major. */
int hikf_dense_gram(const double* xy_host, int64_t m, const hikf_kernel* kernel, double* G_dev, void* stream);
int hikf_kf_predict(int64_t m, const double* P_dev, const double* Q_dev, double* P_out, void* stream);
size_t hikf_kf_workspace_bytes(int64_t m, int64_t n);
int hikf_kf_update(int64_t m, int64_t n, const double* mean_dev, const double* P_dev, const int32_t* indptr_dev,
                   const int32_t* indices_dev, const double* data_dev, double r_variance, const double* z_dev,
                   double* mean_out, double* P_out, void* workspace, size_t workspace_bytes, void* stream);

/* ---- FP64 DMMA GEMM building block (the update's workhorse) ----
 * C (M x N, ldc) = alpha A (M x K, lda) B (K x N, ldb) + beta C, row-major,
 * device pointers.  kmode 0: full; 1: B upper triangular (K-range k <= col
 * tile); 2: B lower triangular.  variant -1 = default tile shape. */
int hikf_dgemm(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B, int64_t ldb,
               double* C, int64_t ldc, double alpha, double beta, int32_t kmode, int32_t variant, void* stream);

/* ---- instrumentation (bench.py) ----
 * Stage timers: CUDA events recorded on the launching stream around each
 * stage (ids in csrc/prof.h: 0 predict, 1 factor, 2 Y GEMM, 3 finalize,
 * 4 C GEMM, 5 P2P, 6 P2M, 7 M2M, 8 M2L, 9 L2P, 10 H^T regrouping, 11 L2L).
 * hikf_launch_count: kernels launched by this library since load. */
int hikf_prof_enable(int on);
int hikf_prof_reset(void);
int hikf_prof_read(int32_t stage, double* total_ms, int64_t* count);
/* useful flops executed by a stage's kernels while profiling was enabled
 * (2 per multiply-add actually performed; skipped zero blocks not counted) */
int hikf_prof_flops(int32_t stage, uint64_t* flops);
int64_t hikf_launch_count(void);
/* A/B switches for tests and tools (results are bit-identical either way):
 * key 0 = the fused small-n chain of the update (csrc/nnchain.cu; 1 on, 0 the
 * multi-launch chain); key 1 = the fused leaf-level L2L + L2P of the Q H^T
 * FMM (csrc/boxgemm.cu leaf_down; 0: separate L2L and L2P kernels); key 2 =
 * P2P reads the near-field kernel blocks stored with the tree (0: evaluates
 * the kernel per (target, entry)); key 3 = the near-field sums are added to
 * the far field inside the fused leaf step (0: by a separate scatter pass);
 * key 4 = the L2L of the inner levels runs child-major (one CTA per occupied
 * child box; 0: parent-major, four children per unit).
 * *previous (optional) receives the old value. */
int hikf_set_tuning(int32_t key, int32_t value, int32_t* previous);

#ifdef __cplusplus
}
#endif
#endif /* HIKF_B200_H */

// Per-step HiKF update and small dense solves (see update.cu).
#pragma once

#include "common.cuh"

namespace hikf {

struct UpdateArgs {
  int64_t m = 0, n = 0;
  const double *mean = nullptr, *C = nullptr, *var = nullptr, *HC = nullptr;
  const double *CQ = nullptr, *dQ = nullptr, *HCQ = nullptr;  // fused predict when CQ != null
  const int32_t *ip = nullptr, *ix = nullptr;
  const double* val = nullptr;
  double r = 0.0;
  const double* z = nullptr;
  double *mean_out = nullptr, *C_out = nullptr, *var_out = nullptr, *HC_out = nullptr;
  void* workspace = nullptr;
  size_t workspace_bytes = 0;
  const double* Hmean = nullptr;  // row-sharded state: all-reduced H mean (else computed from H, mean)
  bool no_check = false;          // row-sharded state: the caller applies the global variance check
  // deferred status (row-sharded state): [min posterior var, max prior var, pivot] written to this
  // device array on the stream; the call neither synchronises nor checks (the caller all-reduces it)
  double* mm_dev = nullptr;
  // deferred host status (hikf_update_chained bit 2): [pivot, negative-variance flag, min var,
  // max prior var] copied into this pinned host array on the stream; the call does not synchronise
  double* status_host = nullptr;
  // chained predict: the caller will pass this call's C_out (untouched) with the same C_Q to the
  // next call; the GEMM epilogue then also writes that call's C' = C_out + C_Q into the workspace
  bool chain = false;     // produce the next call's C'
  bool chain_in = false;  // may consume the C' the previous call produced (pointers are checked too)
  double* mean_host = nullptr;  // optional pinned host copy of mean_out, filled inside the call
  // factored cross-covariance (C = C_Q N, N n x n): C / C_out are unused and CQ is required;
  // Nin -> Nout replaces the m x n state (see update.cu, "factored representation")
  bool factored = false;
  bool predict_in = true;  // factored: the prior is predicted (C' = C_Q (N + I), var + diag_Q, HC + HC_Q)
  const double* Nin = nullptr;
  double* Nout = nullptr;
  // factored with C_0 = alpha0 H^T (alpha0 != 0): C = alpha0 H^T A + C_Q N; Ain -> Aout, and H^T as
  // a CSR (m rows) for the sparse terms
  double alpha0 = 0.0;
  const double* Ain = nullptr;
  double* Aout = nullptr;
  const int32_t *ht_ip = nullptr, *ht_ix = nullptr;
  const double* ht_val = nullptr;
};

struct UpdateResult {
  int pivot = 0;
  double min_var = 0.0;        // min over the rows of the posterior variance
  double max_prior_var = 0.0;  // max over the rows of the prior variance
};

size_t update_workspace_bytes(int64_t m, int64_t n);
size_t update_factored_workspace_bytes(int64_t m, int64_t n);
int update(const UpdateArgs& a, cudaStream_t stream, UpdateResult* res);
int predict(int64_t m, int64_t n, const double* C, const double* var, const double* HC, const double* CQ,
            const double* dQ, const double* HCQ, double* Co, double* varo, double* HCo, cudaStream_t st);
int spmv(int64_t n, const int32_t* ip, const int32_t* ix, const double* val, const double* x, double* y,
         cudaStream_t st);
// Y[i, :] += alpha sum_e val[e] X[ix[e], :] for the rows i of a CSR (rows x cols), X row-major k columns
int csr_spmm_add(int64_t rows, int64_t k, const int32_t* ip, const int32_t* ix, const double* val, const double* X,
                 double alpha, double* Y, cudaStream_t st);
size_t spd_workspace_bytes(int64_t n, int64_t k);
int spd_solve(int64_t n, int64_t k, const double* A, const double* B, double* X, void* ws, size_t ws_bytes,
              int64_t* info, cudaStream_t st);

}  // namespace hikf

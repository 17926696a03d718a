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
};

struct UpdateResult {
  int pivot = 0;
  double min_var = 0.0;
};

size_t update_workspace_bytes(int64_t m, int64_t n);
int update(const UpdateArgs& a, cudaStream_t stream, UpdateResult* res);
int predict(int64_t m, int64_t n, const double* C, const double* var, const double* HC, const double* CQ,
            const double* dQ, const double* HCQ, double* Co, double* varo, double* HCo, cudaStream_t st);
size_t spd_workspace_bytes(int64_t n, int64_t k);
int spd_solve(int64_t n, int64_t k, const double* A, const double* B, double* X, void* ws, size_t ws_bytes,
              int64_t* info, cudaStream_t st);

}  // namespace hikf

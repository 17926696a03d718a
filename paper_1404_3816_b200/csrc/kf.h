// Dense Kalman filter and dense Gram on the GPU (see kf.cu).
#pragma once

#include "common.cuh"

namespace hikf {

int dense_gram(const double* xy_dev, int64_t m, const KParams& kp, double* G, cudaStream_t st);
int kf_predict(int64_t m, const double* P, const double* Q, double* P_out, cudaStream_t st);
size_t kf_workspace_bytes(int64_t m, int64_t n);
int kf_update(int64_t m, int64_t n, const double* mean, const double* P, const int32_t* ip, const int32_t* ix,
              const double* val, double r, const double* z, double* mean_out, double* P_out, void* ws,
              size_t ws_bytes, cudaStream_t st);

}  // namespace hikf

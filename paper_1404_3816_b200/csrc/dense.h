// Direct-sum Q H^T (see dense.cu).
#pragma once

#include "common.cuh"

namespace hikf {

// C_Q (m x n, row-major) = Q H^T with Q[i][j] = K(|x_i - x_j|); xy_dev is m x 2 (original order)
int dense_cq(int64_t m, int64_t n, const double* xy_dev, const int32_t* ip, const int32_t* ix, const double* val,
             const KParams& kp, double* CQ, cudaStream_t st);

}  // namespace hikf

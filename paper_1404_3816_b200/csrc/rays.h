// Straight-ray operator on the device (see rays.cu).
#pragma once

#include "common.cuh"

namespace hikf {

int ray_operator_device(int64_t nx, int64_t ny, double dx, double dy, double x0, double y0, int64_t n,
                        const double* src_host, const double* rcv_host, int32_t* indptr_dev, int32_t* indices_dev,
                        double* data_dev, int64_t capacity, int64_t* nnz_out, cudaStream_t st);

int ray_operator_3d_device(const int64_t n3[3], const double d3[3], const double o3[3], int64_t n,
                           const double* src_host, const double* rcv_host, int32_t* indptr_dev, int32_t* indices_dev,
                           double* data_dev, int64_t capacity, int64_t* nnz_out, cudaStream_t st);

}  // namespace hikf

// 3D octree bbFMM (see fmm3d.cu).
#pragma once

#include "common.cuh"

namespace hikf {

int tree3_build(const double* xyz_host, int64_t m, const hikf_kernel3& k, int n_cheb, int64_t max_leaf,
                cudaStream_t st, hikf_tree3** out);
void tree3_free(hikf_tree3* t);
int tree3_matmat(const hikf_tree3* t, const double* V, int64_t ldv, int64_t k, double* U, int64_t ldu,
                 cudaStream_t st);
int tree3_matmat_csrT(const hikf_tree3* t, int64_t n, const int32_t* ip, const int32_t* ix, const double* val,
                      double* U, cudaStream_t st);
int tree3_info(const hikf_tree3* t, int64_t* m, int32_t* depth, int32_t* n_cheb, int64_t* n_leaves, double* lo3,
               double* size);
void tree3_kernel(const hikf_tree3* t, hikf_kernel3* k);
int tree3_export(const hikf_tree3* t, int64_t* order, int64_t* leaf_keys, int64_t* leaf_starts, int64_t* leaf_counts);

}  // namespace hikf

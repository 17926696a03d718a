// Stage timing scopes and launch counting (see prof.cu).
#pragma once

#include <atomic>

#include "common.cuh"

namespace hikf {

// stage ids, mirrored in paper_1404_3816_b200/_lib.py STAGES
enum Stage {
  ST_PREDICT = 0,
  ST_FACTOR = 1,   // S, Cholesky + inverse, n x n products, innovation
  ST_GEMM_Y = 2,   // unused since the single-GEMM update (kept: stage ids are ABI)
  ST_FINALIZE = 3, // var / mean rows + consistency check
  ST_GEMM_C = 4,   // C_new = C' - Y P
  ST_P2P = 5,
  ST_P2M = 6,
  ST_M2M = 7,
  ST_M2L = 8,
  ST_L2P = 9,
  ST_DENSIFY = 10, // H^T regrouping (sparse charges) / scatter
  ST_L2L = 11,     // parent-to-child locals (sparse path; fused into M2L on the dense path)
  ST_COUNT = 12
};

// device counter of useful flops of a stage while profiling is enabled, else null
unsigned long long* prof_flops_ptr(int stage);

class ProfScope {
 public:
  ProfScope(int stage, cudaStream_t st);
  ~ProfScope();

 private:
  int stage_;
  cudaStream_t st_;
  bool active_;
  cudaEvent_t a_, b_;
};

}  // namespace hikf

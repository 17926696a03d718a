// Probe: CUTLASS 2.x SM80 FP64 tensor-op (DMMA.8x8x4) GEMM tile configurations
// at the K-GEMM shape (M = 1,048,576 state rows, N = K = 1024 rays), timed
// with CUDA events against cuBLAS DGEMM.  Tuning aid for csrc/kgemm.cu.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I<cutlass>/include \
//        tools/cutlass_dgemm_probe.cu -lcublas -o tools/cutlass_dgemm_probe
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cublas_v2.h>
#include <cuda_runtime.h>

#include "cutlass/gemm/device/gemm.h"

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);  \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

using RM = cutlass::layout::RowMajor;

template <int BM, int BN, int BK, int WM, int WN, int WK, int STAGES>
float run_cutlass(int M, int N, int K, const double* A, const double* B, double* C, int reps) {
  using Gemm = cutlass::gemm::device::Gemm<
      double, RM, double, RM, double, RM, double, cutlass::arch::OpClassTensorOp, cutlass::arch::Sm80,
      cutlass::gemm::GemmShape<BM, BN, BK>, cutlass::gemm::GemmShape<WM, WN, WK>, cutlass::gemm::GemmShape<8, 8, 4>,
      cutlass::epilogue::thread::LinearCombination<double, 1, double, double>,
      cutlass::gemm::threadblock::GemmIdentityThreadblockSwizzle<>, STAGES>;
  Gemm op;
  typename Gemm::Arguments args({M, N, K}, {A, K}, {B, N}, {C, N}, {C, N}, {1.0, 0.0});
  if (op.can_implement(args) != cutlass::Status::kSuccess) return -1.f;
  if (op.initialize(args) != cutlass::Status::kSuccess) return -2.f;
  op();
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) op();
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 1 << 20, N = 1024, K = 1024, reps = 3;
  double *A, *B, *C;
  CK(cudaMalloc(&A, (size_t)M * K * 8));
  CK(cudaMalloc(&B, (size_t)K * N * 8));
  CK(cudaMalloc(&C, (size_t)M * N * 8));
  std::vector<double> h((size_t)K * N);
  for (auto& x : h) x = (rand() % 1000) / 1000.0;
  CK(cudaMemcpy(B, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemset(A, 0, (size_t)M * K * 8));
  const double fl = 2.0 * M * N * K;
  auto rep = [&](const char* name, float ms) {
    printf("%-44s %8.3f ms  %6.2f TF/s\n", name, ms, ms > 0 ? fl / ms / 1e9 : 0.0);
    fflush(stdout);
  };
  {
    cublasHandle_t hd;
    cublasCreate(&hd);
    const double one = 1.0, zero = 0.0;
    // row-major C = A B  ==  column-major C^T = B^T A^T
    cublasDgemm(hd, CUBLAS_OP_N, CUBLAS_OP_N, N, M, K, &one, B, N, A, K, &zero, C, N);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) cublasDgemm(hd, CUBLAS_OP_N, CUBLAS_OP_N, N, M, K, &one, B, N, A, K, &zero, C, N);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    rep("cublasDgemm", ms / reps);
  }
  rep("cutlass 64x128x16 w32x64x16 s3", run_cutlass<64, 128, 16, 32, 64, 16, 3>(M, N, K, A, B, C, reps));
  rep("cutlass 64x128x16 w32x64x16 s4", run_cutlass<64, 128, 16, 32, 64, 16, 4>(M, N, K, A, B, C, reps));
  rep("cutlass 128x64x16 w64x32x16 s3", run_cutlass<128, 64, 16, 64, 32, 16, 3>(M, N, K, A, B, C, reps));
  rep("cutlass 128x128x16 w64x64x16 s3", run_cutlass<128, 128, 16, 64, 64, 16, 3>(M, N, K, A, B, C, reps));
  rep("cutlass 128x128x16 w32x64x16 s4", run_cutlass<128, 128, 16, 32, 64, 16, 4>(M, N, K, A, B, C, reps));
  rep("cutlass 64x64x16 w32x32x16 s5", run_cutlass<64, 64, 16, 32, 32, 16, 5>(M, N, K, A, B, C, reps));
  rep("cutlass 64x128x32 w32x64x32 s3", run_cutlass<64, 128, 32, 32, 64, 32, 3>(M, N, K, A, B, C, reps));
  rep("cutlass 128x64x32 w64x32x32 s3", run_cutlass<128, 64, 32, 64, 32, 32, 3>(M, N, K, A, B, C, reps));
  rep("cutlass 64x256x16 w32x64x16 s3", run_cutlass<64, 256, 16, 32, 64, 16, 3>(M, N, K, A, B, C, reps));
  return 0;
}

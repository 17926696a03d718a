// Micro-benchmark of the 64 x 64 Cholesky + inverse base block (chol_block.cuh):
// per-section clock64 stamps of one CTA, and the launch-to-launch time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_1404_3816_b200/csrc -I../include \
//        -o chol_bench chol_bench.cu && ./chol_bench
#include <cstdio>
#include <cstring>
#include <vector>

__device__ long long g_sec[16];
#define CHOL_BENCH_CLOCK g_sec
#include "chol_block.cuh"

using namespace hikf;

__global__ void __launch_bounds__(256) base_kernel(const double* S, double* L, double* Li, int* status,
                                                   long long* clk) {
  extern __shared__ double sm[];
  long long t0 = clock64();
  chol_inv_block(S, 64, 64, 0, L, Li, status, sm);
  long long t1 = clock64();
  if (threadIdx.x == 0) { clk[0] = t1 - t0; clk[1] = g_sec[0]; clk[2] = g_sec[1]; clk[3] = g_sec[2]; }
}

// profiling aid: one CTA per SM, each repeating the block (long enough for ncu's stall sampling)
__global__ void __launch_bounds__(256) rep_kernel(const double* S, double* L, double* Li, int* status, int reps) {
  extern __shared__ double sm[];
  for (int r = 0; r < reps; ++r) chol_inv_block(S, 64, 64, 0, L + blockIdx.x * 4096, Li + blockIdx.x * 4096, status, sm);
}

int main(int argc, char** argv) {
  const int n = 64;
  std::vector<double> h(n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) h[i * n + j] = (i == j ? n : 0.0) + 1.0 / (1 + i + j);
  double *S, *L, *Li;
  int* st;
  long long* clk;
  cudaMalloc(&S, 8 * n * n);
  cudaMalloc(&L, 8 * n * n);
  cudaMalloc(&Li, 8 * n * n);
  cudaMalloc(&st, 16);
  cudaMallocManaged(&clk, 64);
  cudaMemcpy(S, h.data(), 8 * n * n, cudaMemcpyHostToDevice);
  cudaMemset(st, 0, 16);
  cudaFuncSetAttribute(base_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CHOL_SMEM);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    base_kernel<<<1, 256, CHOL_SMEM>>>(S, L, Li, st, clk);
    cudaDeviceSynchronize();
    printf("single launch: %lld cycles in-kernel (chol %lld, store %lld, inverse %lld)\n", clk[0], clk[1], clk[2], clk[3]);
    long long hs[16]; cudaMemcpyFromSymbol(hs, g_sec, sizeof(hs));
    printf("  cholesky %lld, barrier %lld, inverse %lld\n", hs[12] - hs[4], hs[13] - hs[12], hs[14] - hs[13]);
  }
  cudaEventRecord(a);
  for (int rep = 0; rep < 100; ++rep) base_kernel<<<1, 256, CHOL_SMEM>>>(S, L, Li, st, clk);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  printf("back-to-back: %.2f us per launch, last in-kernel %lld cycles, err %s\n", ms * 10, clk[0],
         cudaGetErrorString(cudaGetLastError()));
  std::vector<double> hl(n * n), hli(n * n);
  cudaMemcpy(hl.data(), L, 8 * n * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(hli.data(), Li, 8 * n * n, cudaMemcpyDeviceToHost);
  unsigned long long hsum = 0;
  for (int i = 0; i < n; ++i)
    for (int k = 0; k <= i; ++k) {
      unsigned long long u, v;
      memcpy(&u, &hl[i * n + k], 8);
      memcpy(&v, &hli[i * n + k], 8);
      hsum = hsum * 1099511628211ull + u;
      hsum = hsum * 1099511628211ull + v;
    }
  printf("digest %016llx\n", hsum);
  if (argc > 1) {  // ./chol_bench prof: the long run for ncu
    double *L2, *Li2;
    cudaMalloc(&L2, 8 * 4096 * 148);
    cudaMalloc(&Li2, 8 * 4096 * 148);
    cudaFuncSetAttribute(rep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CHOL_SMEM);
    rep_kernel<<<148, 256, CHOL_SMEM>>>(S, L2, Li2, st, 200);
    printf("rep run: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  }
  return 0;
}

// FP64 pipe microbenchmarks on sm_100a: DFMA (SIMT) vs DMMA (mma.sync .f64) throughput,
// plus double-precision exp() throughput. Prints one JSON object.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

__global__ void dmma_loop(double* out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) { acc[j][0] = 0; acc[j][1] = 0; }
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int j = 0; j < 8; ++j) dmma884(acc[j], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += acc[j][0] + acc[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dexp_loop(double* out, int iters) {
  double x = -(threadIdx.x + 1) * 1e-3, s = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) { s += exp(x); x -= 1e-7; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  double* out; cudaMalloc(&out, sizeof(double) * 148 * 64 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  printf("{\"sms\": %d, \"clock_khz\": %d", sms, p.clockRate);
  // DFMA: blocks = sms*4, 256 threads, iters
  for (int threads : {256, 512}) {
    int blocks = sms * 4, iters = 4096;
    dfma_loop<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0); dfma_loop<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * blocks * threads * (double)iters * 16 * 8;
    printf(", \"dfma_tflops_t%d\": %.3f", threads, flops / (ms * 1e-3) / 1e12);
  }
  for (int threads : {128, 256, 512}) {
    int blocks = sms * 4, iters = 2048;
    dmma_loop<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0); dmma_loop<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double warps = blocks * threads / 32.0;
    double flops = 2.0 * 256 * warps * (double)iters * 4 * 8;
    printf(", \"dmma_tflops_t%d\": %.3f", threads, flops / (ms * 1e-3) / 1e12);
  }
  {
    int blocks = sms * 4, threads = 256, iters = 1024;
    dexp_loop<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0); dexp_loop<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)blocks * threads * iters * 8;
    printf(", \"dexp_gops\": %.3f", n / (ms * 1e-3) / 1e9);
  }
  cudaError_t err = cudaGetLastError();
  printf(", \"err\": \"%s\"}\n", cudaGetErrorString(err));
  return 0;
}

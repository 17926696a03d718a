// FP64 dependent-latency probe: cycles per op of a dependent DFMA / DMUL / sqrt / rcp chain (one thread)
#include <cstdio>
__global__ void k(double* out, long long* clk, double x0) {
  double x = x0, y = 1.0000001;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = fma(x, y, 1e-9);
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = x * y;
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = __dsqrt_rn(x) + 0.5;
  long long t3 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = __drcp_rn(x) + 0.5;
  long long t4 = clock64();
  float f = (float)x;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) f = fmaf(f, 1.0000001f, 1e-9f);
  long long t5 = clock64();
  out[0] = x + f;
  clk[0] = t1 - t0; clk[1] = t2 - t1; clk[2] = t3 - t2; clk[3] = t4 - t3; clk[4] = t5 - t4;
}
int main() {
  double* o; long long* c;
  cudaMallocManaged(&o, 8); cudaMallocManaged(&c, 64);
  for (int r = 0; r < 2; ++r) {
    k<<<1, 1>>>(o, c, 1.5);
    cudaDeviceSynchronize();
    printf("cycles/op: dfma %.1f dmul %.1f dsqrt+add %.1f drcp+add %.1f ffma %.1f\n", c[0] / 1e3, c[1] / 1e3, c[2] / 1e3, c[3] / 1e3, c[4] / 1e3);
  }
}

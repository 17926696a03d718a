// Shared device/host helpers for libhikf_b200 (sm_100a, FP64).
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "hikf_b200.h"

namespace hikf {

// ---------------------------------------------------------------------------
// error reporting (thread-local last error, mirrored to hikf_last_error)
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);
const std::string& last_error();

#define HIKF_CHECK_CUDA(call)                                                                         \
  do {                                                                                                \
    cudaError_t e_ = (call);                                                                          \
    if (e_ != cudaSuccess) {                                                                          \
      ::hikf::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_));           \
      return HIKF_CUDA_ERROR;                                                                         \
    }                                                                                                 \
  } while (0)

extern std::atomic<long long> g_launches;  // kernels launched by this library (prof.cu)
#define HIKF_CHECK_LAUNCH()                   \
  do {                                        \
    ::hikf::g_launches.fetch_add(1);          \
    HIKF_CHECK_CUDA(cudaGetLastError());      \
  } while (0)

#define HIKF_TRY(expr)              \
  do {                              \
    int s_ = (expr);                \
    if (s_ != HIKF_OK) return s_;   \
  } while (0)

// ---------------------------------------------------------------------------
// kernel (covariance function) parameters, kernels.py:25-88
// ---------------------------------------------------------------------------
struct KParams {
  int family;      // HIKF_GAUSSIAN / HIKF_EXPONENTIAL / HIKF_LOGARITHM
  int pmode;       // 1: p == 1, 2: p == 2, 3: p == 0.5, 0: general pow
  double variance;
  double length;
  double power;
  double log_amp;
  double inv_length;  // 1 / length (the near-field fast path multiplies instead of dividing)
};

KParams make_kparams(const hikf_kernel& k);

// K(r) with numpy's evaluation order: variance * exp(-((r / L) ** p)); numpy's
// scalar-power fast paths make p == 1, 2, 0.5 a copy / square / sqrt.
// logarithm: A * log(r) with r == 0 -> 0 (kernels.py:121-130, fmm.py:192-195).
__host__ __device__ __forceinline__ double kernel_of_r(const KParams& k, double r) {
  if (k.family == HIKF_LOGARITHM) return r == 0.0 ? 0.0 : k.log_amp * log(r);
  double t = r / k.length;
  if (k.pmode == 2)
    t = t * t;
  else if (k.pmode == 3)
    t = sqrt(t);
  else if (k.pmode == 0)
    t = pow(t, k.power);
  return k.variance * exp(-t);
}

// Near-field evaluation (P2P): r * (1 / L) instead of r / L.  The argument differs by at
// most 1 ulp and exp(-t) by t ulp (t = r / L < 1 in the near field): reassociation-level,
// while a DDIV costs ~10 FP64 instructions of the ~40 an evaluation takes.  Operators
// (M2L / interpolation) keep kernel_of_r, which follows numpy's rounding.
__host__ __device__ __forceinline__ double kernel_of_r_near(const KParams& k, double r) {
  if (k.family == HIKF_LOGARITHM) return r == 0.0 ? 0.0 : k.log_amp * log(r);
  double t = r * k.inv_length;
  if (k.pmode == 2)
    t = t * t;
  else if (k.pmode == 3)
    t = sqrt(t);
  else if (k.pmode == 0)
    t = pow(t, k.power);
  return k.variance * exp(-t);
}

#ifdef __CUDACC__
// Euclidean distance with cdist / np.linalg.norm rounding: no FMA contraction.
__device__ __forceinline__ double dist2d(double ax, double ay, double bx, double by) {
  double dx = __dsub_rn(ax, bx), dy = __dsub_rn(ay, by);
  return __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
}

// ---------------------------------------------------------------------------
// FP64 tensor op: mma.sync m8n8k4 (SASS DMMA.8x8x4).  Fragments (lane = 4g + t):
//   A (8x4, row): a = A[g][t]      B (4x8, col): b = B[t][g]
//   C (8x8):      c0 = C[g][2t], c1 = C[g][2t+1]
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// cp.async (LDGSTS) helpers; src_size 0 zero-fills the destination.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

#endif  // __CUDACC__

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// grid sizing: number of SMs of the current device (cached)
int num_sms();

}  // namespace hikf

// Stage timers (CUDA events on the launching stream) and a launch counter,
// exposed through the C ABI so bench.py can attribute device time to kernels.
#include <mutex>
#include <vector>

#include "prof.h"

namespace hikf {

std::atomic<long long> g_launches{0};

namespace {
struct Rec {
  int stage;
  cudaEvent_t a, b;
};
std::mutex g_mu;
bool g_on = false;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;
unsigned long long* g_flops = nullptr;  // ST_COUNT device counters

cudaEvent_t take() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

unsigned long long* prof_flops_ptr(int stage) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_on) return nullptr;
  if (!g_flops) {
    if (cudaMalloc(&g_flops, sizeof(unsigned long long) * ST_COUNT) != cudaSuccess) return nullptr;
    cudaMemset(g_flops, 0, sizeof(unsigned long long) * ST_COUNT);
  }
  return g_flops + stage;
}

ProfScope::ProfScope(int stage, cudaStream_t st) : stage_(stage), st_(st), active_(false) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_on) return;
  a_ = take();
  b_ = take();
  cudaEventRecord(a_, st_);
  active_ = true;
}

ProfScope::~ProfScope() {
  if (!active_) return;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEventRecord(b_, st_);
  g_recs.push_back({stage_, a_, b_});
}

}  // namespace hikf

using namespace hikf;

extern "C" {

int hikf_prof_enable(int on) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_on = on != 0;
  return HIKF_OK;
}

int hikf_prof_reset(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& r : g_recs) {
    cudaEventSynchronize(r.b);
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_recs.clear();
  if (g_flops) {
    cudaDeviceSynchronize();
    cudaMemset(g_flops, 0, sizeof(unsigned long long) * ST_COUNT);
  }
  return HIKF_OK;
}

int hikf_prof_flops(int32_t stage, uint64_t* out) {
  if (!out || stage < 0 || stage >= ST_COUNT) return HIKF_BAD_ARGUMENT;
  *out = 0;
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_flops) {
    cudaDeviceSynchronize();
    unsigned long long v = 0;
    cudaMemcpy(&v, g_flops + stage, sizeof(v), cudaMemcpyDeviceToHost);
    *out = v;
  }
  return HIKF_OK;
}

int hikf_prof_read(int32_t stage, double* total_ms, int64_t* count) {
  std::lock_guard<std::mutex> lk(g_mu);
  double tot = 0.0;
  int64_t cnt = 0;
  for (auto& r : g_recs) {
    if (r.stage != stage) continue;
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    tot += ms;
    ++cnt;
  }
  if (total_ms) *total_ms = tot;
  if (count) *count = cnt;
  return HIKF_OK;
}

int64_t hikf_launch_count(void) { return g_launches.load(); }

}  // extern "C"

#include "boxgemm.h"
#include "sparse.h"
#include "nnchain.h"

extern "C" int hikf_set_tuning(int32_t key, int32_t value, int32_t* previous) {
  int prev = 0;
  switch (key) {
    case 0:
      prev = hikf::nn_set_fused(value);
      break;
    case 1:
      prev = hikf::leaf_set_fused(value);
      break;
    case 2:
      prev = hikf::p2p_set_near_blocks(value);
      break;
    case 3:
      prev = hikf::near_set_fold(value);
      break;
    case 4:
      prev = hikf::l2l_set_child_major(value);
      break;
    default:
      hikf::set_error("unknown tuning key %d", (int)key);
      return HIKF_BAD_ARGUMENT;
  }
  if (previous) *previous = prev;
  return HIKF_OK;
}

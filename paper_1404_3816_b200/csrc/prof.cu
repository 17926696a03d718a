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

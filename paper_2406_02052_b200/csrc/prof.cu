// prof.cu -- launch counter and event-based per-category timing (product code).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstring>

#include "../../include/petra.h"
#include "errors.h"
#include "common.cuh"
#include "prof.h"

namespace petra {
std::atomic<int64_t> Prof::launches{0};
bool Prof::enabled = false;
int64_t Prof::scope_grid = 0;
std::vector<Prof::Rec> Prof::recs;
std::vector<std::string> Prof::names;
std::vector<cudaEvent_t> Prof::pool;
static size_t g_pool_next = 0;

int env_int(const char *name, int dflt) {
  const char *e = getenv(name);
  return (e && *e) ? atoi(e) : dflt;
}

// Persistent-grid caps by the number of stages that share the GPU (set by each pipeline
// from its local stage count; 1 for the stage-level API): the fewer stages run
// concurrently, the more of the GPU each kernel should take.  Measured (DESIGN.md 7 "Grid
// sizing"): 1 stage (J = 1) 148 CTAs, 2 -> 96, 3 -> 64, >= 4 -> 40; wgrad splits 48 / 48 /
// 32 / 32.  PETRA_CONV_CTAS / PETRA_WGRAD_CTAS / PETRA_WGRAD_HALO_CTAS override.
static std::atomic<int> g_stages_per_gpu{1};
void set_stages_per_gpu(int n) { g_stages_per_gpu.store(std::max(1, n)); }
int stages_per_gpu() { return g_stages_per_gpu.load(); }
int conv_cap() {
  static const int env = env_int("PETRA_CONV_CTAS", 0);
  if (env > 0) return std::min(kNumSMs, env);
  const int n = stages_per_gpu();
  return n <= 1 ? kNumSMs : (n == 2 ? 96 : (n == 3 ? 64 : 40));
}
int wgrad_ctas(const char *env_name) {
  const int env = env_int(env_name, 0);
  if (env > 0) return env;
  return stages_per_gpu() <= 2 ? 48 : 32;
}
// the largest split target any stage count selects (workspace sizing: a stage's buffers must fit
// the plans of every later launch, whatever the process's pipelines set meanwhile)
int wgrad_ctas_max(const char *env_name) {
  const int env = env_int(env_name, 0);
  return env > 0 ? env : 48;
}
int conv_grid(int work) { return std::max(1, std::min(work, conv_cap())); }

bool pdl_enabled() {
  static const bool on = [] {
    const char *e = getenv("PETRA_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

int Prof::category(const char *name) {
  for (size_t i = 0; i < names.size(); ++i)
    if (names[i] == name) return (int)i;
  names.push_back(name);
  return (int)names.size() - 1;
}

cudaEvent_t Prof::ev() {
  if (g_pool_next == pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    pool.push_back(e);
  }
  return pool[g_pool_next++];
}
}  // namespace petra

using petra::Prof;

extern "C" {

int64_t petra_launch_count(void) { return Prof::launches.load(); }

petra_status petra_profile(int32_t enable) {
  if (enable) {
    cudaDeviceSynchronize();
    Prof::recs.clear();
    petra::g_pool_next = 0;
  }
  Prof::enabled = enable != 0;
  return PETRA_OK;
}

petra_status petra_profile_read(petra_prof_entry *out, int32_t cap, int32_t *n) {
  if (!out || !n) return PETRA_E_ARG;
  if (cudaDeviceSynchronize() != cudaSuccess) return PETRA_E_CUDA;
  int nc = (int)Prof::names.size();
  std::vector<petra_prof_entry> agg(nc);
  for (int i = 0; i < nc; ++i) {
    std::memset(&agg[i], 0, sizeof(petra_prof_entry));
    std::strncpy(agg[i].name, Prof::names[i].c_str(), sizeof(agg[i].name) - 1);
  }
  for (auto &r : Prof::recs) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    agg[r.cat].launches += 1;
    agg[r.cat].ms += ms;
    agg[r.cat].flops += r.flops;
    agg[r.cat].bytes += r.bytes;
  }
  int k = 0;
  for (int i = 0; i < nc && k < cap; ++i)
    if (agg[i].launches) out[k++] = agg[i];
  *n = k;
  return PETRA_OK;
}

petra_status petra_profile_records(petra_prof_record *out, int32_t cap, int32_t *n) {
  if (!out || !n) return PETRA_E_ARG;
  if (cudaDeviceSynchronize() != cudaSuccess) return PETRA_E_CUDA;
  int k = 0;
  for (auto &r : Prof::recs) {
    if (k >= cap) break;
    petra_prof_record &o = out[k++];
    std::memset(&o, 0, sizeof(o));
    std::strncpy(o.name, Prof::names[r.cat].c_str(), sizeof(o.name) - 1);
    cudaEventElapsedTime(&o.ms, r.a, r.b);
    o.flops = r.flops;
    o.bytes = r.bytes;
    o.ctas = (int32_t)std::min<int64_t>(r.ctas, INT32_MAX);
  }
  *n = (int32_t)Prof::recs.size();
  return PETRA_OK;
}
}

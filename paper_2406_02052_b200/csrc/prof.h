// prof.h -- launch counting and optional per-category CUDA-event timing (product code).
// The bench reads these through petra_profile_* to report the dominant
// kernel's achieved FLOP/s or GB/s, measured with events on the launch stream.
#pragma once
#include <cuda_runtime.h>

#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

namespace petra {

// NVTX range (header-only NVTX v3: a no-op unless a tool such as nsys is attached).
// The library marks each pipeline tick, each stage's tick inside it and each exchange
// direction, so an nsys timeline shows per stage and phase where the time goes and how
// the exchange overlaps the compute.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  template <typename... A>
  NvtxRange(const char *fmt, A... a) {
    char buf[96];
    std::snprintf(buf, sizeof(buf), fmt, a...);
    nvtxRangePushA(buf);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};

struct Prof {
  static std::atomic<int64_t> launches;  // every kernel launch of the library
  static bool enabled;
  struct Rec {
    int cat;
    cudaEvent_t a, b;
    double flops, bytes;
    int64_t ctas;  // the largest grid launched inside the scope
  };
  static int64_t scope_grid;  // largest grid since the innermost open ProfScope began
  static void note_grid(const dim3 &g) {
    if (enabled) scope_grid = std::max<int64_t>(scope_grid, (int64_t)g.x * g.y * g.z);
  }
  static std::vector<Rec> recs;
  static std::vector<std::string> names;
  static std::vector<cudaEvent_t> pool;
  static int category(const char *name);
  static cudaEvent_t ev();
};

// RAII scope around one logical kernel (may contain several launches)
struct ProfScope {
  int cat = -1;
  cudaStream_t st;
  cudaEvent_t a{}, b{};
  double flops, bytes;
  int64_t saved_grid = 0;
  ProfScope(const char *name, cudaStream_t s, double fl, double by) : st(s), flops(fl), bytes(by) {
    if (!Prof::enabled) return;
    saved_grid = Prof::scope_grid;
    Prof::scope_grid = 0;
    cat = Prof::category(name);
    a = Prof::ev();
    b = Prof::ev();
    record(a);
  }
  ~ProfScope() {
    if (cat < 0) return;
    record(b);
    Prof::recs.push_back({cat, a, b, flops, bytes, Prof::scope_grid});
    Prof::scope_grid = std::max(saved_grid, Prof::scope_grid);
  }
  // inside a stream capture (the profiled replay runs each stage tick as a one-off graph, so
  // the host's launch work is not between the two events) the record must be an event node
  void record(cudaEvent_t e) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
    else cudaEventRecord(e, st);
  }
};

inline void count_launch(int n = 1) { Prof::launches.fetch_add(n, std::memory_order_relaxed); }

}  // namespace petra

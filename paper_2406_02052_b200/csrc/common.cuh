// common.cuh -- shared device/host helpers of the PETRA B200 library (product code).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdexcept>
#include <string>
#include <utility>

#include "prof.h"

namespace petra {

struct CudaError : std::runtime_error {
  explicit CudaError(const std::string &m) : std::runtime_error(m) {}
};

#define PETRA_CUDA(call)                                                                   \
  do {                                                                                     \
    cudaError_t e__ = (call);                                                              \
    if (e__ != cudaSuccess)                                                                \
      throw ::petra::CudaError(std::string(#call) + ": " + cudaGetErrorString(e__) + " @" + \
                               __FILE__ + ":" + std::to_string(__LINE__));                 \
  } while (0)

#define PETRA_LAUNCH_CHECK()       \
  do {                             \
    ::petra::count_launch();       \
    PETRA_CUDA(cudaGetLastError()); \
  } while (0)

constexpr int kNumSMs = 148;  // B200

// Programmatic dependent launch (PDL).  Every library kernel is launched with
// programmatic stream serialisation and begins with griddepcontrol.wait (all of
// its stream predecessor's memory operations are visible after it) followed by
// griddepcontrol.launch_dependents, so the NEXT kernel of the stream is launched
// and made resident while this one runs, and starts the moment it completes: the
// kernel-boundary gap of a chain of small dependent kernels shrinks to the wait.
// A kernel never touches global memory before its wait, so the ordering is that of
// plain stream serialisation (PETRA_PDL=0 launches without the attribute).
__device__ __forceinline__ void pdl_wait_trigger() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

bool pdl_enabled();
// tuning knob from the environment (read once per name; default if unset)
int env_int(const char *name, int dflt);
// CTAs of a persistent conv kernel: min(work items, cap).  The stages of a tick and a
// stage's two directions run concurrently, so a kernel that leaves SMs to its
// neighbours raises the tick's throughput (measured); PETRA_CONV_CTAS.
int conv_grid(int work);
int conv_cap();
// stages sharing this GPU (persistent-grid caps, prof.cu); set by petra_pipeline_create
void set_stages_per_gpu(int n);
int stages_per_gpu();
int wgrad_ctas(const char *env_name);      // split-K target CTAs of the wgrads
int wgrad_ctas_max(const char *env_name);  // ... the largest (workspace sizing)

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args &&...args) {
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  // the stream's priority on the launch itself, so a captured graph's kernel nodes keep it
  // (the stage's backward stream outranks its forward; the wgrad stream ranks lowest)
  int prio = 0;
  cudaStreamGetPriority(st, &prio);
  attr[1].id = cudaLaunchAttributePriority;
  attr[1].val.priority = prio;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  Prof::note_grid(grid);
  PETRA_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// the same launch as thread-block clusters of `cluster` CTAs along x (grid.x % cluster == 0)
template <typename... KArgs, typename... Args>
inline void launch_k_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int cluster,
                             Args &&...args) {
  cudaLaunchAttribute attr[3];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  int prio = 0;
  cudaStreamGetPriority(st, &prio);
  attr[1].id = cudaLaunchAttributePriority;
  attr[1].val.priority = prio;
  attr[2].id = cudaLaunchAttributeClusterDimension;
  attr[2].val.clusterDim.x = (unsigned)cluster;
  attr[2].val.clusterDim.y = 1;
  attr[2].val.clusterDim.z = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 3;
  Prof::note_grid(grid);
  PETRA_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Geometry of one convolution in NHWC with weights [Co][k][k][Ci], pad = (k-1)/2.
struct ConvGeom {
  int B, H, W, Ci;   // input
  int Ho, Wo, Co;    // output
  int k, s, p;
  __host__ __device__ int64_t M() const { return (int64_t)B * Ho * Wo; }
  __host__ __device__ int64_t Min() const { return (int64_t)B * H * W; }
  __host__ __device__ int K() const { return k * k * Ci; }
};

inline ConvGeom make_geom(int B, int H, int W, int Ci, int Co, int k, int s) {
  ConvGeom g;
  g.B = B; g.H = H; g.W = W; g.Ci = Ci; g.Co = Co; g.k = k; g.s = s; g.p = (k - 1) / 2;
  g.Ho = (H + 2 * g.p - k) / s + 1;
  g.Wo = (W + 2 * g.p - k) / s + 1;
  return g;
}

}  // namespace petra

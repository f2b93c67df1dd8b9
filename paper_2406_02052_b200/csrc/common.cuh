// common.cuh -- shared device/host helpers of the PETRA B200 library (product code).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdexcept>
#include <string>

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

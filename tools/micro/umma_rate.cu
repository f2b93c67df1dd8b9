// UMMA issue-rate microbenchmark (B200): cycles per tcgen05.mma (kind::f16, M=128, K=16)
// for N in {64, 128, 256}, 1..4 independent accumulators, A descriptor 1 KB-aligned or
// shifted by whole 128-byte rows (the halo kernel's tap views).  One CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_2406_02052_b200/csrc/kernels umma_rate.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "tc_common.cuh"
using namespace petra::tc;

// mode 0: lane-0-only loop (as the library kernels); mode 1: warp-uniform loop, elect.sync per MMA;
// mode 2: mode 1 with the loop unrolled by 4 (compile-time descriptor offsets)
template <int N, int MODE>
__global__ void __launch_bounds__(128, 1) bench(int iters, int naccum, int shift_rows, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if ((MODE == 0 && threadIdx.x == 0) || (MODE > 0 && threadIdx.x < 32)) {
    constexpr uint32_t idesc = idesc_bf16(128, N, 0, 0);
    const uint32_t a0 = smem_u32(smem) + shift_rows * 128, b0 = smem_u32(smem + 48 * 1024);
    const uint64_t ad = sw128_desc(a0, 16, 1024), bd = sw128_desc(b0, 16, 1024);
    // warm-up
    auto issue = [&](int i) {
      if (MODE == 0) {
        umma_bf16(tmem + (i % naccum) * N, ad + 2 * (i & 3), bd + 2 * (i & 3), idesc, 1u);
      } else {
        if (petra::tc::elect_one()) umma_bf16(tmem + (i & (naccum - 1)) * N, ad + 2 * (i & 3), bd + 2 * (i & 3), idesc, 1u);
        __syncwarp();
      }
    };
    for (int i = 0; i < 64; ++i) issue(i);
    if (MODE == 0 || petra::tc::elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    const unsigned long long t0 = clock64();
    if (MODE == 2) {
      for (int i = 0; i < iters; i += 4) {
#pragma unroll
        for (int k = 0; k < 4; ++k) issue(i + k);
      }
    } else {
      for (int i = 0; i < iters; ++i) issue(i);
    }
    if (MODE == 0 || petra::tc::elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 1);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int N, int MODE>
void run(int naccum, int shift) {
  unsigned long long *d, h;
  cudaMalloc(&d, 8);
  const int smem = 100 * 1024;
  cudaFuncSetAttribute(bench<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  bench<N, MODE><<<148, 128, smem>>>(iters, naccum, shift, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("mode=%d N=%3d accum=%d shift_rows=%2d: %6.1f cycles/MMA (floor %d)  %s\n", MODE, N, naccum, shift, (double)h / iters,
         128 * N / 256, cudaGetErrorString(e));
  cudaFree(d);
}

int main(int argc, char **argv) {
  const int N = atoi(argv[1]), mode = atoi(argv[2]), na = atoi(argv[3]), sh = argc > 4 ? atoi(argv[4]) : 0;
  setvbuf(stdout, nullptr, _IONBF, 0);
  if (N == 64 && mode == 0) run<64, 0>(na, sh);
  if (N == 64 && mode == 1) run<64, 1>(na, sh);
  if (N == 64 && mode == 2) run<64, 2>(na, sh);
  if (N == 128 && mode == 1) run<128, 1>(na, sh);
  if (N == 128 && mode == 2) run<128, 2>(na, sh);
  if (N == 256 && mode == 1) run<256, 1>(na, sh);
  if (N == 256 && mode == 2) run<256, 2>(na, sh);
  return 0;
}

// TMA fill-rate microbenchmark (B200): bytes per clock per SM that one producer thread
// can stream into a shared-memory ring, by copy shape.  One CTA per SM; a consumer warp
// only waits for each stage and releases it (no compute), so the ring is drained as fast
// as it fills.  Sources cycle over a 64 MB region (L2-resident after the first pass).
//   mode 0: 2-D tiled box {64 bf16, R rows}, 128B swizzle (one 128-byte row per box row)
//   mode 1: 1-D cp.async.bulk of R*128 contiguous bytes (a pre-swizzled tile)
//   mode 2: 4-D box {64 ch, 8, 8, R/64 images} of a [B][8][8][C] bf16 tensor (im2col-like)
//   mode 3: R/128 1-D bulk copies of 16 KB each (several copies per stage)
// usage: tma_rate MODE R STAGES [GRID]
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstdint>

__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c));
}
__device__ __forceinline__ void expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t *b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                   su(b)),
               "r"(ph)
               : "memory");
}
__device__ __forceinline__ void tma2d(void *d, const CUtensorMap *m, uint64_t *b, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          su(d)),
      "l"((uint64_t)m), "r"(su(b)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma4d(void *d, const CUtensorMap *m, uint64_t *b, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(su(d)),
      "l"((uint64_t)m), "r"(su(b)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void bulk(void *d, const void *s, uint32_t bytes, uint64_t *b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(d)),
               "l"((uint64_t)s), "r"(bytes), "r"(su(b))
               : "memory");
}

constexpr size_t REGION = 64ull << 20;

__global__ void __launch_bounds__(64, 1) kern(const __grid_constant__ CUtensorMap m2, const __grid_constant__ CUtensorMap m4,
                                              const uint8_t *src, int mode, int R, int S, int iters,
                                              unsigned long long *cyc) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t *sm = (uint8_t *)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  const uint32_t SB = R * 128;
  uint64_t *full = (uint64_t *)(sm + S * SB), *empty = full + S;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long ntiles = REGION / SB;
  unsigned long long t0 = clock64();
  if (threadIdx.x == 0) {
    int st = 0; uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      wait(&empty[st], ph ^ 1);
      expect_tx(&full[st], SB);
      const long long tile = ((long long)blockIdx.x + (long long)i * gridDim.x) % ntiles;
      uint8_t *d = sm + st * SB;
      if (mode == 0) tma2d(d, &m2, &full[st], 0, (int)(tile * R));
      else if (mode == 1) bulk(d, src + tile * SB, SB, &full[st]);
      else if (mode == 2) tma4d(d, &m4, &full[st], 0, 0, 0, (int)(tile * (R / 64)));
      else for (int c = 0; c < R / 128; ++c) bulk(d + c * 16384, src + tile * SB + c * 16384, 16384, &full[st]);
      if (++st == S) { st = 0; ph ^= 1; }
    }
  } else if (threadIdx.x == 32) {
    int st = 0; uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      wait(&full[st], ph);
      arrive(&empty[st]);
      if (++st == S) { st = 0; ph ^= 1; }
    }
    cyc[blockIdx.x] = clock64() - t0;
  }
}

int main(int argc, char **argv) {
  int mode = atoi(argv[1]), R = atoi(argv[2]), S = atoi(argv[3]);
  int grid = argc > 4 ? atoi(argv[4]) : 148;
  uint8_t *src;
  cudaMalloc(&src, REGION);
  cudaMemset(src, 1, REGION);
  unsigned long long *cyc;
  cudaMalloc(&cyc, grid * 8);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
  CUtensorMap m2, m4;
  {
    cuuint64_t dims[2] = {64, REGION / 128}, st[1] = {128};
    cuuint32_t box[2] = {64, (cuuint32_t)R}, es[2] = {1, 1};
    if (R <= 256)
      enc(&m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    cuuint64_t dims[4] = {64, 8, 8, REGION / (64 * 128)}, st[3] = {128, 8 * 128, 64 * 128};
    cuuint32_t box[4] = {64, 8, 8, (cuuint32_t)(R / 64 > 0 ? R / 64 : 1)}, es[4] = {1, 1, 1, 1};
    enc(&m4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, src, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  size_t smem = 1024 + (size_t)S * R * 128 + 2 * S * 8 + 64;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int iters = 4000;
  kern<<<grid, 64, smem>>>(m2, m4, src, mode, R, S, 200, cyc);  // warm L2
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<grid, 64, smem>>>(m2, m4, src, mode, R, S, iters, cyc);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) { printf("mode %d R %d S %d: %s\n", mode, R, S, cudaGetErrorString(err)); return 1; }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long *h = new unsigned long long[grid];
  cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < grid; ++i) avg += h[i];
  avg /= grid;
  double bytes = (double)iters * R * 128;
  printf("mode %d rows %4d stages %d grid %3d: %6.1f B/clk/SM  %7.1f GB/s chip  (%.0f clk per %d B stage)\n", mode, R, S,
         grid, bytes / avg, bytes * grid / (ms * 1e6), avg / iters, R * 128);
  return 0;
}

// TMA burst microbenchmark (B200): cycles from issuing N copies back to back (one thread)
// until all N have landed, per copy shape -- do copies overlap in flight or serialise?
// One CTA per SM (grid G); each CTA repeats the burst `reps` times on different sources
// (64 MB region, L2-resident after a warm-up pass) and reports the median burst cycles.
//   kind 0: 2-D tiled boxes {64 bf16, R rows}, 128B swizzle
//   kind 1: 1-D cp.async.bulk of R*128 bytes
// bars 0: one mbarrier per copy; 1: all copies on one mbarrier
// usage: tma_burst KIND R N BARS [GRID]
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c));
}
__device__ __forceinline__ void expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(bytes) : "memory");
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
__device__ __forceinline__ void bulk(void *d, const void *s, uint32_t bytes, uint64_t *b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(d)),
               "l"((uint64_t)s), "r"(bytes), "r"(su(b))
               : "memory");
}

constexpr size_t REGION = 64ull << 20;

__global__ void __launch_bounds__(32, 1) kern(const __grid_constant__ CUtensorMap m2, const uint8_t *src, int kind,
                                              int R, int N, int bars, int reps, unsigned *cyc) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t *sm = (uint8_t *)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  const uint32_t SB = R * 128;
  __shared__ uint64_t bar[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  const long long ntiles = REGION / SB;
  uint32_t ph = 0;
  for (int r = 0; r < reps; ++r) {
    const long long t0 = clock64();
    if (bars) expect_tx(&bar[0], SB * N);
    for (int i = 0; i < N; ++i) {
      uint64_t *b = bars ? &bar[0] : &bar[i];
      if (!bars) expect_tx(b, SB);
      const long long tile = ((long long)blockIdx.x * 977 + (long long)r * 131 + i * 7) % ntiles;
      if (kind == 0) tma2d(sm + i * SB, &m2, b, 0, (int)(tile * R));
      else bulk(sm + i * SB, src + tile * SB, SB, b);
    }
    for (int i = 0; i < (bars ? 1 : N); ++i) wait(&bar[i], ph);
    ph ^= 1;
    const long long t1 = clock64();
    cyc[(size_t)blockIdx.x * reps + r] = (unsigned)(t1 - t0);
  }
}

int main(int argc, char **argv) {
  int kind = atoi(argv[1]), R = atoi(argv[2]), N = atoi(argv[3]), bars = atoi(argv[4]);
  int grid = argc > 5 ? atoi(argv[5]) : 148;
  const int reps = 64;
  uint8_t *src;
  cudaMalloc(&src, REGION);
  cudaMemset(src, 1, REGION);
  unsigned *cyc;
  cudaMalloc(&cyc, (size_t)grid * reps * 4);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
  CUtensorMap m2;
  cuuint64_t dims[2] = {64, REGION / 128}, st[1] = {128};
  cuuint32_t box[2] = {64, (cuuint32_t)std::min(R, 256)}, es[2] = {1, 1};
  enc(&m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  size_t smem = 1024 + (size_t)N * R * 128;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int pass = 0; pass < 2; ++pass) kern<<<grid, 32, smem>>>(m2, src, kind, R, N, bars, reps, cyc);  // warm
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) { printf("kind %d R %d N %d: %s\n", kind, R, N, cudaGetErrorString(err)); return 1; }
  std::vector<unsigned> h((size_t)grid * reps);
  cudaMemcpy(h.data(), cyc, h.size() * 4, cudaMemcpyDeviceToHost);
  std::sort(h.begin(), h.end());
  const double med = h[h.size() / 2];
  printf("kind %d rows %3d N %2d bars %d grid %3d: burst %6.0f clk (p10 %5u p90 %5u)  %6.1f B/clk  %5.0f clk/copy\n",
         kind, R, N, bars, grid, med, h[h.size() / 10], h[h.size() * 9 / 10], (double)N * R * 128 / med, med / N);
  return 0;
}

// Multi-block TMA boxes (B200): can ONE copy fetch KG 64-channel blocks of a K-major bf16
// matrix as KG consecutive 128B-swizzled [rows][64] slabs (the layout UMMA reads), through a
// tensor map whose outermost dimension is the channel block (stride 128 B, i.e. global
// strides not increasing)?  Checks the landed bytes against the host and times bursts.
//   usage: tma_multiblock
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void kern(const __grid_constant__ CUtensorMap m, int rank, int kg, int rows, uint16_t *out, int reps,
                     unsigned *cyc) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t *sm = (uint8_t *)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t bytes = (uint32_t)kg * rows * 128;
  if (threadIdx.x == 0) {
    uint32_t ph = 0;
    for (int r = 0; r < reps; ++r) {
      const long long t0 = clock64();
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(bytes) : "memory");
      if (rank == 3)
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
            "[%2];" ::"r"(su(sm)),
            "l"((uint64_t)&m), "r"(su(&bar)), "r"(0), "r"(0), "r"(0)
            : "memory");
      else
        asm volatile(
            "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, "
            "%7}], [%2];" ::"r"(su(sm)),
            "l"((uint64_t)&m), "r"(su(&bar)), "r"(0), "r"(0), "r"(0), "r"(0), "r"(0)
            : "memory");
      asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                       su(&bar)),
                   "r"(ph)
                   : "memory");
      ph ^= 1;
      cyc[r] = (unsigned)(clock64() - t0);
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < bytes / 2; i += blockDim.x) out[i] = reinterpret_cast<uint16_t *>(sm)[i];
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  // K-major weight matrix [R][K] bf16 with K = 512: value = (r * 1000 + k) & 0x7fff
  const int R = 256, K = 512;
  std::vector<uint16_t> h((size_t)R * K);
  for (int r = 0; r < R; ++r)
    for (int k = 0; k < K; ++k) h[(size_t)r * K + k] = (uint16_t)((r * 1000 + k) & 0x7fff);
  uint16_t *d, *out;
  cudaMalloc(&d, h.size() * 2);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  cudaMalloc(&out, 200 * 1024);
  unsigned *cyc;
  cudaMalloc(&cyc, 64 * 4);
  for (int kg : {1, 2, 4}) {
    for (int rows : {64, 128, 256}) {
      if (kg * rows * 128 > 160 * 1024) continue;
      // rank 3: {64 k, rows, K/64 blocks}, strides {K*2, 128}
      CUtensorMap m;
      cuuint64_t dims[3] = {64, (cuuint64_t)R, (cuuint64_t)K / 64}, st[2] = {(cuuint64_t)K * 2, 128};
      cuuint32_t box[3] = {64, (cuuint32_t)rows, (cuuint32_t)kg}, es[3] = {1, 1, 1};
      CUresult e = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, d, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (e != CUDA_SUCCESS) {
        printf("rank3 kg %d rows %d: encode failed (%d)\n", kg, rows, (int)e);
        continue;
      }
      const int reps = 32;
      kern<<<1, 128, 200 * 1024>>>(m, 3, kg, rows, out, reps, cyc);
      cudaError_t ce = cudaDeviceSynchronize();
      if (ce != cudaSuccess) {
        printf("rank3 kg %d rows %d: %s\n", kg, rows, cudaGetErrorString(ce));
        return 1;
      }
      std::vector<uint16_t> o((size_t)kg * rows * 64);
      cudaMemcpy(o.data(), out, o.size() * 2, cudaMemcpyDeviceToHost);
      // expected: slab g, row r, 16-byte chunk c stored at chunk c ^ (r & 7)
      long bad = 0;
      for (int g = 0; g < kg; ++g)
        for (int r = 0; r < rows; ++r)
          for (int c = 0; c < 8; ++c)
            for (int e8 = 0; e8 < 8; ++e8) {
              const uint16_t want = h[(size_t)r * K + g * 64 + c * 8 + e8];
              const uint16_t got = o[((size_t)g * rows + r) * 64 + ((c ^ (r & 7)) * 8) + e8];
              bad += want != got;
            }
      std::vector<unsigned> c(reps);
      cudaMemcpy(c.data(), cyc, reps * 4, cudaMemcpyDeviceToHost);
      unsigned best = c[1];
      for (int i = 1; i < reps; ++i) best = std::min(best, c[i]);
      printf("rank3 {64, rows, KB} box {64, %3d, %d}: %s (%ld mismatches), %u clk per copy of %d B\n", rows, kg,
             bad ? "WRONG" : "exact", bad, best, kg * rows * 128);
    }
  }
  return 0;
}

// umma_shift_probe.cu -- does a tcgen05 K-major SW128 operand accept a start address
// shifted by r 128-byte rows (not 1024-aligned), and what must the descriptor's
// base-offset field (bits 49-51) hold?  Experiment for the halo (shifted-window)
// convolution: A tile rows = padded pixels, tap (dh, dw) = a row shift.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2406_02052_b200/csrc/kernels
//        tools/umma_shift_probe.cu -o build/umma_shift_probe -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"

using namespace petra;

constexpr int ROWS = 256, NB = 64, K = 64;

__global__ void probe(const __nv_bfloat16 *A, const __nv_bfloat16 *B, float *D, int shift, int boff_mode) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = smem;                 // ROWS x 128 B
  uint8_t *sB = smem + ROWS * 128;    // NB x 128 B
  uint64_t *bar = reinterpret_cast<uint64_t *>(sB + NB * 128);
  uint32_t *slot = reinterpret_cast<uint32_t *>(bar + 1);
  const int t = threadIdx.x;
  // swizzled stores: 16-byte chunk c of row r at r*128 + ((c ^ (r & 7)) * 16)  (address-based)
  for (int i = t; i < ROWS * 8; i += blockDim.x) {
    int r = i >> 3, c = i & 7;
    *reinterpret_cast<uint4 *>(sA + r * 128 + ((c ^ (r & 7)) << 4)) = reinterpret_cast<const uint4 *>(A)[i];
  }
  for (int i = t; i < NB * 8; i += blockDim.x) {
    int r = i >> 3, c = i & 7;
    *reinterpret_cast<uint4 *>(sB + r * 128 + ((c ^ (r & 7)) << 4)) = reinterpret_cast<const uint4 *>(B)[i];
  }
  tc::fence_proxy_async_smem();
  if (t == 0) {
    tc::mbar_init(bar, 1);
    tc::fence_mbar_init();
  }
  if (t < 32) tc::tmem_alloc(slot, 64);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tm = *slot;
  if (t == 0) {
    const uint32_t a0 = tc::smem_u32(sA) + shift * 128;
    uint64_t ad = tc::sw128_desc(a0, 16, 1024);
    if (boff_mode == 1) ad |= (uint64_t)((a0 >> 7) & 7) << 49;
    const uint64_t bd = tc::sw128_desc(tc::smem_u32(sB), 16, 1024);
    constexpr uint32_t idesc = tc::idesc_bf16(128, NB, 0, 0);
    for (int k = 0; k < 4; ++k) tc::umma_bf16(tm, ad + 2 * k, bd + 2 * k, idesc, k > 0 ? 1u : 0u);
    tc::umma_commit(bar);
  }
  __syncwarp();
  tc::mbar_wait(bar, 0);
  tc::tc_fence_after();
  if (t < 128) {
    const int q = t >> 5, lane = t & 31;
    for (int c = 0; c < NB; c += 16) {
      float v[16];
      tc::tmem_ld16(tm + ((uint32_t)(q * 32) << 16) + c, v);
      for (int j = 0; j < 16; ++j) D[(q * 32 + lane) * NB + c + j] = v[j];
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (t < 32) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tm, 64);
  }
}

int main() {
  std::vector<__nv_bfloat16> hA(ROWS * K), hB(NB * K);
  std::vector<float> fA(ROWS * K), fB(NB * K);
  srand(1);
  for (int i = 0; i < ROWS * K; ++i) {
    float v = (float)(rand() % 17 - 8);
    hA[i] = __float2bfloat16(v);
    fA[i] = v;
  }
  for (int i = 0; i < NB * K; ++i) {
    float v = (float)(rand() % 9 - 4);
    hB[i] = __float2bfloat16(v);
    fB[i] = v;
  }
  __nv_bfloat16 *dA, *dB;
  float *dD;
  cudaMalloc(&dA, ROWS * K * 2);
  cudaMalloc(&dB, NB * K * 2);
  cudaMalloc(&dD, 128 * NB * 4);
  cudaMemcpy(dA, hA.data(), ROWS * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), NB * K * 2, cudaMemcpyHostToDevice);
  const int smem = 1024 + ROWS * 128 + NB * 128 + 64;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::vector<float> hD(128 * NB);
  for (int mode = 0; mode < 2; ++mode)
    for (int shift : {0, 1, 2, 3, 5, 7, 8, 9, 13, 34, 35, 100}) {
      probe<<<1, 128, smem>>>(dA, dB, dD, shift, mode);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("mode %d shift %d: CUDA error %s\n", mode, shift, cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(hD.data(), dD, 128 * NB * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < NB; ++n) {
          float ref = 0;
          for (int k = 0; k < K; ++k) ref += fA[(m + shift) * K + k] * fB[n * K + k];
          if (ref != hD[m * NB + n]) ++bad;
        }
      printf("base_offset %s  shift %3d rows: %s (%d mismatches)\n", mode ? "=(addr>>7)&7" : "=0          ", shift,
             bad ? "WRONG" : "exact", bad);
    }
  return 0;
}

// stem_tc.cu -- tcgen05 convolutions for inputs with few channels (the stem).
//
// forward  z[m][co] = sum_{kk} A[m][kk] * w[co][kk],   kk = (kh*k + kw)*Ci + c,  K = k*k*Ci
// wgrad    dw[co][kk] = sum_m dz[m][co] * A[m][kk]
// with the implicit im2col A[m][kk] = bf16(x[b][s*ho+kh-p][s*wo+kw-p][c]) (0 outside).
//
// The TMA im2col boxes of conv_tc.cu need 64 channels per tap; a 3-channel image
// (the ImageNet 7x7/s2 stem, the CIFAR 3x3 stem) has 3.  Here the A operand is
// GATHERED from a bf16 copy of the image padded to 4 channels (8 bytes per pixel,
// image_to_bf16x4): the reduction index is laid out per kernel row as
// kk = kh*S + kw*4 + c (S = k*4 rounded up to a power of two; zero weights on the
// padding slots), so every 4 consecutive kk are one pixel = one 8-byte load.  8
// producer warps build each 128 x 64 (fwd, K-major) or 64 x 128 (wgrad, MN-major)
// bf16 tile in the 128B-swizzled smem layout UMMA reads (an unchecked fast path for
// interior pixels), then publish it with fence.proxy.async + mbarrier.  No im2col
// tensor ever touches HBM.  The weights (fwd) sit in smem for the whole persistent CTA.
// Warp roles: 0-7 gather producers, 8-11 epilogue (TMEM lane quarters 0-3), 12 MMA.
#include <cudaTypedefs.h>

#include <mutex>

#include "../errors.h"
#include "../kernels.h"
#include "tc_common.cuh"

namespace petra {
namespace {

constexpr int kStages = 4;
constexpr int kThreads = 13 * 32;
constexpr int kProducers = 256;
constexpr uint32_t kATile = 128 * 64 * 2;  // 16 KB
constexpr int kMaxKK = 256;

struct StemParams {
  const uint2 *xq;  // [B][H][W] x 4 bf16 (the image, channels zero-padded to 4)
  const float *w;   // [Co][k][k][Ci] fp32 (forward)
  int B, H, W, Ci, k, s, p, Ho, Wo;
  int M, K, N;                         // K = k*k*Ci (the weight layout)
  int S, shS, Kp;                      // padded reduction: kk = kh*S + kw*4 + c, Kp = k*S
  int KB;                              // forward: 64-wide blocks of Kp
  int n_mt, KBtot, kb_per_split, splits;  // wgrad: kk tiles of 128, pixel blocks of 64, split-K
  void *out;                           // fwd: z fp32 or bf16 (OUT16); wgrad: fp32
  float *stats;
};

struct Pixel {
  int64_t base;  // pixel index of the receptive-field corner (b, hi0, wi0)
  int hi0, wi0;
  bool valid, interior;
};

__device__ __forceinline__ Pixel pixel(const StemParams &P, int m) {
  Pixel q{0, 0, 0, m < P.M, false};
  if (!q.valid) return q;
  const int hw = P.Ho * P.Wo;
  const int b = m / hw, r = m % hw, ho = r / P.Wo, wo = r % P.Wo;
  q.hi0 = ho * P.s - P.p;
  q.wi0 = wo * P.s - P.p;
  q.interior = q.hi0 >= 0 && q.wi0 >= 0 && q.hi0 + P.k <= P.H && q.wi0 + P.k <= P.W;
  q.base = ((int64_t)b * P.H + q.hi0) * P.W + q.wi0;
  return q;
}

// kk -> weight index (kh*k + kw)*Ci + c, or -1 on a padding slot
__device__ __forceinline__ int real_kk(const StemParams &P, int kk) {
  const int kh = kk >> P.shS, j = kk & (P.S - 1), kw = j >> 2, c = j & 3;
  return (kh < P.k && kw < P.k && c < P.Ci) ? (kh * P.k + kw) * P.Ci + c : -1;
}

// 32 consecutive kk of one output pixel = 8 pixels of the 4-channel image: 8-byte loads
__device__ __forceinline__ void gather32(const StemParams &P, int kk0, const Pixel &q, uint32_t (&pk)[16]) {
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const int kk = kk0 + 4 * g;
    const int kh = kk >> P.shS, kw = (kk & (P.S - 1)) >> 2;
    uint2 u = make_uint2(0u, 0u);
    if (q.valid && kh < P.k && kw < P.k) {
      const int hi = q.hi0 + kh, wi = q.wi0 + kw;
      if (q.interior || (hi >= 0 && hi < P.H && wi >= 0 && wi < P.W)) u = __ldg(P.xq + q.base + kh * P.W + kw);
    }
    pk[2 * g] = u.x;
    pk[2 * g + 1] = u.y;
  }
}

// four 16-byte chunks (chunk index c0..c0+3) of row `row` of a 128B-swizzled tile
__device__ __forceinline__ void store_row_chunks(uint8_t *tile, int row, int c0, const uint32_t (&pk)[16]) {
  uint8_t *dst = tile + (row >> 3) * 1024 + (row & 7) * 128;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    *reinterpret_cast<uint4 *>(dst + (((c0 + i) ^ (row & 7)) << 4)) =
        make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
}

template <int BN, bool OUT16>
__global__ void __launch_bounds__(kThreads, 1) stem_fwd_kernel(const __grid_constant__ StemParams P) {
  pdl_wait_trigger();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = smem;
  uint8_t *sB = smem + kStages * kATile;  // [KB][BN rows x 128 B], resident
  uint64_t *full = reinterpret_cast<uint64_t *>(sB + (size_t)P.KB * BN * 128);
  uint64_t *empty = full + kStages;
  uint64_t *tfull = empty + kStages;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
  float *sstat = reinterpret_cast<float *>(tmem_slot + 4);  // [4 quarters][N][3] (shift k, S, Q), then [4][N][2]
  int *scnt = reinterpret_cast<int *>(sstat + 4 * 3 * P.N);  // [4 quarters] valid rows

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles = (int)cdiv(P.M, 128);
  // weights fp32 [Co][K] -> bf16 K-major swizzled tiles in the padded kk order
  const int kchunks = P.KB * 8;
  for (int i = threadIdx.x; i < BN * kchunks; i += blockDim.x) {
    const int n = i / kchunks, r = i % kchunks, kb = r >> 3, c = r & 7;
    uint32_t pk[4];
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      const int kk = kb * 64 + c * 8 + e;
      const int r0 = real_kk(P, kk), r1 = real_kk(P, kk + 1);
      const float v0 = r0 >= 0 ? P.w[(int64_t)n * P.K + r0] : 0.f;
      const float v1 = r1 >= 0 ? P.w[(int64_t)n * P.K + r1] : 0.f;
      __nv_bfloat162 h = __floats2bfloat162_rn(v0, v1);
      pk[e >> 1] = *reinterpret_cast<uint32_t *>(&h);
    }
    uint8_t *dst = sB + (size_t)kb * BN * 128 + (n >> 3) * 1024 + (n & 7) * 128 + ((c ^ (n & 7)) << 4);
    *reinterpret_cast<uint4 *>(dst) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
  }
  tc::fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full[s], kProducers);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 4);
    }
    tc::fence_mbar_init();
  }
  if (warp == 12) tc::tmem_alloc(tmem_slot, 2 * BN);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < 8) {  // ---------------- gather producers: thread -> (row, half of the 64 kk)
    const int row = threadIdx.x & 127, half = threadIdx.x >> 7;
    int stage = 0;
    uint32_t phase = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const Pixel q = pixel(P, t * 128 + row);
      for (int kb = 0; kb < P.KB; ++kb) {
        uint32_t pk[16];
        gather32(P, kb * 64 + half * 32, q, pk);  // loads in flight before the wait
        tc::mbar_wait_idle(&empty[stage], phase ^ 1);
        store_row_chunks(sA + stage * kATile, row, half * 4, pk);
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(&full[stage]);
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 12) {  // ---------------- MMA issuer: warp-uniform loop, elected lane issues
    constexpr uint32_t idesc = tc::idesc_bf16(128, BN, 0, 0);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
      const int acc = it & 1;
      tc::mbar_wait_idle(&tempty[acc], ((it >> 1) & 1) ^ 1);
      tc::tc_fence_after();
      const uint32_t dtm = tmem_base + acc * BN;
      for (int kb = 0; kb < P.KB; ++kb) {
        tc::mbar_wait(&full[stage], phase);
        tc::tc_fence_after();
        const uint64_t ad = tc::sw128_desc(tc::smem_u32(sA + stage * kATile), 16, 1024);
        const uint64_t bd = tc::sw128_desc(tc::smem_u32(sB + (size_t)kb * BN * 128), 16, 1024);
        if (tc::elect_one()) {
#pragma unroll
          for (int k = 0; k < 4; ++k) tc::umma_bf16(dtm, ad + 2 * k, bd + 2 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
          tc::umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
      if (tc::elect_one()) tc::umma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else {  // ---------------- epilogue warps 8..11
    const int q = warp & 3;
    const int row = q * 32 + lane;
    // shifted statistics per column of this quarter's rows (tc::ColStats, kept in smem
    // here: the lanes of a warp hold rows, colsum16 reduces them): k = mean of the first
    // tile with valid rows, S = sum (z - k), Q = sum (z - k)^2 over valid rows
    float *my_stat = sstat + (size_t)q * P.N * 3;
    if (P.stats)
      for (int i = lane; i < 3 * P.N; i += 32) my_stat[i] = 0.f;
    __syncwarp();
    int nrows = 0;
    int it = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
      const int acc = it & 1;
      tc::mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc::tc_fence_after();
      const int m = t * 128 + row;
      const bool valid = m < P.M;
      const int nvalid = __popc(__ballot_sync(0xffffffffu, valid));
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        float v[16];
        tc::tmem_ld16(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c, v);
        if (valid) {
          if constexpr (OUT16) {  // z stored in bf16; statistics of the stored values (reading c24)
            uint32_t w[8];
#pragma unroll
            for (int jj = 0; jj < 16; jj += 2) {
              __nv_bfloat162 h = __floats2bfloat162_rn(v[jj], v[jj + 1]);
              w[jj >> 1] = *reinterpret_cast<uint32_t *>(&h);
              const float2 f = __bfloat1622float2(h);
              v[jj] = f.x;
              v[jj + 1] = f.y;
            }
            uint4 *o = reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(P.out) + (int64_t)m * P.N + c);
            o[0] = make_uint4(w[0], w[1], w[2], w[3]);
            o[1] = make_uint4(w[4], w[5], w[6], w[7]);
          } else {
            float *orow = static_cast<float *>(P.out) + (int64_t)m * P.N + c;
#pragma unroll
            for (int jj = 0; jj < 16; jj += 4)
              *reinterpret_cast<float4 *>(orow + jj) = make_float4(v[jj], v[jj + 1], v[jj + 2], v[jj + 3]);
          }
        } else {
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) v[jj] = 0.f;
        }
        if (P.stats && nvalid > 0) {
          if (nrows == 0) {  // first tile: the shifts are the first valid row's values
            const int r0 = __ffs(__ballot_sync(0xffffffffu, valid)) - 1;
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) {
              const float k0 = __shfl_sync(0xffffffffu, v[jj], r0);
              if (lane == 0) my_stat[3 * (c + jj)] = k0;
            }
            __syncwarp();
          }
          float d[16], sq[16];
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            d[jj] = valid ? v[jj] - my_stat[3 * (c + jj)] : 0.f;
            sq[jj] = d[jj] * d[jj];
          }
          tc::colsum16(d, lane);
          tc::colsum16(sq, lane);
          __syncwarp();
          if (!(lane & 1)) {
            const int col = c + (lane >> 1);
            my_stat[3 * col + 1] += d[0];
            my_stat[3 * col + 2] += sq[0];
          }
          __syncwarp();
        }
      }
      nrows += nvalid;
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
    }
    if (P.stats) {  // this CTA's partial row: the 4 quarters' (count, mean, M2) merged (Chan) in order
      const float inv = nrows > 0 ? 1.f / (float)nrows : 0.f;
      float mu[8], m2[8];  // this warp's quarter, columns lane, lane + 32, ... (N <= 256)
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int col = lane + 32 * r;
        if (col < P.N) {
          const float k = my_stat[3 * col], S = my_stat[3 * col + 1], Q = my_stat[3 * col + 2];
          mu[r] = nrows > 0 ? k + S * inv : 0.f;
          m2[r] = nrows > 0 ? fmaxf(fmaf(-S * inv, S, Q), 0.f) : 0.f;
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");  // every quarter has read its (k, S, Q)
      float *fin = sstat;  // reuse as [4][N][2] (mean, M2)
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int col = lane + 32 * r;
        if (col < P.N) {
          fin[(q * P.N + col) * 2] = mu[r];
          fin[(q * P.N + col) * 2 + 1] = m2[r];
        }
      }
      if (lane == 0) scnt[q] = nrows;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      tc::cta_stats_row(fin, scnt, P.N, q * 32 + lane, 128, P.stats + (size_t)blockIdx.x * P.N * 2,
                        P.stats + (size_t)gridDim.x * P.N * 2 + blockIdx.x);
    }
  }
  __syncthreads();
  if (warp == 12) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem_base, 2 * BN);
  }
}

// wgrad: D[kk][co] = sum_pixels A[pixel][kk] dz[pixel][co]; M side = kk (tiles of 128),
// N side = co, K = pixels (blocks of 64, split over CTAs).  A and B are MN-major:
// A = two 64-kk blocks of [64 pixel rows x 128 B] gathered, B = BN/64 TMA boxes of dz.
template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
stem_wgrad_kernel(const __grid_constant__ CUtensorMap tmDZ, const __grid_constant__ StemParams P) {
  pdl_wait_trigger();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr uint32_t B_BYTES = BN * 64 * 2;
  constexpr uint32_t STAGE_BYTES = kATile + B_BYTES;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kStages * STAGE_BYTES);
  uint64_t *empty = full + kStages;
  uint64_t *tfull = empty + kStages;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_work = P.n_mt * P.splits;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full[s], kProducers + 1);  // + the expect_tx arrival of the dz TMA
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 4);
    }
    tc::fence_mbar_init();
    tc::tma_prefetch(&tmDZ);
  }
  if (warp == 12) tc::tmem_alloc(tmem_slot, 2 * BN);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < 8) {
    const int r = threadIdx.x & 63, qq = threadIdx.x >> 6, j = qq >> 1, half = qq & 1;
    int stage = 0;
    uint32_t phase = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
      const int sp = w % P.splits, mt = w / P.splits;
      const int kb0 = sp * P.kb_per_split, kb1 = min(P.KBtot, kb0 + P.kb_per_split);
      const int kk0 = mt * 128 + j * 64 + half * 32;
      for (int kb = kb0; kb < kb1; ++kb) {
        const Pixel q = pixel(P, kb * 64 + r);
        uint32_t pk[16];
        gather32(P, kk0, q, pk);
        tc::mbar_wait_idle(&empty[stage], phase ^ 1);
        uint8_t *sa = smem + stage * STAGE_BYTES;
        if (threadIdx.x == 0) {
          tc::mbar_arrive_expect_tx(&full[stage], B_BYTES);
          for (int nb = 0; nb < BN / 64; ++nb)
            tc::tma_load_2d(sa + kATile + nb * 8192, &tmDZ, &full[stage], nb * 64, kb * 64);
        }
        store_row_chunks(sa + j * 8192, r, half * 4, pk);
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(&full[stage]);
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 12) {  // MMA issuer: warp-uniform loop, elected lane issues
    constexpr uint32_t idesc = tc::idesc_bf16(128, BN, 1, 1);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++it) {
      const int sp = w % P.splits;
      const int kb0 = sp * P.kb_per_split, kb1 = min(P.KBtot, kb0 + P.kb_per_split);
      const int acc = it & 1;
      tc::mbar_wait_idle(&tempty[acc], ((it >> 1) & 1) ^ 1);
      tc::tc_fence_after();
      const uint32_t dtm = tmem_base + acc * BN;
      for (int kb = kb0; kb < kb1; ++kb) {
        tc::mbar_wait(&full[stage], phase);
        tc::tc_fence_after();
        const uint32_t sa = tc::smem_u32(smem + stage * STAGE_BYTES);
        const uint64_t ad = tc::sw128_desc(sa, 8192, 1024);
        const uint64_t bd = tc::sw128_desc(sa + kATile, 8192, 1024);
        if (tc::elect_one()) {
#pragma unroll
          for (int k = 0; k < 4; ++k)  // 16 pixels = 16 rows x 128 B per step
            tc::umma_bf16(dtm, ad + (uint64_t)(k * 2048 >> 4), bd + (uint64_t)(k * 2048 >> 4), idesc,
                          (kb > kb0 || k) ? 1u : 0u);
          tc::umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
      if (tc::elect_one()) tc::umma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else {
    const int q = warp & 3;
    const int row = q * 32 + lane;
    int it = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++it) {
      const int sp = w % P.splits, mt = w / P.splits;
      const int acc = it & 1;
      tc::mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc::tc_fence_after();
      const int kk = mt * 128 + row;
      const int r = kk < P.Kp ? real_kk(P, kk) : -1;  // padding slots of kk carry no weight
      float *o = static_cast<float *>(P.out) + (int64_t)sp * P.N * P.K;
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        float v[16];
        tc::tmem_ld16(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c, v);
        if (r >= 0) {
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) o[(int64_t)(c + jj) * P.K + r] = v[jj];
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 12) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem_base, 2 * BN);
  }
}

// ------------------------------------------------------------------ host side
StemParams base_params(const ConvGeom &g) {
  StemParams P{};
  P.B = g.B; P.H = g.H; P.W = g.W; P.Ci = g.Ci; P.k = g.k; P.s = g.s; P.p = g.p; P.Ho = g.Ho; P.Wo = g.Wo;
  P.M = (int)g.M();
  P.K = g.K();
  P.N = g.Co;
  P.S = 4;
  P.shS = 2;
  while (P.S < 4 * g.k) {
    P.S <<= 1;
    ++P.shS;
  }
  P.Kp = g.k * P.S;
  P.KB = (int)cdiv(P.Kp, 64);
  return P;
}

int padded_k(const ConvGeom &g) { return base_params(g).Kp; }

__global__ void image_to_bf16x4_kernel(const float *__restrict__ x, uint2 *__restrict__ xq, int64_t pixels, int C) {
  pdl_wait_trigger();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pixels; i += (int64_t)gridDim.x * blockDim.x) {
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    for (int c = 0; c < C; ++c) v[c] = x[i * C + c];
    __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]), b = __floats2bfloat162_rn(v[2], v[3]);
    xq[i] = make_uint2(*reinterpret_cast<uint32_t *>(&a), *reinterpret_cast<uint32_t *>(&b));
  }
}

size_t fwd_smem(int BN, int KB) {
  return 1024 + (size_t)kStages * kATile + (size_t)KB * BN * 128 + 256 + (size_t)4 * BN * 3 * 4 + 16;
}
size_t wgrad_smem(int BN) { return 1024 + (size_t)kStages * (kATile + BN * 128) + 256; }

struct WPlan {
  int n_mt, KBtot, kb_per_split, splits;
};
WPlan wplan(const ConvGeom &g) {
  WPlan w{};
  w.n_mt = (int)cdiv(padded_k(g), 128);
  w.KBtot = (int)cdiv(g.M(), 64);
  static const int wctas = std::max(1, std::min(kNumSMs, env_int("PETRA_STEM_WGRAD_CTAS", kNumSMs)));
  const int want = std::max(1, std::min(w.KBtot, (int)cdiv(wctas, w.n_mt)));
  w.kb_per_split = (int)cdiv(w.KBtot, want);
  w.splits = (int)cdiv(w.KBtot, w.kb_per_split);
  return w;
}

}  // namespace

void stem_tc_prepare() {
  static std::once_flag once;
  std::call_once(once, [] {
    auto set = [](const void *f, size_t smem) {
      PETRA_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    };
    set((const void *)stem_fwd_kernel<64, false>, fwd_smem(64, 4));
    set((const void *)stem_fwd_kernel<128, false>, fwd_smem(128, 4));
    set((const void *)stem_fwd_kernel<256, false>, fwd_smem(256, 4));
    set((const void *)stem_fwd_kernel<64, true>, fwd_smem(64, 4));
    set((const void *)stem_fwd_kernel<128, true>, fwd_smem(128, 4));
    set((const void *)stem_fwd_kernel<256, true>, fwd_smem(256, 4));
    set((const void *)stem_wgrad_kernel<64>, wgrad_smem(64));
    set((const void *)stem_wgrad_kernel<128>, wgrad_smem(128));
    set((const void *)stem_wgrad_kernel<256>, wgrad_smem(256));
  });
}

bool stem_tc_supported(const ConvGeom &g) {
  return g.Ci >= 1 && g.Ci <= 4 && g.k <= 8 && padded_k(g) <= kMaxKK && (g.Co == 64 || g.Co == 128 || g.Co == 256) &&
         g.M() < ((int64_t)1 << 31) && g.Min() < ((int64_t)1 << 31);
}

size_t stem_operand_elems(const ConvGeom &g) { return (size_t)g.Min() * 4; }

void image_to_bf16x4(const float *x, __nv_bfloat16 *xq, const ConvGeom &g, cudaStream_t st) {
  const int64_t pix = g.Min();
  launch_k(image_to_bf16x4_kernel, (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(pix, 256), 8 * kNumSMs)),
           256, 0, st, x, reinterpret_cast<uint2 *>(xq), pix, g.Ci);
  PETRA_LAUNCH_CHECK();
}

size_t stem_tc_workspace(const ConvGeom &g) {
  if (!stem_tc_supported(g)) return 0;
  WPlan w = wplan(g);
  return w.splits > 1 ? (size_t)w.splits * g.Co * g.K() * sizeof(float) : 0;
}

StatsRows stem_fwd_tc(const ConvGeom &g, const __nv_bfloat16 *xq, const float *w, void *z, bool z_bf16,
                      float *stats_part, cudaStream_t st) {
  if (!stem_tc_supported(g)) throw PetraError(PETRA_E_UNSUPPORTED, "stem_fwd_tc: geometry");
  stem_tc_prepare();
  StemParams P = base_params(g);
  P.xq = reinterpret_cast<const uint2 *>(xq);
  P.w = w;
  P.out = z;
  P.stats = stats_part;
  static const int fctas = std::max(1, std::min(kNumSMs, env_int("PETRA_STEM_CTAS", kNumSMs)));
  const int grid = (int)std::min<int64_t>(cdiv(P.M, 128), fctas);
  const size_t smem = fwd_smem(P.N, P.KB);
  if (z_bf16) {
    if (P.N == 64) launch_k(stem_fwd_kernel<64, true>, grid, kThreads, smem, st, P);
    else if (P.N == 128) launch_k(stem_fwd_kernel<128, true>, grid, kThreads, smem, st, P);
    else launch_k(stem_fwd_kernel<256, true>, grid, kThreads, smem, st, P);
  } else {
    if (P.N == 64) launch_k(stem_fwd_kernel<64, false>, grid, kThreads, smem, st, P);
    else if (P.N == 128) launch_k(stem_fwd_kernel<128, false>, grid, kThreads, smem, st, P);
    else launch_k(stem_fwd_kernel<256, false>, grid, kThreads, smem, st, P);
  }
  PETRA_LAUNCH_CHECK();
  StatsRows r;
  r.rows = stats_part ? grid : 0;  // one N tile (BN = Co): every CTA writes all columns
  return r;
}

void stem_wgrad_tc(const ConvGeom &g, const __nv_bfloat16 *dz, const __nv_bfloat16 *xq, float *dw, float *ws,
                   cudaStream_t st) {
  if (!stem_tc_supported(g)) throw PetraError(PETRA_E_UNSUPPORTED, "stem_wgrad_tc: geometry");
  stem_tc_prepare();
  StemParams P = base_params(g);
  WPlan wp = wplan(g);
  P.xq = reinterpret_cast<const uint2 *>(xq);
  P.n_mt = wp.n_mt;
  P.KBtot = wp.KBtot;
  P.kb_per_split = wp.kb_per_split;
  P.splits = wp.splits;
  if (wp.splits > 1 && !ws) throw PetraError(PETRA_E_ARG, "stem_wgrad_tc: workspace required");
  P.out = wp.splits > 1 ? ws : dw;
  CUtensorMap tdz = kmajor_map_bf16(dz, P.M, P.N, 64);  // dz [pixels][Co], box (64 ch, 64 pixels)
  const int grid = std::min(wp.n_mt * wp.splits, kNumSMs);
  const size_t smem = wgrad_smem(P.N);
  if (P.N == 64) launch_k(stem_wgrad_kernel<64>, grid, kThreads, smem, st, tdz, P);
  else if (P.N == 128) launch_k(stem_wgrad_kernel<128>, grid, kThreads, smem, st, tdz, P);
  else launch_k(stem_wgrad_kernel<256>, grid, kThreads, smem, st, tdz, P);
  PETRA_LAUNCH_CHECK();
  if (wp.splits > 1) splitk_sum(ws, wp.splits, (int64_t)g.Co * g.K(), dw, st);
}

}  // namespace petra

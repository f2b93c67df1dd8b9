// opt_tail.cu -- immediate Nesterov-SGD update, classifier tail, max-pool, small helpers.
//
// update  (reading c11):  g = Delta + lambda*theta (lambda = 0 on
//          BN parameters and biases), v <- mu*v + g, theta <- theta - lr*(g + mu*v).
//          One launch over every tensor of the stage (segment table); it also
//          refreshes the bf16 shadows of the conv weights used by the tensor-core
//          path ([Co][K] and the flipped/transposed dgrad operand) -- a shadow of
//          the single live parameter version, not a stash.
// tail: GAP over H,W of concat(x1,x2), Linear + bias,
//          batch-mean softmax cross-entropy, its VJP; deterministic reductions.
// maxpool 3x3/s2/p1 with first-index ties.
#include <cmath>

#include "../kernels.h"

namespace petra {
namespace {

// One launch over the whole stage: a work item is a 32(co) x 32(ci) tile of one tap of a
// conv weight with bf16 shadows, or a run of up to 1024 elements of any other tensor
// (kernels.h SgdChunk, built once per stage); blocks stride over the items, so small
// tensors (BN gamma / beta, biases) cost one item instead of a grid row of idle blocks.
__global__ void __launch_bounds__(256) sgd_kernel(const SgdSeg *__restrict__ segs, const SgdChunk *__restrict__ chunks,
                                                  int nchunks, float *__restrict__ theta, float *__restrict__ v,
                                                  const float *__restrict__ grad, float *__restrict__ acc, float inv_k,
                                                  int mode, const float *__restrict__ lr_dev, float mom, float wd,
                                                  int nesterov, int shadow_only, int *__restrict__ nonfinite) {
  pdl_wait_trigger();
  // mode (Alg. 1 lines 19-22):  SGD_PLAIN   k = 1, update with Delta;
  // SGD_ACCUMULATE  acc += Delta/k, no update;  SGD_ACC_UPDATE  update with acc + Delta/k, acc = 0
  const float lr_all = shadow_only ? 0.f : *lr_dev;  // device-resident: graph replays read the tick's lr
  __shared__ __nv_bfloat16 tile[32][33];
  for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const SgdChunk ch = chunks[c];
    const SgdSeg sg = segs[ch.seg];
    if (shadow_only && !sg.w_bf16) continue;  // block-uniform
    const float lam = sg.decay ? wd : 0.f;
    const float lr = lr_all;
    // theta[o] after this tick's update (or unchanged for shadow_only)
    auto update = [&](int64_t o) -> float {
      float th = theta[o];
      if (shadow_only) return th;
      float d = grad[o];
      if (!isfinite(d)) atomicOr(nonfinite, 2);  // latched (bit 1: Delta); reported by petra_stage_get_params
      if (mode == SGD_ACC_UPDATE) {
        d = fmaf(d, inv_k, acc[o]);
        acc[o] = 0.f;
      }
      const float g = fmaf(lam, th, d);
      const float vv = fmaf(mom, v[o], g);
      v[o] = vv;
      th -= lr * (nesterov ? fmaf(mom, vv, g) : vv);
      theta[o] = th;
      return th;
    };
    auto accumulate = [&](int64_t o) {  // Delta_j += Delta / k; theta (and its shadows) unchanged
      const float d = grad[o];
      if (!isfinite(d)) atomicOr(nonfinite, 2);
      acc[o] += d * inv_k;
    };
    if (sg.wt_bf16) {
      // conv weight [Co][kh][kw][Ci], tile ch.lo = (tap, co block, ci block): theta, v and
      // the bf16 copy w_bf16 (same order) are read / written along ci, the dgrad operand
      // wT[ci][tap'][co] = w[co][tap][ci] (tap' = k*k-1-tap, flipped) along co through a
      // shared-memory transpose -- every global access coalesced
      const int taps = sg.k * sg.k;
      const int nco = (sg.co + 31) / 32, nci = (sg.ci + 31) / 32;
      const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
      const int t = (int)ch.lo;
      const int cib = t % nci, r = t / nci, cob = r % nco, tap = r / nco;
      const int ci = cib * 32 + tx;
      if (mode == SGD_ACCUMULATE) {  // block-uniform
#pragma unroll
        for (int rr = ty; rr < 32; rr += 8) {
          const int co = cob * 32 + rr;
          if (co < sg.co && ci < sg.ci) accumulate(sg.offset + ((int64_t)co * taps + tap) * sg.ci + ci);
        }
        continue;
      }
#pragma unroll
      for (int rr = ty; rr < 32; rr += 8) {
        const int co = cob * 32 + rr;
        if (co < sg.co && ci < sg.ci) {
          const int64_t i = ((int64_t)co * taps + tap) * sg.ci + ci;
          const __nv_bfloat16 hb = __float2bfloat16_rn(update(sg.offset + i));
          sg.w_bf16[i] = hb;
          tile[rr][tx] = hb;
        }
      }
      __syncthreads();
      const int co = cob * 32 + tx;
#pragma unroll
      for (int rr = ty; rr < 32; rr += 8) {
        const int cj = cib * 32 + rr;
        if (co < sg.co && cj < sg.ci) sg.wt_bf16[((int64_t)cj * taps + (taps - 1 - tap)) * sg.co + co] = tile[tx][rr];
      }
      __syncthreads();
      continue;
    }
    for (int64_t i = ch.lo + threadIdx.x; i < ch.hi; i += blockDim.x) {
      if (mode == SGD_ACCUMULATE) {
        accumulate(sg.offset + i);
        continue;
      }
      const float th = update(sg.offset + i);
      if (sg.w_bf16) sg.w_bf16[i] = __float2bfloat16_rn(th);
    }
  }
}

__global__ void gap_kernel(const float *__restrict__ x1, const float *__restrict__ x2, int B, int HW, int C,
                           float *__restrict__ feat) {
  pdl_wait_trigger();
  // feat[b][c'] for c' in [0, 2C): mean over HW (fixed summation order)
  int b = blockIdx.y;
  int c2 = blockIdx.x * blockDim.x + threadIdx.x;
  if (c2 >= 2 * C) return;
  const float *src = c2 < C ? x1 : x2;
  int c = c2 < C ? c2 : c2 - C;
  float s = 0.f;
  for (int p = 0; p < HW; ++p) s += src[((int64_t)b * HW + p) * C + c];
  feat[(int64_t)b * 2 * C + c2] = s / (float)HW;
}

// Small fp32 GEMM of the classifier: C[m][n] = sum_k A(m, k) B(k, n) (+ bias[n]), with
// A(m, k) = A[m*sam + k*sak] and B(k, n) = B[k*sbk + n*sbn] (the transposes of the FC
// forward / weight gradient / input gradient).  16 x 32 output tiles, 128 threads of 2 x 2
// outputs, K in chunks of 32 through shared memory; blockIdx.z = a K split of kspan
// (partials to ws[z][M][N], summed in z order by fc_splitk_reduce: deterministic).  M =
// batch is small: small tiles and split K keep enough blocks resident to hide latency.
constexpr int GM = 16, GN = 32, GK = 32;
__global__ void __launch_bounds__(128) fc_gemm_kernel(const float *__restrict__ A, int64_t sam, int64_t sak,
                                                      const float *__restrict__ Bm, int64_t sbk, int64_t sbn,
                                                      const float *__restrict__ bias, int M, int N, int K,
                                                      int kspan, float *__restrict__ C) {
  pdl_wait_trigger();
  __shared__ float sa[GK][GM + 1], sb[GK][GN + 1];
  const int m0 = blockIdx.y * GM, n0 = blockIdx.x * GN;
  const int kbeg = blockIdx.z * kspan, kend = min(K, kbeg + kspan);
  C += (int64_t)blockIdx.z * M * N;
  if (gridDim.z > 1) bias = nullptr;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 8 threads: cols 2tx.., rows 2ty..
  float acc[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
  for (int k0 = kbeg; k0 < kend; k0 += GK) {
    // consecutive threads walk the operand's contiguous index (coalesced loads)
    for (int i = threadIdx.x; i < GK * GM; i += 128) {
      const bool kfast = sak == 1;
      const int kk = kfast ? i % GK : i / GM, mm = kfast ? i / GK : i % GM, m = m0 + mm, k = k0 + kk;
      sa[kk][mm] = (m < M && k < kend) ? A[m * sam + k * sak] : 0.f;
    }
    for (int i = threadIdx.x; i < GK * GN; i += 128) {
      const bool kfast = sbk == 1;
      const int kk = kfast ? i % GK : i / GN, nn = kfast ? i / GK : i % GN, n = n0 + nn, k = k0 + kk;
      sb[kk][nn] = (n < N && k < kend) ? Bm[k * sbk + n * sbn] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < GK; ++kk) {
      const float a0 = sa[kk][2 * ty], a1 = sa[kk][2 * ty + 1];
      const float b0 = sb[kk][2 * tx], b1 = sb[kk][2 * tx + 1];
      acc[0][0] = fmaf(a0, b0, acc[0][0]);
      acc[0][1] = fmaf(a0, b1, acc[0][1]);
      acc[1][0] = fmaf(a1, b0, acc[1][0]);
      acc[1][1] = fmaf(a1, b1, acc[1][1]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int m = m0 + 2 * ty + i, n = n0 + 2 * tx + j;
      if (m < M && n < N) C[(int64_t)m * N + n] = acc[i][j] + (bias ? bias[n] : 0.f);
    }
}

__global__ void fc_splitk_reduce_kernel(const float *__restrict__ ws, int splits, int64_t n, int N,
                                        const float *__restrict__ bias, float *__restrict__ C) {
  pdl_wait_trigger();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += ws[(int64_t)z * n + i];
    C[i] = s + (bias ? bias[i % N] : 0.f);
  }
}

// bias gradient: db[n] = sum_b dlogits[b][n]
__global__ void fc_bias_grad_kernel(const float *__restrict__ dlogits, int B, int N, float *__restrict__ db) {
  pdl_wait_trigger();
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  float s = 0.f;
  for (int b = 0; b < B; ++b) s += dlogits[(int64_t)b * N + n];
  db[n] = s;
}


__global__ void ce_kernel(const float *__restrict__ logits, const int32_t *__restrict__ labels, int B, int N,
                          float *__restrict__ dlogits, float *__restrict__ loss_row) {
  pdl_wait_trigger();
  // one block (256 threads) per row; dlogits = (softmax - onehot)/B
  __shared__ float red[32];
  int b = blockIdx.x;
  const float *l = logits + (int64_t)b * N;
  float mx = -INFINITY;
  for (int n = threadIdx.x; n < N; n += blockDim.x) mx = fmaxf(mx, l[n]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : -INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  mx = red[0];
  __syncthreads();
  float s = 0.f;
  for (int n = threadIdx.x; n < N; n += blockDim.x) s += expf(l[n] - mx);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  s = red[0];
  int y = labels[b];
  float lse = mx + logf(s);
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    float p = expf(l[n] - lse);
    dlogits[(int64_t)b * N + n] = (p - (n == y ? 1.f : 0.f)) / (float)B;
  }
  if (threadIdx.x == 0) loss_row[b] = lse - l[y];
}

__global__ void loss_mean_kernel(const float *__restrict__ loss_row, int B, float *__restrict__ loss,
                                 int *__restrict__ nonfinite) {
  pdl_wait_trigger();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < B; ++b) s += loss_row[b];
    float l = (float)(s / B);
    if (loss) *loss = l;
    if (!isfinite(l)) atomicOr(nonfinite, 1);  // latched (bit 0: loss)
  }
}



__global__ void gap_bwd_kernel(const float *__restrict__ dfeat, int B, int HW, int C, float *__restrict__ d1,
                               float *__restrict__ d2) {
  pdl_wait_trigger();
  int64_t n = (int64_t)B * HW * C;
  float inv = 1.f / (float)HW;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int c = (int)(i % C);
    int b = (int)(i / ((int64_t)HW * C));
    d1[i] = dfeat[(int64_t)b * 2 * C + c] * inv;
    d2[i] = dfeat[(int64_t)b * 2 * C + C + c] * inv;
  }
}

// max-pool on a [B][H][W][C] activation, writes split halves of the output
__global__ void maxpool_fwd_kernel(const float *__restrict__ a, int B, int H, int W, int C, int Ho, int Wo,
                                   float *__restrict__ o1, float *__restrict__ o2, uint8_t *__restrict__ arg) {
  pdl_wait_trigger();
  int64_t n = (int64_t)B * Ho * Wo * C;
  int Ch = C / 2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int c = (int)(i % C);
    int64_t r = i / C;
    int wo = (int)(r % Wo);
    r /= Wo;
    int ho = (int)(r % Ho);
    int b = (int)(r / Ho);
    float best = -INFINITY;
    int bi = 0;
    for (int kh = 0; kh < 3; ++kh)
      for (int kw = 0; kw < 3; ++kw) {
        int h = ho * 2 + kh - 1, w = wo * 2 + kw - 1;
        if (h < 0 || h >= H || w < 0 || w >= W) continue;
        float v = a[(((int64_t)b * H + h) * W + w) * C + c];
        if (v > best) { best = v; bi = kh * 3 + kw; }
      }
    arg[i] = (uint8_t)bi;
    int64_t pix = ((int64_t)b * Ho + ho) * Wo + wo;
    if (c < Ch) o1[pix * Ch + c] = best;
    else o2[pix * Ch + c - Ch] = best;
  }
}

__global__ void maxpool_bwd_kernel(const float *__restrict__ d1, const float *__restrict__ d2,
                                   const uint8_t *__restrict__ arg, int B, int H, int W, int C, int Ho, int Wo,
                                   float *__restrict__ da) {
  pdl_wait_trigger();
  int64_t n = (int64_t)B * H * W * C;
  int Ch = C / 2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int c = (int)(i % C);
    int64_t r = i / C;
    int w = (int)(r % W);
    r /= W;
    int h = (int)(r % H);
    int b = (int)(r / H);
    float s = 0.f;
    // output windows (ho, wo) with ho*2-1 <= h <= ho*2+1
    for (int ho = h / 2; ho <= min(Ho - 1, (h + 1) / 2); ++ho) {
      int kh = h - (ho * 2 - 1);
      if (kh < 0 || kh > 2) continue;
      for (int wo = w / 2; wo <= min(Wo - 1, (w + 1) / 2); ++wo) {
        int kw = w - (wo * 2 - 1);
        if (kw < 0 || kw > 2) continue;
        int64_t pix = ((int64_t)b * Ho + ho) * Wo + wo;
        if (arg[pix * C + c] == kh * 3 + kw) s += (c < Ch) ? d1[pix * Ch + c] : d2[pix * Ch + c - Ch];
      }
    }
    da[i] = s;
  }
}

// vectorised variants (C % 8 == 0, 32-bit indexing): one thread = 4 channels of one
// pixel, float4 loads/stores, the 4 argmax bytes as one 32-bit word
// one output pixel row (b, ho) per block iteration: threads walk (wo, c) with a shift when
// C4 is a power of two (no per-element 32-bit divisions)
__global__ void maxpool_fwd_v4_kernel(const float4 *__restrict__ a, int B, int H, int W, int C4, int Ho, int Wo,
                                      float4 *__restrict__ o1, float4 *__restrict__ o2, uchar4 *__restrict__ arg) {
  pdl_wait_trigger();
  const int Ch4 = C4 / 2, rowlen = Wo * C4;
  const int sh = (C4 & (C4 - 1)) == 0 ? __ffs(C4) - 1 : -1;
  for (int row = blockIdx.x; row < B * Ho; row += gridDim.x) {
    const int b = row / Ho, ho = row - b * Ho;
    for (int j = threadIdx.x; j < rowlen; j += blockDim.x) {
      const int wo = sh >= 0 ? j >> sh : j / C4, c = j - wo * C4;
      float4 best = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      uchar4 bi = make_uchar4(0, 0, 0, 0);
#pragma unroll
      for (int kh = 0; kh < 3; ++kh)
#pragma unroll
        for (int kw = 0; kw < 3; ++kw) {
          const int h = ho * 2 + kh - 1, w = wo * 2 + kw - 1;
          if (h < 0 || h >= H || w < 0 || w >= W) continue;
          const float4 v = a[((b * H + h) * W + w) * C4 + c];
          const unsigned char t = (unsigned char)(kh * 3 + kw);
          if (v.x > best.x) { best.x = v.x; bi.x = t; }  // strict >: first index wins ties
          if (v.y > best.y) { best.y = v.y; bi.y = t; }
          if (v.z > best.z) { best.z = v.z; bi.z = t; }
          if (v.w > best.w) { best.w = v.w; bi.w = t; }
        }
      const int pix = row * Wo + wo;
      arg[pix * C4 + c] = bi;
      if (c < Ch4) o1[pix * Ch4 + c] = best;
      else o2[pix * Ch4 + c - Ch4] = best;
    }
  }
}

__global__ void maxpool_bwd_v4_kernel(const float4 *__restrict__ d1, const float4 *__restrict__ d2,
                                      const uchar4 *__restrict__ arg, int B, int H, int W, int C4, int Ho, int Wo,
                                      float4 *__restrict__ da) {
  pdl_wait_trigger();
  // one input pixel row (b, h) per block iteration (as the forward: no per-element divisions)
  const int Ch4 = C4 / 2, rowlen = W * C4;
  const int sh = (C4 & (C4 - 1)) == 0 ? __ffs(C4) - 1 : -1;
  for (int row = blockIdx.x; row < B * H; row += gridDim.x) {
    const int b = row / H, h = row - b * H;
    for (int j = threadIdx.x; j < rowlen; j += blockDim.x) {
      const int w = sh >= 0 ? j >> sh : j / C4, c = j - w * C4;
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
      // output windows (ho, wo) with 2*ho-1 <= h <= 2*ho+1, in increasing (ho, wo) order
      for (int ho = h / 2; ho <= min(Ho - 1, (h + 1) / 2); ++ho) {
        const int kh = h - (ho * 2 - 1);
        if (kh < 0 || kh > 2) continue;
        for (int wo = w / 2; wo <= min(Wo - 1, (w + 1) / 2); ++wo) {
          const int kw = w - (wo * 2 - 1);
          if (kw < 0 || kw > 2) continue;
          const int op = (b * Ho + ho) * Wo + wo;
          const uchar4 g = arg[op * C4 + c];
          const float4 d = c < Ch4 ? d1[op * Ch4 + c] : d2[op * Ch4 + c - Ch4];
          const unsigned char t = (unsigned char)(kh * 3 + kw);
          if (g.x == t) s.x += d.x;
          if (g.y == t) s.y += d.y;
          if (g.z == t) s.z += d.z;
          if (g.w == t) s.w += d.w;
        }
      }
      da[(int64_t)row * rowlen + j] = s;
    }
  }
}

__global__ void f32_to_bf16_kernel(const float *__restrict__ x, __nv_bfloat16 *__restrict__ y, int64_t n) {
  pdl_wait_trigger();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x, t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if ((n & 3) == 0 && ((uintptr_t)x & 15) == 0 && ((uintptr_t)y & 7) == 0) {  // 16-byte loads, 8-byte stores
    const float4 *x4 = reinterpret_cast<const float4 *>(x);
    uint2 *y4 = reinterpret_cast<uint2 *>(y);
    for (int64_t i = t0; i < n / 4; i += stride) {
      const float4 v = x4[i];
      __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
      y4[i] = make_uint2(*reinterpret_cast<uint32_t *>(&lo), *reinterpret_cast<uint32_t *>(&hi));
    }
    return;
  }
  for (int64_t i = t0; i < n; i += stride) y[i] = __float2bfloat16_rn(x[i]);
}

// bf16 wire format of the pipeline messages: x = float(bf16_rn(x)) in place (mode 0),
// or the exact widening y = float(x_bf16) (mode 1, unpacking a received message)
__global__ void round_bf16_kernel(float *__restrict__ x, int64_t n) {
  pdl_wait_trigger();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x, t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if ((n & 3) == 0 && ((uintptr_t)x & 15) == 0) {
    float4 *x4 = reinterpret_cast<float4 *>(x);
    for (int64_t i = t0; i < n / 4; i += stride) {
      float4 v = x4[i];
      v.x = __bfloat162float(__float2bfloat16_rn(v.x));
      v.y = __bfloat162float(__float2bfloat16_rn(v.y));
      v.z = __bfloat162float(__float2bfloat16_rn(v.z));
      v.w = __bfloat162float(__float2bfloat16_rn(v.w));
      x4[i] = v;
    }
    return;
  }
  for (int64_t i = t0; i < n; i += stride) x[i] = __bfloat162float(__float2bfloat16_rn(x[i]));
}
__global__ void bf16_to_f32_kernel(const __nv_bfloat16 *__restrict__ x, float *__restrict__ y, int64_t n) {
  pdl_wait_trigger();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x, t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t i = t0; i < n; i += stride) y[i] = __bfloat162float(x[i]);
}

// interior of a zero-bordered [B][H+2][W+2][C] bf16 buffer (C % 4 == 0)
__global__ void f32_to_bf16_padded_kernel(const float4 *__restrict__ x, uint2 *__restrict__ y, int B, int H, int W,
                                          int C4) {
  pdl_wait_trigger();
  // one pixel row (b, h) per block iteration: W * C4 contiguous float4 in, the same run
  // of uint2 out one padded pixel in (no per-element index divisions)
  const int rowlen = W * C4;
  for (int r = blockIdx.x; r < B * H; r += gridDim.x) {
    const int b = r / H, h = r - b * H;
    const float4 *src = x + (int64_t)r * rowlen;
    uint2 *dst = y + (((int64_t)b * (H + 2) + h + 1) * (W + 2) + 1) * C4;
    for (int j = threadIdx.x; j < rowlen; j += blockDim.x) {
      const float4 v = src[j];
      __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
      dst[j] = make_uint2(*reinterpret_cast<uint32_t *>(&lo), *reinterpret_cast<uint32_t *>(&hi));
    }
  }
}

// grid-stride elementwise kernels: at most PETRA_EW_BLOCKS_PER_SM (default 8) 256-thread blocks per SM
inline unsigned ew_grid(int64_t n) {
  static const int per_sm = std::max(1, env_int("PETRA_EW_BLOCKS_PER_SM", 8));
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), (int64_t)per_sm * kNumSMs));
}
// row-stride kernels (one pixel row per block iteration): PETRA_ROW_BLOCKS_PER_SM (default 16)
inline int64_t row_blocks() {
  static const int per_sm = std::max(1, env_int("PETRA_ROW_BLOCKS_PER_SM", 16));
  return (int64_t)per_sm * kNumSMs;
}

}  // namespace

std::vector<SgdChunk> sgd_chunks(const std::vector<SgdSeg> &segs) {
  std::vector<SgdChunk> out;
  for (int s = 0; s < (int)segs.size(); ++s) {
    const SgdSeg &g = segs[s];
    if (g.wt_bf16) {
      const int64_t tiles = (int64_t)g.k * g.k * ((g.co + 31) / 32) * ((g.ci + 31) / 32);
      for (int64_t t = 0; t < tiles; ++t) out.push_back({s, t, t + 1});
    } else {
      for (int64_t lo = 0; lo < g.count; lo += 1024) out.push_back({s, lo, std::min<int64_t>(g.count, lo + 1024)});
    }
  }
  return out;
}

void sgd_update(const SgdSeg *segs_dev, int nseg, const SgdChunk *chunks_dev, int nchunks, float *theta, float *v,
                const float *grad, float *acc, int k, int mode, const float *lr_dev, float mom, float wd, int nesterov,
                cudaStream_t st, bool shadow_only, int *nonfinite) {
  // blocks stride over the items: PETRA_SGD_BLOCKS caps the grid (default 8 per SM)
  static const int cap = std::max(1, env_int("PETRA_SGD_BLOCKS", 8 * kNumSMs));
  const unsigned grid = (unsigned)std::max(1, std::min(nchunks, cap));
  launch_k(sgd_kernel, grid, 256, 0, st, segs_dev, chunks_dev, nchunks, theta, v, grad, acc, 1.f / (float)k, mode,
           lr_dev, mom, wd, nesterov, shadow_only ? 1 : 0, nonfinite);
  PETRA_LAUNCH_CHECK();
}

// Evaluation of the classifier (the running statistics "are then used
// during model evaluation"): per row, the CE loss and whether the first-index argmax of
// the logits equals the label; correct counts are integer atomics (exact)
__global__ void eval_rows_kernel(const float *__restrict__ logits, const int32_t *__restrict__ labels, int B, int N,
                                 float *__restrict__ loss_row, int *__restrict__ correct) {
  pdl_wait_trigger();
  __shared__ float sm[32];
  __shared__ int si[32];
  const int b = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5, nw = blockDim.x >> 5;
  const float *z = logits + (size_t)b * N;
  float m = -INFINITY;
  int im = N;
  for (int n = t; n < N; n += blockDim.x)
    if (z[n] > m) { m = z[n]; im = n; }
  for (int o = 16; o; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, im, o);
    if (m2 > m || (m2 == m && i2 < im)) { m = m2; im = i2; }
  }
  if (lane == 0) { sm[w] = m; si[w] = im; }
  __syncthreads();
  if (t == 0) {
    for (int k = 1; k < nw; ++k)
      if (sm[k] > sm[0] || (sm[k] == sm[0] && si[k] < si[0])) { sm[0] = sm[k]; si[0] = si[k]; }
  }
  __syncthreads();
  m = sm[0];
  const int arg = si[0];
  float e = 0.f;
  for (int n = t; n < N; n += blockDim.x) e += expf(z[n] - m);
  for (int o = 16; o; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
  __syncthreads();
  if (lane == 0) sm[w] = e;
  __syncthreads();
  if (t == 0) {
    float tot = 0.f;
    for (int k = 0; k < nw; ++k) tot += sm[k];
    const int y = labels[b];
    loss_row[b] = logf(tot) + m - z[y];
    if (arg == y) atomicAdd(correct, 1);
  }
}

void tail_forward_backward(const float *x1, const float *x2, int B, int HW, int C, const float *w,
                           const float *bias, int N, const int32_t *labels, float *feat, float *logits,
                           float *dlogits, float *loss_row, float *dfeat, float *dw, float *db, float *d1,
                           float *d2, float *loss, int *nonfinite, float *fc_ws, int64_t fc_ws_floats,
                           cudaStream_t st, int *correct) {
  int Cin = 2 * C;
  launch_k(gap_kernel, dim3((unsigned)cdiv(Cin, 128), B), 128, 0, st, x1, x2, B, HW, C, feat);
  PETRA_LAUNCH_CHECK();
  auto gemm = [&](const float *A, int64_t sam, int64_t sak, const float *Bm, int64_t sbk, int64_t sbn,
                  const float *bs, int M, int Nn, int K, float *C) {
    // split K until ~2048 blocks or 8 chunks per block, within the workspace
    const int64_t tiles = cdiv(Nn, GN) * cdiv(M, GM);
    int splits = 1;
    while (splits < 64 && tiles * splits * 2 <= 2048 && cdiv(K, (int64_t)GK * splits * 2) >= 1 &&
           (int64_t)(splits * 2) * M * Nn <= fc_ws_floats)
      splits *= 2;
    const int kspan = (int)(cdiv(cdiv(K, splits), GK) * GK);
    splits = (int)cdiv(K, kspan);
    launch_k(fc_gemm_kernel, dim3((unsigned)cdiv(Nn, GN), (unsigned)cdiv(M, GM), (unsigned)splits), 128, 0, st, A,
             sam, sak, Bm, sbk, sbn, bs, M, Nn, K, kspan, splits > 1 ? fc_ws : C);
    PETRA_LAUNCH_CHECK();
    if (splits > 1) {
      const int64_t n = (int64_t)M * Nn;
      launch_k(fc_splitk_reduce_kernel, (unsigned)std::min<int64_t>(cdiv(n, 256), 4 * kNumSMs), 256, 0, st, fc_ws,
               splits, n, Nn, bs, C);
      PETRA_LAUNCH_CHECK();
    }
  };
  // logits[b][n] = sum_c feat[b][c] w[n][c] + bias[n]
  gemm(feat, Cin, 1, w, 1, Cin, bias, B, N, Cin, logits);
  if (correct) {  // evaluation: loss and correct count only (no gradients)
    launch_k(eval_rows_kernel, B, 256, 0, st, logits, labels, B, N, loss_row, correct);
    PETRA_LAUNCH_CHECK();
    launch_k(loss_mean_kernel, 1, 32, 0, st, loss_row, B, loss, nonfinite);
    PETRA_LAUNCH_CHECK();
    return;
  }
  launch_k(ce_kernel, B, 256, 0, st, logits, labels, B, N, dlogits, loss_row);
  PETRA_LAUNCH_CHECK();
  launch_k(loss_mean_kernel, 1, 32, 0, st, loss_row, B, loss, nonfinite);
  PETRA_LAUNCH_CHECK();
  // dw[n][c] = sum_b dlogits[b][n] feat[b][c];  db[n] = sum_b dlogits[b][n]
  gemm(dlogits, 1, N, feat, Cin, 1, nullptr, N, Cin, B, dw);
  launch_k(fc_bias_grad_kernel, (unsigned)cdiv(N, 256), 256, 0, st, dlogits, B, N, db);
  PETRA_LAUNCH_CHECK();
  // dfeat[b][c] = sum_n dlogits[b][n] w[n][c]
  gemm(dlogits, N, 1, w, Cin, 1, nullptr, B, Cin, N, dfeat);
  launch_k(gap_bwd_kernel, ew_grid((int64_t)B * HW * C), 256, 0, st, dfeat, B, HW, C, d1, d2);
  PETRA_LAUNCH_CHECK();
}

void maxpool_fwd(const float *a, int B, int H, int W, int C, int Ho, int Wo, float *o1, float *o2, uint8_t *arg,
                 cudaStream_t st) {
  if (C % 8 == 0 && (int64_t)B * H * W * C < ((int64_t)1 << 31)) {
    const int C4 = C / 4;
    launch_k(maxpool_fwd_v4_kernel, (unsigned)std::min<int64_t>((int64_t)B * Ho, row_blocks()), 256, 0, st, 
        reinterpret_cast<const float4 *>(a), B, H, W, C4, Ho, Wo, reinterpret_cast<float4 *>(o1),
        reinterpret_cast<float4 *>(o2), reinterpret_cast<uchar4 *>(arg));
  } else {
    launch_k(maxpool_fwd_kernel, ew_grid((int64_t)B * Ho * Wo * C), 256, 0, st, a, B, H, W, C, Ho, Wo, o1, o2, arg);
  }
  PETRA_LAUNCH_CHECK();
}

void maxpool_bwd(const float *d1, const float *d2, const uint8_t *arg, int B, int H, int W, int C, int Ho, int Wo,
                 float *da, cudaStream_t st) {
  if (C % 8 == 0 && (int64_t)B * H * W * C < ((int64_t)1 << 31)) {
    const int C4 = C / 4;
    launch_k(maxpool_bwd_v4_kernel, (unsigned)std::min<int64_t>((int64_t)B * H, row_blocks()), 256, 0, st, 
        reinterpret_cast<const float4 *>(d1), reinterpret_cast<const float4 *>(d2),
        reinterpret_cast<const uchar4 *>(arg), B, H, W, C4, Ho, Wo, reinterpret_cast<float4 *>(da));
  } else {
    launch_k(maxpool_bwd_kernel, ew_grid((int64_t)B * H * W * C), 256, 0, st, d1, d2, arg, B, H, W, C, Ho, Wo, da);
  }
  PETRA_LAUNCH_CHECK();
}

void f32_to_bf16_padded(const float *x, __nv_bfloat16 *y, int B, int H, int W, int C, cudaStream_t st) {
  const int C4 = C / 4;
  launch_k(f32_to_bf16_padded_kernel, (unsigned)std::min<int64_t>((int64_t)B * H, row_blocks()), 256, 0, st, 
      reinterpret_cast<const float4 *>(x), reinterpret_cast<uint2 *>(y), B, H, W, C4);
  PETRA_LAUNCH_CHECK();
}

void round_bf16_inplace(float *x, int64_t n, cudaStream_t st) {
  const bool v4 = (n & 3) == 0 && ((uintptr_t)x & 15) == 0;
  launch_k(round_bf16_kernel, ew_grid(v4 ? n / 4 : n), 256, 0, st, x, n);
  PETRA_LAUNCH_CHECK();
}

void bf16_to_f32(const __nv_bfloat16 *x, float *y, int64_t n, cudaStream_t st) {
  launch_k(bf16_to_f32_kernel, ew_grid(n), 256, 0, st, x, y, n);
  PETRA_LAUNCH_CHECK();
}

void f32_to_bf16(const float *x, __nv_bfloat16 *y, int64_t n, cudaStream_t st) {
  const bool v4 = (n & 3) == 0 && ((uintptr_t)x & 15) == 0 && ((uintptr_t)y & 7) == 0;
  launch_k(f32_to_bf16_kernel, ew_grid(v4 ? n / 4 : n), 256, 0, st, x, y, n);
  PETRA_LAUNCH_CHECK();
}

}  // namespace petra

// bn.cu -- BatchNorm (training mode) + ReLU + additive coupling, HBM-streaming kernels.
//
//   stats     : mu_c, sigma2_c = biased batch mean / variance of z over all rows
//               (B*H*W), invstd = 1/sqrt(sigma2+eps); optional running-stat EMA
//               (only in the backward recomputation; reading c9).
//   apply     : out = acc + sign * act(gamma*(z-mu)*invstd + beta)
//               forward coupling (sign +1) / DS / stem / bottleneck
//               inner activations; optionally also writes a bf16 copy of out (the
//               next convolution's tensor-core operand).
//   bwd_reduce: per channel  sum g,  sum g*xhat  with g = dy * 1[out > 0]
//               (= dbeta, dgamma), optionally fused with the reconstruction
//               dst_out = dst_in - act(bn(z))  (approximate inversion).
//   bwd_dz    : dz = gamma*invstd*(g - sum(g)/n - xhat*sum(g*xhat)/n).
// Deterministic: per-block fp64 partials, merged in a fixed order by the last
// block to finish (atomic ticket after a fence) -- one launch per reduction, no
// float atomics.  Streaming passes move 4 channels per thread (16-byte accesses).
#include <mutex>
#include <type_traits>

#include "../kernels.h"
#include "tc_common.cuh"
#include "tc_common.cuh"

namespace petra {
namespace {

__device__ __forceinline__ float ldv(const float *p, int64_t i) { return p[i]; }
__device__ __forceinline__ float ldv(const __nv_bfloat16 *p, int64_t i) { return __bfloat162float(p[i]); }
__device__ __forceinline__ void stv(float *p, int64_t i, float v) { p[i] = v; }
__device__ __forceinline__ void stv(__nv_bfloat16 *p, int64_t i, float v) { p[i] = __float2bfloat16_rn(v); }

__device__ __forceinline__ float4 ld4(const float *p, int64_t i) { return *reinterpret_cast<const float4 *>(p + i); }
__device__ __forceinline__ float4 ld4(const __nv_bfloat16 *p, int64_t i) {
  uint2 u = *reinterpret_cast<const uint2 *>(p + i);
  __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162 *>(&u.x), b = *reinterpret_cast<__nv_bfloat162 *>(&u.y);
  float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
  return make_float4(fa.x, fa.y, fb.x, fb.y);
}
__device__ __forceinline__ void st4(float *p, int64_t i, float4 v) { *reinterpret_cast<float4 *>(p + i) = v; }
__device__ __forceinline__ void st4(__nv_bfloat16 *p, int64_t i, float4 v) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t *>(&a);
  u.y = *reinterpret_cast<uint32_t *>(&b);
  *reinterpret_cast<uint2 *>(p + i) = u;
}
__device__ __forceinline__ float f4(const float4 &v, int k) { return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w; }

// row of flat index i over rows of C4 float4 groups (shift when C4 is a power of two)
__device__ __forceinline__ int64_t row_of(int64_t i, int C4, int sh) { return sh >= 0 ? (i >> sh) : i / C4; }
inline int log2_or_neg(int v) {
  if (v <= 0 || (v & (v - 1))) return -1;
  int s = 0;
  while ((1 << s) < v) ++s;
  return s;
}
// row m of an H x W grid -> row of the zero-bordered (H+2) x (W+2) layout (pH <= 0: m).
// The two divisions are multiply-high with magic numbers computed once per thread
// (PadMap): an integer division costs ~25 instructions, and these kernels run one per
// row of four channels -- ncu showed them instruction-bound (issue 54 %) on it.
struct PadMap {
  tc::FastDiv fhw, fw;
  int pH, pW;
};
__device__ __forceinline__ tc::FastDiv fastdiv_dev(uint32_t d) {
  tc::FastDiv f;
  f.d = d;
  if (d <= 1) {
    f.m = 0;
    f.s = -1;
  } else {
    const int l = 32 - __clz(d - 1);  // ceil(log2 d)
    f.m = (uint32_t)(((1ull << (31 + l)) + d - 1) / d);
    f.s = l - 1;
  }
  return f;
}
__device__ __forceinline__ PadMap pad_map(int pH, int pW) {
  PadMap p;
  p.pH = pH;
  p.pW = pW;
  if (pH > 0) {
    p.fhw = fastdiv_dev((uint32_t)(pH * pW));
    p.fw = fastdiv_dev((uint32_t)pW);
  }
  return p;
}
__device__ __forceinline__ int64_t pad_row(int64_t m, const PadMap &p) {
  if (p.pH <= 0) return m;
  // 32-bit index math: the padded operand buffers hold < 2^31 rows (host-checked)
  const int mi = (int)m;
  const int b = tc::fdiv(mi, p.fhw), r = mi - b * (int)p.fhw.d, h = tc::fdiv(r, p.fw), w = r - h * p.pW;
  return ((int64_t)b * (p.pH + 2) + h + 1) * (p.pW + 2) + w + 1;
}

// reduction blocks: one wave of NT-thread blocks (stats 1024, backward reduce 512:
// >= 64 KB of loads in flight per SM)
constexpr int RT_STATS = 1024, RT_BWD = 512;
constexpr int kMaxRing = 4;  // deepest TMA ring of the BN passes

// Reduction geometry: a block covers a tile of CT channels (TPR threads per row,
// 4 channels each; RG = 256/TPR row groups) and a contiguous chunk of rpb rows.
struct RedGeom {
  int CT, TPR, RG, ctiles, nrb;
  int64_t rpb;
};
inline RedGeom red_geom(int64_t M, int C, int RT, int per_sm = 1) {
  RedGeom g;
  if (C % 4 == 0) {
    g.CT = std::min(C, 128);
    while (C % g.CT) g.CT -= 4;  // a multiple of 4 dividing C
    g.TPR = g.CT / 4;
  } else {
    g.CT = 32;
    g.TPR = 32;
  }
  g.RG = RT / g.TPR;
  g.ctiles = (int)cdiv(C, g.CT);
  // one wave: one block per SM (1024 / 512 threads, >= 64 KB of loads in flight), few
  // partials to merge
  int64_t want = std::max<int64_t>(1, (int64_t)per_sm * kNumSMs / g.ctiles);
  // PETRA_BN_BLOCKS (experiment): at most that many blocks per pass (0: no cap)
  static const int cap_blocks = env_int("PETRA_BN_BLOCKS", 0);
  if (cap_blocks > 0) want = std::min<int64_t>(want, std::max(1, cap_blocks / g.ctiles));
  // at least `min_rows` rows per block (PETRA_BN_MIN_ROWS, default 128; at least 4 row groups): small
  // tensors otherwise spread over hundreds of blocks of a few rows each
  static const int min_rows = env_int("PETRA_BN_MIN_ROWS", 128);  // 128: R18 +2.9 % (DESIGN 7)
  g.nrb = (int)std::max<int64_t>(1, std::min<int64_t>(want, cdiv(M, std::max(4 * g.RG, min_rows))));
  g.rpb = cdiv(M, g.nrb);
  g.nrb = (int)cdiv(M, g.rpb);
  return g;
}

// dy(m, c): single [M][C] tensor, or split halves dy0 = channels [0, cs), dy1 = [cs, C)
__device__ __forceinline__ float load_dy(const float *dy0, const float *dy1, int cs, int C, int64_t m, int c) {
  if (dy1 == nullptr) return dy0[m * C + c];
  return c < cs ? dy0[m * cs + c] : dy1[m * (C - cs) + (c - cs)];
}
__device__ __forceinline__ float4 load_dy4(const float *dy0, const float *dy1, int cs, int C, int64_t m, int c) {
  if (dy1 == nullptr) return ld4(dy0, m * C + c);
  return c < cs ? ld4(dy0, m * cs + c) : ld4(dy1, m * (C - cs) + (c - cs));
}

// Block-level fixed-order combine of per-thread sums (row groups) into this
// block's partial part[blk][c][0..1]; sh is a [RT][4] double scratch, used for one
// quantity at a time.
template <int RT>
__device__ __forceinline__ void write_partial(double (*sh)[4], const double *a, const double *b, bool vec, int TPR,
                                              int RG, int c0, int C, double *part) {
  const int t = threadIdx.x;
  const int nslots = vec ? TPR * 4 : TPR;
  for (int q = 0; q < 2; ++q) {
    const double *src = q == 0 ? a : b;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; ++k) sh[t][k] = src[k];
    __syncthreads();
    for (int slot = t; slot < nslots; slot += RT) {
      int cjs = vec ? slot / 4 : slot, k = vec ? slot % 4 : 0;
      int cc = vec ? c0 + 4 * cjs + k : c0 + cjs;
      if (cc >= C) continue;
      double x = 0;
      for (int g = 0; g < RG; ++g) x += sh[g * TPR + cjs][k];
      part[((int64_t)blockIdx.x * C + cc) * 2 + q] = x;
    }
  }
}

// true in exactly one block per channel tile: the last to finish its partial
__device__ __forceinline__ bool last_block(unsigned *counter, int nrb) {
  __shared__ unsigned ticket;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) ticket = atomicAdd(&counter[blockIdx.y], 1u);
  __syncthreads();
  if (ticket != (unsigned)(nrb - 1)) return false;
  __threadfence();
  return true;
}

// merge the nrb partials of channels [c0, c0+CT) in a fixed order: RT/CT threads
// per channel over fixed strided subsets (4 L2-coherent 16-byte loads in flight),
// then a fixed-order shared-memory combine.  Result valid in threads t < CT.
template <int RT>
__device__ __forceinline__ void merge_tile(const double *part, int nrb, int C, int c0, int CT, double (*sh)[4],
                                           double &a, double &b) {
  const int t = threadIdx.x;
  const int per = RT / CT;
  const int cl = t % CT, sub = t / CT;
  const int c = c0 + cl;
  double2 acc[4] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  if (sub < per && c < C) {
    const double2 *p2 = reinterpret_cast<const double2 *>(part);
    int i = sub;
    for (; i + 3 * per < nrb; i += 4 * per) {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcg(p2 + (int64_t)(i + u * per) * C + c);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc[u].x += v[u].x;
        acc[u].y += v[u].y;
      }
    }
    for (; i < nrb; i += per) {
      double2 v = __ldcg(p2 + (int64_t)i * C + c);
      acc[0].x += v.x;
      acc[0].y += v.y;
    }
  }
  __syncthreads();
  sh[t][0] = (acc[0].x + acc[1].x) + (acc[2].x + acc[3].x);
  sh[t][1] = (acc[0].y + acc[1].y) + (acc[2].y + acc[3].y);
  __syncthreads();
  a = 0;
  b = 0;
  if (t < CT)
    for (int k = 0; k < per; ++k) {
      a += sh[k * CT + t][0];
      b += sh[k * CT + t][1];
    }
}

// ---------------------------------------------------------------- stats
template <typename TZ>
__global__ void __launch_bounds__(RT_STATS) bn_stats_kernel(const TZ *__restrict__ z, int64_t M, int C, int CT, int TPR,
                                                      int RG, int64_t rpb, int nrb, double *__restrict__ part,
                                                      unsigned *__restrict__ counter, float eps,
                                                      float *__restrict__ mean, float *__restrict__ invstd,
                                                      float *__restrict__ rmean, float *__restrict__ rvar,
                                                      float mom) {
  pdl_wait_trigger();
  constexpr int RT = RT_STATS;
  __shared__ double sh[RT][4];
  const int t = threadIdx.x, cj = t % TPR, rgi = t / TPR;
  const int c0 = blockIdx.y * CT;
  const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = min(M, r0 + rpb);
  double s[4] = {0, 0, 0, 0}, ss[4] = {0, 0, 0, 0};
  const bool vec = (C % 4 == 0);
  const int c = vec ? c0 + 4 * cj : c0 + cj;
  if (c < C && rgi < RG && vec) {
    int64_t r = r0 + rgi;
    for (; r + 3 * RG < r1; r += 4 * RG) {  // 4 independent 16-byte loads in flight
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = ld4(z, (r + u * RG) * C + c);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          double d = f4(v[u], k);
          s[k] += d;
          ss[k] += d * d;
        }
    }
    for (; r < r1; r += RG) {
      float4 v = ld4(z, r * C + c);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        double d = f4(v, k);
        s[k] += d;
        ss[k] += d * d;
      }
    }
  } else if (c < C && rgi < RG) {
    for (int64_t r = r0 + rgi; r < r1; r += RG) {
      {
        double d = ldv(z, r * C + c);
        s[0] += d;
        ss[0] += d * d;
      }
    }
  }
  write_partial<RT>(sh, s, ss, vec, TPR, RG, c0, C, part);
  if (!last_block(counter, nrb)) return;
  double su, sq;
  merge_tile<RT>(part, nrb, C, c0, CT, sh, su, sq);
  const int ch = c0 + t;
  if (t < CT && ch < C) {
    double mu = su / (double)M;
    double var = sq / (double)M - mu * mu;
    if (var < 0.0) var = 0.0;
    mean[ch] = (float)mu;
    invstd[ch] = (float)(1.0 / sqrt(var + (double)eps));
    if (rmean) {
      double unb = M > 1 ? var * (double)M / (double)(M - 1) : var;
      rmean[ch] = (float)((1.0 - mom) * rmean[ch] + mom * mu);
      rvar[ch] = (float)((1.0 - mom) * rvar[ch] + mom * unb);
    }
  }
  if (t == 0) counter[blockIdx.y] = 0u;  // ready for the next launch
}

// ---------------------------------------------------------------- apply
template <typename TZ, typename TO>
__global__ void bn_apply_kernel(int64_t M, int C, const TZ *__restrict__ z, int ldz, int zc0,
                                const float *__restrict__ mean, const float *__restrict__ invstd,
                                const float *__restrict__ gamma, const float *__restrict__ beta, int relu,
                                float sign, const float *acc, TO *out, __nv_bfloat16 *out_bf16, int pH, int pW,
                                int sh) {
  pdl_wait_trigger();
  const PadMap pm = pad_map(pH, pW);
  const bool vec = (C % 4 == 0) && (ldz % 4 == 0) && (zc0 % 4 == 0);
  if (vec) {
    const int C4 = C / 4;
    const int64_t n = M * C4;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      int64_t m = row_of(i, C4, sh);
      int c = (int)(i - m * C4) * 4;
      int cz = zc0 + c;
      float4 zv = ld4(z, m * ldz + cz);
      float4 o;
      float *op = &o.x;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float y = fmaf(gamma[cz + k] * invstd[cz + k], f4(zv, k) - mean[cz + k], beta[cz + k]);
        if (relu) y = y > 0.f ? y : 0.f;
        op[k] = sign * y;
      }
      if (acc) {
        float4 a = ld4(acc, m * C + c);
        o.x += a.x; o.y += a.y; o.z += a.z; o.w += a.w;
      }
      if (out) st4(out, m * C + c, o);
      if (out_bf16) st4(out_bf16, pad_row(m, pm) * C + c, o);
    }
    return;
  }
  const int64_t n = M * C;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t m = i / C;
    int c = (int)(i - m * C);
    int cz = zc0 + c;
    float y = fmaf(gamma[cz] * invstd[cz], ldv(z, m * ldz + cz) - mean[cz], beta[cz]);
    if (relu) y = y > 0.f ? y : 0.f;
    float o = sign * y;
    if (acc) o += acc[i];
    if (out) stv(out, i, o);
    if (out_bf16) out_bf16[pad_row(m, pm) * C + c] = __float2bfloat16_rn(o);
  }
}

// Per-channel passes with one 4-channel group per thread: the grid stride is a
// multiple of C/4 (chan_grid), so the BN constants of a thread live in registers and
// rows advance by stride / (C/4); two rows per trip, loads issued before use.  Row
// indices are 32-bit (M < 2^31, host-checked).
template <typename TZ>
__global__ void __launch_bounds__(256, 4) bn_apply_fixed_kernel(
    int M, int C, const TZ *__restrict__ z, int ldz, int zc0, const float *__restrict__ mean,
    const float *__restrict__ invstd, const float *__restrict__ gamma, const float *__restrict__ beta, int relu,
    float sign, const float *__restrict__ acc, float *__restrict__ out, __nv_bfloat16 *__restrict__ out_bf16, int pH,
    int pW) {
  pdl_wait_trigger();
  const PadMap pm = pad_map(pH, pW);
  const int C4 = C / 4;
  const int stride = gridDim.x * blockDim.x;
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = (t0 % C4) * 4, cz = zc0 + c;
  const int dm = stride / C4;
  float a[4], mu[4], be[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    a[k] = gamma[cz + k] * invstd[cz + k];
    mu[k] = mean[cz + k];
    be[k] = beta[cz + k];
  }
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int m = t0 / C4; m < M; m += 2 * dm) {
    const bool two = m + dm < M;
    const float4 z0 = ld4(z, (int64_t)m * ldz + cz);
    const float4 z1 = two ? ld4(z, (int64_t)(m + dm) * ldz + cz) : zero;
    const float4 a0 = acc ? ld4(acc, (int64_t)m * C + c) : zero;
    const float4 a1 = (acc && two) ? ld4(acc, (int64_t)(m + dm) * C + c) : zero;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (u && !two) break;
      const int mm = m + u * dm;
      const float4 zv = u ? z1 : z0, av = u ? a1 : a0;
      float4 o;
      float *op = &o.x;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float y = fmaf(a[k], f4(zv, k) - mu[k], be[k]);
        if (relu) y = y > 0.f ? y : 0.f;
        op[k] = sign * y;
      }
      o.x += av.x; o.y += av.y; o.z += av.z; o.w += av.w;
      if (out) st4(out, (int64_t)mm * C + c, o);
      if (out_bf16) st4(out_bf16, pad_row(mm, pm) * C + c, o);
    }
  }
}

template <typename TZ>
__global__ void __launch_bounds__(256, 4) bn_bwd_dz_fixed_kernel(
    int M, int C, const TZ *__restrict__ z, const float *__restrict__ mean, const float *__restrict__ invstd,
    const float *__restrict__ gamma, const float *__restrict__ beta, int relu, const float *__restrict__ dy,
    const float *__restrict__ dgamma, const float *__restrict__ dbeta, float *__restrict__ dz,
    __nv_bfloat16 *__restrict__ dz_bf16, int pH, int pW) {
  pdl_wait_trigger();
  const PadMap pm = pad_map(pH, pW);
  const float invM = 1.0f / (float)M;
  const int C4 = C / 4;
  const int stride = gridDim.x * blockDim.x;
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = (t0 % C4) * 4;
  const int dm = stride / C4;
  float is[4], mu[4], ga[4], be[4], db[4], dg[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    is[k] = invstd[c + k];
    mu[k] = mean[c + k];
    ga[k] = gamma[c + k];
    be[k] = beta[c + k];
    db[k] = dbeta[c + k] * invM;
    dg[k] = dgamma[c + k];
  }
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int m = t0 / C4; m < M; m += 2 * dm) {
    const bool two = m + dm < M;
    const float4 z0 = ld4(z, (int64_t)m * C + c);
    const float4 z1 = two ? ld4(z, (int64_t)(m + dm) * C + c) : zero;
    const float4 g0 = ld4(dy, (int64_t)m * C + c);
    const float4 g1 = two ? ld4(dy, (int64_t)(m + dm) * C + c) : zero;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (u && !two) break;
      const int mm = m + u * dm;
      const float4 zv = u ? z1 : z0;
      float4 g4 = u ? g1 : g0;
      float4 o;
      float *op = &o.x, *gp = &g4.x;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float xh = (f4(zv, k) - mu[k]) * is[k];
        float g = gp[k];
        if (relu && !(fmaf(ga[k], xh, be[k]) > 0.f)) g = 0.f;
        op[k] = ga[k] * is[k] * (g - db[k] - xh * dg[k] * invM);  // same rounding as bn_bwd_dz_kernel
      }
      if (dz) st4(dz, (int64_t)mm * C + c, o);
      if (dz_bf16) st4(dz_bf16, pad_row(mm, pm) * C + c, o);
    }
  }
}


// ---------------------------------------------------------------- statistics fold
// Merge of a conv epilogue's BN partial rows (StatsFold; layout kernels.h StatsRows) for
// channels [cb, cb + CT) of the conv output, in the prologue of the consuming BN pass
// (instead of a stats_finalize launch).  Eight threads per channel (thread bits 0-2) take
// rows j, j + 8, ... of the channel's column group and accumulate in fp64, shifted by the
// group's first row mean m0:  A = sum n_r (m_r - m0),  B = sum n_r (m_r - m0)^2,
// W = sum M2_r,  n = sum n_r;  the eight are combined by a fixed xor tree (deterministic).
// mean = m0 + A / n, M2 = W + B - A^2 / n (the pairwise / Chan combination of (count,
// mean, M2) triples written as sums); biased variance M2 / M for the normalisation,
// unbiased M2 / (M - 1) for the running EMA (reading c9).  Results go to s_mu / s_is;
// `writer` (block 0 of the channel tile) also stores mean / invstd and updates the
// running statistics.  Ends with __syncthreads.  blockDim.x must be a multiple of 32.
__device__ void fold_stats(const StatsFold &f, int cb, int CT, float *s_mu, float *s_is, bool writer,
                           float *__restrict__ mean, float *__restrict__ invstd) {
  const int t = threadIdx.x;
  const float *cnt = f.part + (size_t)f.rows * f.N * 2;
  const int gsz = f.N / f.groups;
  for (int base = 0; base < CT * 8; base += blockDim.x) {  // same trip count in every thread
    const int slot = base + t, cl = slot >> 3, sub = slot & 7, c = cb + cl;
    double A = 0, Bq = 0, Wm = 0, n = 0, m0 = 0;
    if (cl < CT) {
      const int grp = c / gsz, nr = (f.rows - grp + f.groups - 1) / f.groups;
      m0 = f.part[((size_t)grp * f.N + c) * 2];
      for (int j = sub; j < nr; j += 8) {
        const int r = grp + j * f.groups;
        const float2 u = __ldcg(reinterpret_cast<const float2 *>(f.part + ((size_t)r * f.N + c) * 2));
        const double nr_ = __ldcg(cnt + r), d = (double)u.x - m0;
        A += nr_ * d;
        Bq += nr_ * d * d;
        Wm += u.y;
        n += nr_;
      }
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      A += __shfl_xor_sync(0xffffffffu, A, o);
      Bq += __shfl_xor_sync(0xffffffffu, Bq, o);
      Wm += __shfl_xor_sync(0xffffffffu, Wm, o);
      n += __shfl_xor_sync(0xffffffffu, n, o);
    }
    if (cl < CT && sub == 0) {
      const double mu = n > 0 ? m0 + A / n : 0.0;
      double M2 = n > 0 ? Wm + Bq - A * A / n : 0.0;
      if (M2 < 0.0) M2 = 0.0;
      const double var = f.M > 0 ? M2 / (double)f.M : 0.0;  // n == M: every valid output row once
      const float is = (float)(1.0 / sqrt(var + (double)f.eps));
      s_mu[cl] = (float)mu;
      s_is[cl] = is;
      if (writer) {
        mean[c] = (float)mu;
        invstd[c] = is;
        if (f.rmean) {
          const double unb = f.M > 1 ? M2 / (double)(f.M - 1) : var;
          f.rmean[c] = (float)((1.0 - f.mom) * f.rmean[c] + f.mom * mu);
          f.rvar[c] = (float)((1.0 - f.mom) * f.rvar[c] + f.mom * unb);
        }
      }
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------- TMA-staged BN passes
// BN apply, TMA-staged per channel tile (bitwise the arithmetic of
// bn_apply_fixed_kernel): thread (cj, rgi) keeps channels c0 + 4cj .. +3 and their
// constants in registers; z (a [M][ldz] view starting at column zc0) and the addend
// arrive per row chunk by 2-D TMA boxes into a two-stage smem ring.
template <typename TZ>
__global__ void __launch_bounds__(256) bn_apply_tma_kernel(
    const __grid_constant__ CUtensorMap tmZ, const __grid_constant__ CUtensorMap tmA, int has_acc, int64_t M, int C,
    int CT, int TPR, int RG, int64_t rpb, int Rc, int zc0, const float *__restrict__ mean,
    const float *__restrict__ invstd, const float *__restrict__ gamma, const float *__restrict__ beta, int relu,
    float sign, float *__restrict__ out, __nv_bfloat16 *__restrict__ out_bf16, int pH, int pW,
    const StatsFold fold) {
  pdl_wait_trigger();
  const PadMap pm = pad_map(pH, pW);
  __shared__ uint64_t full[2];
  __shared__ float s_mu[128], s_is[128];
  extern __shared__ __align__(128) uint8_t ring[];
  const int t = threadIdx.x, cj = t % TPR, rgi = t / TPR;
  const int c0 = blockIdx.y * CT;
  const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = min(M, r0 + rpb);
  const int c = c0 + 4 * cj;
  const bool mine = c < C && rgi < RG;
  const uint32_t zb = (uint32_t)Rc * CT * sizeof(TZ), ab = has_acc ? (uint32_t)Rc * CT * 4 : 0;
  const uint32_t sbytes = (zb + ab + 127) & ~127u;
  if (t == 0) {
    tc::mbar_init(&full[0], 1);
    tc::mbar_init(&full[1], 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  const int64_t nchunk = (r1 - r0 + Rc - 1) / Rc;
  auto issue = [&](int64_t k, int s) {
    const int y = (int)(r0 + k * Rc);
    uint8_t *st = ring + s * sbytes;
    tc::mbar_arrive_expect_tx(&full[s], zb + ab);
    tc::tma_load_2d(st, &tmZ, &full[s], c0, y);
    if (has_acc) tc::tma_load_2d(st + zb, &tmA, &full[s], c0, y);
  };
  if (t == 0 && nchunk > 0) issue(0, 0);  // the first chunk streams in while the statistics merge
  if (fold.part)  // this tile's statistics from the conv epilogue's partial rows
    fold_stats(fold, zc0 + c0, min(CT, C - c0), s_mu, s_is, blockIdx.x == 0, const_cast<float *>(mean),
               const_cast<float *>(invstd));
  float a[4], mu[4], be[4];  // BN constants of z's columns zc0 + c .. (the split-halves view)
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float is = !mine ? 0.f : fold.part ? s_is[4 * cj + k] : invstd[zc0 + c + k];
    a[k] = mine ? gamma[zc0 + c + k] * is : 0.f;
    mu[k] = !mine ? 0.f : fold.part ? s_mu[4 * cj + k] : mean[zc0 + c + k];
    be[k] = mine ? beta[zc0 + c + k] : 0.f;
  }
  uint32_t ph0 = 0, ph1 = 0;
  int s = 0;
  for (int64_t k = 0; k < nchunk; ++k, s ^= 1) {
    if (t == 0 && k + 1 < nchunk) issue(k + 1, s ^ 1);
    tc::mbar_wait(&full[s], s ? ph1 : ph0);
    if (s) ph1 ^= 1; else ph0 ^= 1;
    const int64_t a0 = r0 + k * Rc;
    const int rows = (int)min((int64_t)Rc, r1 - a0);
    const uint8_t *st = ring + s * sbytes;
    if (mine) {
      for (int i = rgi; i < rows; i += RG) {
        const int64_t m = a0 + i;
        const float4 zv = ld4(reinterpret_cast<const TZ *>(st), (int64_t)i * CT + 4 * cj);
        const float4 av = has_acc ? *reinterpret_cast<const float4 *>(st + zb + ((size_t)i * CT + 4 * cj) * 4)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
        float4 o;
        float *op = &o.x;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float y = fmaf(a[q], f4(zv, q) - mu[q], be[q]);
          if (relu) y = y > 0.f ? y : 0.f;
          op[q] = sign * y;
        }
        o.x += av.x; o.y += av.y; o.z += av.z; o.w += av.w;
        if (out) st4(out, m * C + c, o);
        if (out_bf16) st4(out_bf16, pad_row(m, pm) * C + c, o);
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- backward reduce (+ reconstruction)
template <typename TZ>
__global__ void __launch_bounds__(RT_BWD) bn_bwd_reduce_kernel(
    const TZ *__restrict__ z, int64_t M, int C, int CT, int TPR, int RG, int64_t rpb, int nrb,
    const float *__restrict__ mean, const float *__restrict__ invstd, const float *__restrict__ gamma,
    const float *__restrict__ beta, int relu, const float *dy0, const float *dy1, int cs, const float *dst_in,
    float *dst_out, __nv_bfloat16 *dst_bf16, int pH, int pW, double *__restrict__ part,
    unsigned *__restrict__ counter, float *__restrict__ dgamma, float *__restrict__ dbeta) {
  pdl_wait_trigger();
  const PadMap pm = pad_map(pH, pW);
  constexpr int RT = RT_BWD;
  __shared__ double sh[RT][4];
  const int t = threadIdx.x, cj = t % TPR, rgi = t / TPR;
  const int c0 = blockIdx.y * CT;
  const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = min(M, r0 + rpb);
  double sg[4] = {0, 0, 0, 0}, sgx[4] = {0, 0, 0, 0};
  const bool vec = (C % 4 == 0) && (dy1 == nullptr || cs % 4 == 0);
  const int c = vec ? c0 + 4 * cj : c0 + cj;
  if (c < C && rgi < RG) {
    if (vec) {
      float mu[4], is[4], ga[4], be[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        mu[k] = mean[c + k];
        is[k] = invstd[c + k];
        ga[k] = gamma[c + k];
        be[k] = beta[c + k];
      }
      auto row = [&](int64_t r, const float4 &zv, float4 g4, float4 d4) {
        float *gp = &g4.x, *dp = &d4.x;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float xh = (f4(zv, k) - mu[k]) * is[k];
          float y = fmaf(ga[k], xh, be[k]);
          float g = gp[k];
          if (relu) {
            if (!(y > 0.f)) g = 0.f;
            y = y > 0.f ? y : 0.f;
          }
          dp[k] -= y;
          sg[k] += (double)g;
          sgx[k] += (double)g * (double)xh;
        }
        if (dst_out) {
          st4(dst_out, r * C + c, d4);
          if (dst_bf16) st4(dst_bf16, pad_row(r, pm) * C + c, d4);
        }
      };
      int64_t r = r0 + rgi;
      for (; r + 3 * RG < r1; r += 4 * RG) {  // all loads of 4 rows first
        float4 zv[4], g4[4], d4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t ru = r + u * RG;
          zv[u] = ld4(z, ru * C + c);
          g4[u] = load_dy4(dy0, dy1, cs, C, ru, c);
          d4[u] = dst_out ? ld4(dst_in, ru * C + c) : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) row(r + u * RG, zv[u], g4[u], d4[u]);
      }
      for (; r < r1; r += RG) {
        float4 zv = ld4(z, r * C + c);
        float4 g4 = load_dy4(dy0, dy1, cs, C, r, c);
        float4 d4 = dst_out ? ld4(dst_in, r * C + c) : make_float4(0, 0, 0, 0);
        row(r, zv, g4, d4);
      }
    } else {
      const float mu = mean[c], is = invstd[c], ga = gamma[c], be = beta[c];
      for (int64_t r = r0 + rgi; r < r1; r += RG) {
        float xh = (ldv(z, r * C + c) - mu) * is;
        float y = fmaf(ga, xh, be);
        float g = load_dy(dy0, dy1, cs, C, r, c);
        if (relu) {
          if (!(y > 0.f)) g = 0.f;
          y = y > 0.f ? y : 0.f;
        }
        if (dst_out) {
          float o = dst_in[r * C + c] - y;
          dst_out[r * C + c] = o;
          if (dst_bf16) dst_bf16[pad_row(r, pm) * C + c] = __float2bfloat16_rn(o);
        }
        sg[0] += (double)g;
        sgx[0] += (double)g * (double)xh;
      }
    }
  }
  write_partial<RT>(sh, sg, sgx, vec, TPR, RG, c0, C, part);
  if (!last_block(counter, nrb)) return;
  double a, b;
  merge_tile<RT>(part, nrb, C, c0, CT, sh, a, b);
  const int ch = c0 + t;
  if (t < CT && ch < C) {
    dbeta[ch] = (float)a;
    dgamma[ch] = (float)b;
  }
  if (t == 0) counter[blockIdx.y] = 0u;
}


// BN backward reduce, TMA-staged: per chunk of Rc rows the block's z / dy (/ dst_in)
// tiles for its channel tile arrive by one 2-D TMA load each (box CT x Rc) into an
// S-stage smem ring (S - 1 chunks in flight while one is computed; one block per SM, so
// the ring depth is what covers the DRAM latency).  Every thread keeps the (rows, channels) it has in
// bn_bwd_reduce_kernel and adds them in the same order (chunks are whole multiples of
// the row-group count), so the sums -- and the partial rows / merge that follow -- are
// bitwise those of the register-loading kernel.
template <typename TZ>
__global__ void __launch_bounds__(RT_BWD) bn_bwd_reduce_tma_kernel(
    const __grid_constant__ CUtensorMap tmZ, const __grid_constant__ CUtensorMap tmY,
    const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmY1, int cs, int64_t M, int C,
    int CT, int TPR, int RG, int64_t rpb, int nrb, int Rc, int S,
    const float *__restrict__ mean, const float *__restrict__ invstd, const float *__restrict__ gamma,
    const float *__restrict__ beta, int relu, int has_dst, float *dst_out, __nv_bfloat16 *dst_bf16, int pH, int pW,
    double *__restrict__ part, unsigned *__restrict__ counter, float *__restrict__ dgamma,
    float *__restrict__ dbeta, const StatsFold fold) {
  pdl_wait_trigger();
  const PadMap pm = pad_map(pH, pW);
  constexpr int RT = RT_BWD;
  __shared__ double sh[RT][4];
  __shared__ uint64_t full[kMaxRing];  // S <= kMaxRing stages in flight (one block per SM)
  __shared__ float s_mu[128], s_is[128];
  extern __shared__ __align__(128) uint8_t ring[];
  const int t = threadIdx.x, cj = t % TPR, rgi = t / TPR;
  const int c0 = blockIdx.y * CT;
  const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = min(M, r0 + rpb);
  double sg[4] = {0, 0, 0, 0}, sgx[4] = {0, 0, 0, 0};
  const int c = c0 + 4 * cj;
  const bool mine = c < C && rgi < RG;
  const uint32_t zb = (uint32_t)Rc * CT * sizeof(TZ), fb = (uint32_t)Rc * CT * 4;
  const uint32_t sbytes = (zb + fb + (has_dst ? fb : 0) + 127) & ~127u;
  if (t == 0) {
    for (int q = 0; q < S; ++q) tc::mbar_init(&full[q], 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  const int64_t nchunk = (r1 - r0 + Rc - 1) / Rc;
  auto issue = [&](int64_t k, int s) {  // thread 0
    const int y = (int)(r0 + k * Rc);
    uint8_t *st = ring + s * sbytes;
    tc::mbar_arrive_expect_tx(&full[s], zb + fb + (has_dst ? fb : 0));
    tc::tma_load_2d(st, &tmZ, &full[s], c0, y);
    if (cs) {  // split halves (the stem): [Rc][cs] from dy0, then [Rc][C - cs] from dy1 (one tile = all C)
      tc::tma_load_2d(st + zb, &tmY, &full[s], 0, y);
      tc::tma_load_2d(st + zb + (size_t)Rc * cs * 4, &tmY1, &full[s], 0, y);
    } else {
      tc::tma_load_2d(st + zb, &tmY, &full[s], c0, y);
    }
    if (has_dst) tc::tma_load_2d(st + zb + fb, &tmD, &full[s], c0, y);
  };
  if (t == 0)  // the first S-1 chunks stream in while the statistics merge
    for (int q = 0; q < S - 1 && q < nchunk; ++q) issue(q, q);
  if (fold.part)
    fold_stats(fold, c0, min(CT, C - c0), s_mu, s_is, blockIdx.x == 0, const_cast<float *>(mean),
               const_cast<float *>(invstd));
  float mu[4], is[4], ga[4], be[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    mu[k] = !mine ? 0.f : fold.part ? s_mu[4 * cj + k] : mean[c + k];
    is[k] = !mine ? 0.f : fold.part ? s_is[4 * cj + k] : invstd[c + k];
    ga[k] = mine ? gamma[c + k] : 0.f;
    be[k] = mine ? beta[c + k] : 0.f;
  }
  uint32_t phases = 0;  // bit q: parity of stage q's next completion
  int s = 0;
  for (int64_t k = 0; k < nchunk; ++k, s = (s + 1 == S) ? 0 : s + 1) {
    // chunk k + S - 1 goes into the stage chunk k - 1 released at the end of the last iteration
    if (t == 0 && k + S - 1 < nchunk) issue(k + S - 1, (int)((k + S - 1) % S));
    tc::mbar_wait(&full[s], (phases >> s) & 1u);
    phases ^= 1u << s;
    const int64_t a0 = r0 + k * Rc;
    const int rows = (int)min((int64_t)Rc, r1 - a0);
    const uint8_t *st = ring + s * sbytes;
    if (mine) {
      for (int i = rgi; i < rows; i += RG) {
        const int64_t r = a0 + i;
        const float4 zv = ld4(reinterpret_cast<const TZ *>(st), (int64_t)i * CT + 4 * cj);
        const size_t yo = !cs ? (size_t)i * CT + 4 * cj
                              : (4 * cj < cs ? (size_t)i * cs + 4 * cj
                                             : (size_t)Rc * cs + (size_t)i * (C - cs) + 4 * cj - cs);
        float4 g4 = *reinterpret_cast<const float4 *>(st + zb + yo * 4);
        float4 d4 = has_dst ? *reinterpret_cast<const float4 *>(st + zb + fb + ((size_t)i * CT + 4 * cj) * 4)
                            : make_float4(0, 0, 0, 0);
        float *gp = &g4.x, *dp = &d4.x;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float xh = (f4(zv, q) - mu[q]) * is[q];
          float y = fmaf(ga[q], xh, be[q]);
          float g = gp[q];
          if (relu) {
            if (!(y > 0.f)) g = 0.f;
            y = y > 0.f ? y : 0.f;
          }
          dp[q] -= y;
          sg[q] += (double)g;
          sgx[q] += (double)g * (double)xh;
        }
        if (has_dst) {
          st4(dst_out, r * C + c, d4);
          if (dst_bf16) st4(dst_bf16, pad_row(r, pm) * C + c, d4);
        }
      }
    }
    __syncthreads();  // stage s read by every thread before it is refilled
  }
  write_partial<RT>(sh, sg, sgx, true, TPR, RG, c0, C, part);
  if (!last_block(counter, nrb)) return;
  double a, b;
  merge_tile<RT>(part, nrb, C, c0, CT, sh, a, b);
  const int ch = c0 + t;
  if (t < CT && ch < C) {
    dbeta[ch] = (float)a;
    dgamma[ch] = (float)b;
  }
  if (t == 0) counter[blockIdx.y] = 0u;
}


// BN backward dz, TMA-staged per channel tile (bitwise the arithmetic of
// bn_bwd_dz_fixed_kernel): thread (cj, rgi) keeps channels c0 + 4cj .. +3 and their
// constants in registers and takes rows rgi, rgi + RG, ... of each chunk; the z / dy
// tiles (box CT x Rc) arrive by TMA into a two-stage smem ring.
template <typename TZ>
__global__ void __launch_bounds__(256) bn_bwd_dz_tma_kernel(
    const __grid_constant__ CUtensorMap tmZ, const __grid_constant__ CUtensorMap tmY,
    const __grid_constant__ CUtensorMap tmY1, int cs, int64_t M, int C, int CT, int TPR, int RG, int64_t rpb, int Rc, const float *__restrict__ mean, const float *__restrict__ invstd,
    const float *__restrict__ gamma, const float *__restrict__ beta, int relu, const float *__restrict__ dgamma,
    const float *__restrict__ dbeta, float *__restrict__ dz, __nv_bfloat16 *__restrict__ dz_bf16, int pH, int pW) {
  pdl_wait_trigger();
  const PadMap pm = pad_map(pH, pW);
  __shared__ uint64_t full[2];
  extern __shared__ __align__(128) uint8_t ring[];
  const int t = threadIdx.x, cj = t % TPR, rgi = t / TPR;
  const int c0 = blockIdx.y * CT;
  const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = min(M, r0 + rpb);
  const int c = c0 + 4 * cj;
  const bool mine = c < C && rgi < RG;
  const float invM = 1.0f / (float)M;
  const uint32_t zb = (uint32_t)Rc * CT * sizeof(TZ), fb = (uint32_t)Rc * CT * 4;
  const uint32_t sbytes = (zb + fb + 127) & ~127u;
  if (t == 0) {
    tc::mbar_init(&full[0], 1);
    tc::mbar_init(&full[1], 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  float is[4], mu[4], ga[4], be[4], db[4], dg[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    is[k] = mine ? invstd[c + k] : 0.f;
    mu[k] = mine ? mean[c + k] : 0.f;
    ga[k] = mine ? gamma[c + k] : 0.f;
    be[k] = mine ? beta[c + k] : 0.f;
    db[k] = mine ? dbeta[c + k] * invM : 0.f;
    dg[k] = mine ? dgamma[c + k] : 0.f;
  }
  const int64_t nchunk = (r1 - r0 + Rc - 1) / Rc;
  auto issue = [&](int64_t k, int s) {
    const int y = (int)(r0 + k * Rc);
    uint8_t *st = ring + s * sbytes;
    tc::mbar_arrive_expect_tx(&full[s], zb + fb);
    tc::tma_load_2d(st, &tmZ, &full[s], c0, y);
    if (cs) {  // split halves: see bn_bwd_reduce_tma_kernel
      tc::tma_load_2d(st + zb, &tmY, &full[s], 0, y);
      tc::tma_load_2d(st + zb + (size_t)Rc * cs * 4, &tmY1, &full[s], 0, y);
    } else {
      tc::tma_load_2d(st + zb, &tmY, &full[s], c0, y);
    }
  };
  if (t == 0 && nchunk > 0) issue(0, 0);
  uint32_t ph0 = 0, ph1 = 0;
  int s = 0;
  for (int64_t k = 0; k < nchunk; ++k, s ^= 1) {
    if (t == 0 && k + 1 < nchunk) issue(k + 1, s ^ 1);
    tc::mbar_wait(&full[s], s ? ph1 : ph0);
    if (s) ph1 ^= 1; else ph0 ^= 1;
    const int64_t a0 = r0 + k * Rc;
    const int rows = (int)min((int64_t)Rc, r1 - a0);
    const uint8_t *st = ring + s * sbytes;
    if (mine) {
      for (int i = rgi; i < rows; i += RG) {
        const int64_t m = a0 + i;
        const float4 zv = ld4(reinterpret_cast<const TZ *>(st), (int64_t)i * CT + 4 * cj);
        const size_t yo = !cs ? (size_t)i * CT + 4 * cj
                              : (4 * cj < cs ? (size_t)i * cs + 4 * cj
                                             : (size_t)Rc * cs + (size_t)i * (C - cs) + 4 * cj - cs);
        float4 g4 = *reinterpret_cast<const float4 *>(st + zb + yo * 4);
        float4 o;
        float *op = &o.x, *gp = &g4.x;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float xh = (f4(zv, q) - mu[q]) * is[q];
          float g = gp[q];
          if (relu && !(fmaf(ga[q], xh, be[q]) > 0.f)) g = 0.f;
          op[q] = ga[q] * is[q] * (g - db[q] - xh * dg[q] * invM);  // same rounding as bn_bwd_dz_kernel
        }
        if (dz) st4(dz, m * C + c, o);
        if (dz_bf16) st4(dz_bf16, pad_row(m, pm) * C + c, o);
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- dz
template <typename TZ>
__global__ void bn_bwd_dz_kernel(int64_t M, int C, const TZ *__restrict__ z, const float *__restrict__ mean,
                                 const float *__restrict__ invstd, const float *__restrict__ gamma,
                                 const float *__restrict__ beta, int relu, const float *dy0, const float *dy1,
                                 int cs, const float *__restrict__ dgamma, const float *__restrict__ dbeta,
                                 float *__restrict__ dz, __nv_bfloat16 *__restrict__ dz_bf16, int pH, int pW,
                                 int sh) {
  pdl_wait_trigger();
  const PadMap pm = pad_map(pH, pW);
  const float invM = 1.0f / (float)M;
  const bool vec = (C % 4 == 0) && (dy1 == nullptr || cs % 4 == 0);
  if (vec) {
    const int C4 = C / 4;
    const int64_t n = M * C4;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      int64_t m = row_of(i, C4, sh);
      int c = (int)(i - m * C4) * 4;
      float4 zv = ld4(z, m * C + c);
      float4 g4 = load_dy4(dy0, dy1, cs, C, m, c);
      float4 o;
      float *op = &o.x, *gp = &g4.x;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float is = invstd[c + k];
        float xh = (f4(zv, k) - mean[c + k]) * is;
        float g = gp[k];
        if (relu && !(fmaf(gamma[c + k], xh, beta[c + k]) > 0.f)) g = 0.f;
        op[k] = gamma[c + k] * is * (g - dbeta[c + k] * invM - xh * dgamma[c + k] * invM);
      }
      if (dz) st4(dz, m * C + c, o);
      if (dz_bf16) st4(dz_bf16, pad_row(m, pm) * C + c, o);
    }
    return;
  }
  const int64_t n = M * C;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t m = i / C;
    int c = (int)(i - m * C);
    float is = invstd[c];
    float xh = (ldv(z, i) - mean[c]) * is;
    float g = load_dy(dy0, dy1, cs, C, m, c);
    if (relu && !(fmaf(gamma[c], xh, beta[c]) > 0.f)) g = 0.f;
    float v = gamma[c] * is * (g - dbeta[c] * invM - xh * dgamma[c] * invM);
    if (dz) stv(dz, i, v);
    if (dz_bf16) dz_bf16[pad_row(m, pm) * C + c] = __float2bfloat16_rn(v);
  }
}

// a byte offset inside a TMA ring stage that can start a tensor-copy destination
inline bool ring_aligned(size_t bytes) { return bytes % 128 == 0; }

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

// grid of a per-channel elementwise pass over M x C (256 threads, 4 channels each):
// a multiple of q = (C/4) / gcd(C/4, 256) blocks, so the grid stride is a multiple of
// C/4 and every thread keeps one channel group; 0 if C % 4 or q is unreasonable
inline unsigned chan_grid(int64_t M, int C) {
  if (C % 4) return 0;
  const int C4 = C / 4;
  int a = C4, b = 256;
  while (b) { const int t = a % b; a = b; b = t; }
  const int64_t q = C4 / a;
  if (q > 8 * kNumSMs) return 0;
  const int64_t g = ew_grid(M * C4);
  return (unsigned)std::max<int64_t>(q, g / q * q);
}

// the fold as a separate stats_finalize launch (the passes without a fused prologue)
void finalize_fold(const StatsFold &f, float *mean, float *invstd, cudaStream_t st) {
  StatsRows r;
  r.rows = f.rows;
  r.groups = f.groups;
  bn_stats_from_partials(f.part, r, f.N, f.M, f.eps, mean, invstd, f.rmean, f.rvar, f.mom, st);
}

__global__ void running_constants_kernel(const float *__restrict__ rm, const float *__restrict__ rv, int C, float eps,
                                         float *__restrict__ mean, float *__restrict__ invstd) {
  pdl_wait_trigger();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < C) {
    mean[c] = rm[c];
    invstd[c] = (float)(1.0 / sqrt((double)rv[c] + (double)eps));
  }
}

}  // namespace

void bn_running_constants(const float *rm, const float *rv, int C, float eps, float *mean, float *invstd,
                          cudaStream_t st) {
  launch_k(running_constants_kernel, (unsigned)cdiv(C, 256), 256, 0, st, rm, rv, C, eps, mean, invstd);
  PETRA_LAUNCH_CHECK();
}

size_t bn_partial_bytes(int64_t M, int C) {
  return (size_t)std::max(red_geom(M, C, RT_STATS).nrb, red_geom(M, C, RT_BWD).nrb) * C * 2 * sizeof(double);
}
size_t bn_counter_count(int C) { return (size_t)red_geom(1 << 20, C, RT_BWD).ctiles; }

template <typename TZ>
void bn_stats(const TZ *z, int64_t M, int C, float eps, float *mean, float *invstd, float *rmean, float *rvar,
              float mom, double *part, unsigned *counter, cudaStream_t st) {
  RedGeom g = red_geom(M, C, RT_STATS);
  launch_k(bn_stats_kernel<TZ>, dim3(g.nrb, g.ctiles), RT_STATS, 0, st, z, M, C, g.CT, g.TPR, g.RG, g.rpb, g.nrb, part, counter,
                                                            eps, mean, invstd, rmean, rvar, mom);
  PETRA_LAUNCH_CHECK();
}
template void bn_stats<float>(const float *, int64_t, int, float, float *, float *, float *, float *, float,
                              double *, unsigned *, cudaStream_t);
template void bn_stats<__nv_bfloat16>(const __nv_bfloat16 *, int64_t, int, float, float *, float *, float *,
                                      float *, float, double *, unsigned *, cudaStream_t);

template <typename TZ, typename TO>
void bn_apply(int64_t M, int C, const TZ *z, int ldz, int zc0, const float *mean, const float *invstd,
              const float *gamma, const float *beta, int relu, float sign, const float *acc, TO *out,
              __nv_bfloat16 *out_bf16, int pH, int pW, cudaStream_t st, const StatsFold *fold) {
  static const bool tma_on = env_int("PETRA_BN_TMA_APPLY", 1) != 0;
  if (tma_on && std::is_same<TO, float>::value && C % 8 == 0 && (uintptr_t)(z + zc0) % 16 == 0 &&
      ((size_t)ldz * sizeof(TZ)) % 16 == 0 && (uintptr_t)acc % 16 == 0 && M < ((int64_t)1 << 31)) {
    static const int per_sm = env_int("PETRA_BN_PER_SM", 2), chunk = env_int("PETRA_BN_CHUNK", 24576);
    RedGeom g = red_geom(M, C, 256, per_sm);
    const int es = (int)sizeof(TZ) + (acc ? 4 : 0);
    const int Rc = std::min(256 / g.RG * g.RG, std::max(g.RG, (chunk / (g.CT * es)) / g.RG * g.RG));
    const size_t sbytes = (((size_t)Rc * g.CT * es) + 127) & ~(size_t)127;
    // every TMA destination inside a ring stage must be 128-byte aligned (else the register kernel)
    const bool ring_ok = ring_aligned((size_t)Rc * g.CT * sizeof(TZ)) && g.CT % 8 == 0;
    if (ring_ok) {
      static std::once_flag once;
      std::call_once(once, [] {
        cudaFuncSetAttribute(bn_apply_tma_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        cudaFuncSetAttribute(bn_apply_tma_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             160 * 1024);
      });
      const CUtensorMapDataType zt = sizeof(TZ) == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
      // z: [M][C] view of a [M][ldz] buffer from column zc0
      const CUtensorMap tz = plain_map_2d_strided(z + zc0, zt, (int)sizeof(TZ), M, C, ldz, g.CT, Rc);
      const CUtensorMap ta = acc ? plain_map_2d(acc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, M, C, g.CT, Rc) : tz;
      launch_k(bn_apply_tma_kernel<TZ>, dim3(g.nrb, g.ctiles), 256, 2 * sbytes, st, tz, ta, acc ? 1 : 0, M, C, g.CT,
               g.TPR, g.RG, g.rpb, Rc, zc0, mean, invstd, gamma, beta, relu, sign, reinterpret_cast<float *>(out), out_bf16,
               pH, pW, fold ? *fold : StatsFold{});
      PETRA_LAUNCH_CHECK();
      return;
    }
  }
  if (fold) finalize_fold(*fold, const_cast<float *>(mean), const_cast<float *>(invstd), st);  // the register kernels read final statistics
  const unsigned cg = (ldz % 4 == 0 && zc0 % 4 == 0) ? chan_grid(M, C) : 0;
  if (cg && std::is_same<TO, float>::value && M < ((int64_t)1 << 31) / 4) {
    launch_k(bn_apply_fixed_kernel<TZ>, cg, 256, 0, st, (int)M, C, z, ldz, zc0, mean, invstd, gamma, beta, relu, sign,
             acc, reinterpret_cast<float *>(out), out_bf16, pH, pW);
  } else {
    launch_k(bn_apply_kernel<TZ, TO>, ew_grid(M * C / 4), 256, 0, st, M, C, z, ldz, zc0, mean, invstd, gamma, beta,
             relu, sign, acc, out, out_bf16, pH, pW, log2_or_neg(C / 4));
  }
  PETRA_LAUNCH_CHECK();
}
template void bn_apply<float, float>(int64_t, int, const float *, int, int, const float *, const float *,
                                     const float *, const float *, int, float, const float *, float *,
                                     __nv_bfloat16 *, int, int, cudaStream_t, const StatsFold *);
template void bn_apply<__nv_bfloat16, float>(int64_t, int, const __nv_bfloat16 *, int, int, const float *,
                                             const float *, const float *, const float *, int, float,
                                             const float *, float *, __nv_bfloat16 *, int, int, cudaStream_t,
                                             const StatsFold *);

template <typename TZ>
void bn_bwd_reduce(const TZ *z, int64_t M, int C, const float *mean, const float *invstd, const float *gamma,
                   const float *beta, int relu, const float *dy0, const float *dy1, int cs, const float *dst_in,
                   float *dst_out, __nv_bfloat16 *dst_bf16, int pH, int pW, float *dgamma, float *dbeta,
                   double *part, unsigned *counter, cudaStream_t st, const StatsFold *fold) {
  RedGeom g = red_geom(M, C, RT_BWD);
  static const bool tma_on = env_int("PETRA_BN_TMA_REDUCE", 1) != 0;
  const bool aligned = (uintptr_t)z % 16 == 0 && (uintptr_t)dy0 % 16 == 0 && (uintptr_t)dst_in % 16 == 0 &&
                       (uintptr_t)dy1 % 16 == 0;
  // split dy halves (the stem): one channel tile covering both (same geometry as the register kernel)
  const bool split_ok = dy1 == nullptr || (g.ctiles == 1 && cs % 4 == 0 && (C - cs) % 4 == 0 && cs > 0 && cs < C);
  if (tma_on && split_ok && C % 8 == 0 && aligned && g.CT % 8 == 0 && M < ((int64_t)1 << 31)) {
    const int es = (int)sizeof(TZ) + 4 + (dst_out ? 4 : 0);
    static const int rchunk = env_int("PETRA_BN_RCHUNK", 40960);
    const int Rc = std::min(256 / g.RG * g.RG, std::max(g.RG, (rchunk / (g.CT * es)) / g.RG * g.RG));
    const size_t sbytes = (((size_t)Rc * g.CT * es) + 127) & ~(size_t)127;
    // ring depth: one block per SM, so the stages in flight are what hides the DRAM latency
    static const int ring = std::max(2, std::min(kMaxRing, env_int("PETRA_BN_REDUCE_STAGES", 2)));
    const int S = (size_t)ring * sbytes <= 180 * 1024 ? ring : 2;
    // every TMA destination inside a ring stage must be 128-byte aligned (else the register kernel)
    const bool ring_ok = ring_aligned((size_t)Rc * g.CT * sizeof(TZ)) && ring_aligned((size_t)Rc * g.CT * 4) &&
                         (!dy1 || ring_aligned((size_t)Rc * cs * 4));
    if (ring_ok) {
      static std::once_flag once;
      std::call_once(once, [] {
        cudaFuncSetAttribute(bn_bwd_reduce_tma_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 184 * 1024);
        cudaFuncSetAttribute(bn_bwd_reduce_tma_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             184 * 1024);
      });
      const CUtensorMapDataType zt = sizeof(TZ) == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
      const CUtensorMap tz = plain_map_2d(z, zt, (int)sizeof(TZ), M, C, g.CT, Rc);
      const int s0 = dy1 ? cs : 0;
      const CUtensorMap ty = dy1 ? plain_map_2d(dy0, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, M, cs, cs, Rc)
                                 : plain_map_2d(dy0, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, M, C, g.CT, Rc);
      const CUtensorMap ty1 = dy1 ? plain_map_2d(dy1, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, M, C - cs, C - cs, Rc) : ty;
      const CUtensorMap td = dst_out ? plain_map_2d(dst_in, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, M, C, g.CT, Rc) : ty;
      launch_k(bn_bwd_reduce_tma_kernel<TZ>, dim3(g.nrb, g.ctiles), RT_BWD, S * sbytes, st, tz, ty, td, ty1, s0, M, C,
               g.CT,
               g.TPR, g.RG, g.rpb, g.nrb, Rc, S, mean, invstd, gamma, beta, relu, dst_out ? 1 : 0, dst_out, dst_bf16, pH,
               pW, part, counter, dgamma, dbeta, fold ? *fold : StatsFold{});
      PETRA_LAUNCH_CHECK();
      return;
    }
  }
  if (fold) finalize_fold(*fold, const_cast<float *>(mean), const_cast<float *>(invstd), st);
  launch_k(bn_bwd_reduce_kernel<TZ>, dim3(g.nrb, g.ctiles), RT_BWD, 0, st, z, M, C, g.CT, g.TPR, g.RG, g.rpb, g.nrb, mean,
                                                                 invstd, gamma, beta, relu, dy0, dy1, cs, dst_in,
                                                                 dst_out, dst_bf16, pH, pW, part, counter, dgamma,
                                                                 dbeta);
  PETRA_LAUNCH_CHECK();
}
template void bn_bwd_reduce<float>(const float *, int64_t, int, const float *, const float *, const float *,
                                   const float *, int, const float *, const float *, int, const float *, float *,
                                   __nv_bfloat16 *, int, int, float *, float *, double *, unsigned *, cudaStream_t,
                                   const StatsFold *);
template void bn_bwd_reduce<__nv_bfloat16>(const __nv_bfloat16 *, int64_t, int, const float *, const float *,
                                           const float *, const float *, int, const float *, const float *, int,
                                           const float *, float *, __nv_bfloat16 *, int, int, float *, float *,
                                           double *, unsigned *, cudaStream_t, const StatsFold *);

template <typename TZ>
void bn_bwd_dz(int64_t M, int C, const TZ *z, const float *mean, const float *invstd, const float *gamma,
               const float *beta, int relu, const float *dy0, const float *dy1, int cs, const float *dgamma,
               const float *dbeta, float *dz, __nv_bfloat16 *dz_bf16, int pH, int pW, cudaStream_t st) {
  static const bool tma_on = env_int("PETRA_BN_TMA_DZ", 1) != 0;
  static const int per_sm = env_int("PETRA_BN_PER_SM", 2), chunk = env_int("PETRA_BN_CHUNK", 24576);
  const RedGeom gs = red_geom(M, C, 256, per_sm);
  const bool split_ok = dy1 == nullptr || (gs.ctiles == 1 && cs % 4 == 0 && (C - cs) % 4 == 0 && cs > 0 && cs < C);
  if (tma_on && split_ok && C % 8 == 0 && (uintptr_t)z % 16 == 0 && (uintptr_t)dy0 % 16 == 0 &&
      (uintptr_t)dy1 % 16 == 0 && M < ((int64_t)1 << 31)) {
    const RedGeom &g = gs;
    const int es = (int)sizeof(TZ) + 4;
    const int Rc = std::min(256 / g.RG * g.RG, std::max(g.RG, (chunk / (g.CT * es)) / g.RG * g.RG));
    const size_t sbytes = (((size_t)Rc * g.CT * es) + 127) & ~(size_t)127;
    // every TMA destination inside a ring stage must be 128-byte aligned (else the register kernel)
    const bool ring_ok = ring_aligned((size_t)Rc * g.CT * sizeof(TZ)) && g.CT % 8 == 0 &&
                         (!dy1 || ring_aligned((size_t)Rc * cs * 4));
    if (ring_ok) {
      static std::once_flag once;
      std::call_once(once, [] {
        cudaFuncSetAttribute(bn_bwd_dz_tma_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        cudaFuncSetAttribute(bn_bwd_dz_tma_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             160 * 1024);
      });
      const CUtensorMapDataType zt = sizeof(TZ) == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
      const CUtensorMap tz = plain_map_2d(z, zt, (int)sizeof(TZ), M, C, g.CT, Rc);
      const int s0 = dy1 ? cs : 0;
      const CUtensorMap ty = dy1 ? plain_map_2d(dy0, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, M, cs, cs, Rc)
                                 : plain_map_2d(dy0, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, M, C, g.CT, Rc);
      const CUtensorMap ty1 = dy1 ? plain_map_2d(dy1, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, M, C - cs, C - cs, Rc) : ty;
      launch_k(bn_bwd_dz_tma_kernel<TZ>, dim3(g.nrb, g.ctiles), 256, 2 * sbytes, st, tz, ty, ty1, s0, M, C, g.CT, g.TPR,
               g.RG,
               g.rpb, Rc, mean, invstd, gamma, beta, relu, dgamma, dbeta, dz, dz_bf16, pH, pW);
      PETRA_LAUNCH_CHECK();
      return;
    }
  }
  const unsigned cg = dy1 == nullptr ? chan_grid(M, C) : 0;  // split halves (stem): generic pass
  if (cg && M < ((int64_t)1 << 31) / 4)
    launch_k(bn_bwd_dz_fixed_kernel<TZ>, cg, 256, 0, st, (int)M, C, z, mean, invstd, gamma, beta, relu, dy0, dgamma,
             dbeta, dz, dz_bf16, pH, pW);
  else
    launch_k(bn_bwd_dz_kernel<TZ>, ew_grid(M * C / 4), 256, 0, st, M, C, z, mean, invstd, gamma, beta, relu, dy0, dy1,
             cs, dgamma, dbeta, dz, dz_bf16, pH, pW, log2_or_neg(C / 4));
  PETRA_LAUNCH_CHECK();
}
template void bn_bwd_dz<float>(int64_t, int, const float *, const float *, const float *, const float *,
                               const float *, int, const float *, const float *, int, const float *, const float *,
                               float *, __nv_bfloat16 *, int, int, cudaStream_t);
template void bn_bwd_dz<__nv_bfloat16>(int64_t, int, const __nv_bfloat16 *, const float *, const float *,
                                       const float *, const float *, int, const float *, const float *, int,
                                       const float *, const float *, float *, __nv_bfloat16 *, int, int,
                                       cudaStream_t);

}  // namespace petra

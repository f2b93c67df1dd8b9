// bn.cu -- BatchNorm (training mode) + ReLU + additive coupling, HBM-streaming kernels.
//
//   stats    : mu_c, sigma2_c = biased batch mean / variance of z over all rows
//              (B*H*W), invstd = 1/sqrt(sigma2+eps); optional running-stat EMA
//              (only in the backward recomputation; reading c9).
//   apply    : out = acc + sign * act(gamma*(z-mu)*invstd + beta)
//              forward coupling (sign +1) / DS / stem / bottleneck
//              inner activations.
//   bwd_reduce: per channel  sum g,  sum g*xhat  with g = dy * 1[out > 0]
//              (= dbeta, dgamma), optionally fused with the reconstruction
//              dst_out = dst_in - act(bn(z))  (approximate inversion).
//   bwd_dz   : dz = gamma*invstd*(g - sum(g)/n - xhat*sum(g*xhat)/n).
// All reductions are deterministic: per-block fp64 partials merged in a fixed
// order by a finalize kernel (no float atomics).
#include "../kernels.h"

namespace petra {
namespace {

__device__ __forceinline__ float ldv(const float *p, int64_t i) { return p[i]; }
__device__ __forceinline__ float ldv(const __nv_bfloat16 *p, int64_t i) { return __bfloat162float(p[i]); }
__device__ __forceinline__ void stv(float *p, int64_t i, float v) { p[i] = v; }
__device__ __forceinline__ void stv(__nv_bfloat16 *p, int64_t i, float v) { p[i] = __float2bfloat16_rn(v); }

constexpr int RT = 256;  // threads per reduce block: 32 channels x 8 row-warps

inline int reduce_row_blocks(int64_t M, int C) {
  int ctiles = (int)cdiv(C, 32);
  int64_t want = std::max<int64_t>(1, (4 * kNumSMs) / ctiles);
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, cdiv(M, 32)));
}

template <typename TZ>
__global__ void __launch_bounds__(RT) bn_stats_partial_kernel(const TZ *__restrict__ z, int64_t M, int C,
                                                              int64_t rows_per_blk, double *__restrict__ part) {
  __shared__ double sh[2][8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.y * 32 + lane;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_blk;
  const int64_t r1 = min(M, r0 + rows_per_blk);
  double s = 0.0, ss = 0.0;
  if (c < C) {
    for (int64_t r = r0 + w; r < r1; r += 8) {
      double v = (double)ldv(z, r * C + c);
      s += v;
      ss += v * v;
    }
  }
  sh[0][w][lane] = s;
  sh[1][w][lane] = ss;
  __syncthreads();
  if (w == 0 && c < C) {
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) { a += sh[0][i][lane]; b += sh[1][i][lane]; }
    part[((int64_t)blockIdx.x * C + c) * 2 + 0] = a;
    part[((int64_t)blockIdx.x * C + c) * 2 + 1] = b;
  }
}

__global__ void bn_stats_finalize_kernel(const double *__restrict__ part, int nrb, int C, int64_t M,
                                         float eps, float *__restrict__ mean, float *__restrict__ invstd,
                                         float *__restrict__ rmean, float *__restrict__ rvar, float mom) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double s = 0.0, ss = 0.0;
  for (int i = 0; i < nrb; ++i) {
    s += part[((int64_t)i * C + c) * 2 + 0];
    ss += part[((int64_t)i * C + c) * 2 + 1];
  }
  double mu = s / (double)M;
  double var = ss / (double)M - mu * mu;
  if (var < 0.0) var = 0.0;
  mean[c] = (float)mu;
  invstd[c] = (float)(1.0 / sqrt(var + (double)eps));
  if (rmean) {
    double unb = M > 1 ? var * (double)M / (double)(M - 1) : var;
    rmean[c] = (float)((1.0 - mom) * rmean[c] + mom * mu);
    rvar[c] = (float)((1.0 - mom) * rvar[c] + mom * unb);
  }
}

template <typename TZ, typename TO>
__global__ void bn_apply_kernel(int64_t M, int C, const TZ *__restrict__ z, int ldz, int zc0,
                                const float *__restrict__ mean, const float *__restrict__ invstd,
                                const float *__restrict__ gamma, const float *__restrict__ beta, int relu,
                                float sign, const float *acc, TO *out, __nv_bfloat16 *out_bf16) {
  const int64_t n = M * C;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t m = i / C;
    int c = (int)(i - m * C);
    int cz = zc0 + c;
    float y = fmaf(gamma[cz] * invstd[cz], ldv(z, m * ldz + cz) - mean[cz], beta[cz]);
    if (relu) y = y > 0.f ? y : 0.f;
    float o = sign * y;
    if (acc) o += acc[i];
    stv(out, i, o);
    if (out_bf16) out_bf16[i] = __float2bfloat16_rn(o);
  }
}

// dy(m, c): single [M][C] tensor, or split halves dy0 = channels [0, cs), dy1 = [cs, C)
__device__ __forceinline__ float load_dy(const float *dy0, const float *dy1, int cs, int C, int64_t m, int c) {
  if (dy1 == nullptr) return dy0[m * C + c];
  return c < cs ? dy0[m * cs + c] : dy1[m * (C - cs) + (c - cs)];
}

template <typename TZ>
__global__ void __launch_bounds__(RT) bn_bwd_reduce_kernel(
    const TZ *__restrict__ z, int64_t M, int C, const float *__restrict__ mean, const float *__restrict__ invstd,
    const float *__restrict__ gamma, const float *__restrict__ beta, int relu, const float *dy0, const float *dy1,
    int cs, const float *dst_in, float *dst_out, __nv_bfloat16 *dst_bf16, int64_t rows_per_blk,
    double *__restrict__ part) {
  __shared__ double sh[2][8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.y * 32 + lane;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_blk;
  const int64_t r1 = min(M, r0 + rows_per_blk);
  double sg = 0.0, sgx = 0.0;
  if (c < C) {
    const float mu = mean[c], is = invstd[c], ga = gamma[c], be = beta[c];
    for (int64_t r = r0 + w; r < r1; r += 8) {
      float xh = (ldv(z, r * C + c) - mu) * is;
      float y = fmaf(ga, xh, be);
      float g = load_dy(dy0, dy1, cs, C, r, c);
      if (relu) {
        if (!(y > 0.f)) g = 0.f;
        y = y > 0.f ? y : 0.f;
      }
      if (dst_out) {
        float o = dst_in[r * C + c] - y;   // reconstruct: dst - Phi(src)
        dst_out[r * C + c] = o;
        if (dst_bf16) dst_bf16[r * C + c] = __float2bfloat16_rn(o);
      }
      sg += (double)g;
      sgx += (double)g * (double)xh;
    }
  }
  sh[0][w][lane] = sg;
  sh[1][w][lane] = sgx;
  __syncthreads();
  if (w == 0 && c < C) {
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) { a += sh[0][i][lane]; b += sh[1][i][lane]; }
    part[((int64_t)blockIdx.x * C + c) * 2 + 0] = a;
    part[((int64_t)blockIdx.x * C + c) * 2 + 1] = b;
  }
}

__global__ void bn_bwd_finalize_kernel(const double *__restrict__ part, int nrb, int C,
                                       float *__restrict__ dgamma, float *__restrict__ dbeta) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double a = 0.0, b = 0.0;
  for (int i = 0; i < nrb; ++i) {
    a += part[((int64_t)i * C + c) * 2 + 0];
    b += part[((int64_t)i * C + c) * 2 + 1];
  }
  dbeta[c] = (float)a;
  dgamma[c] = (float)b;
}

template <typename TZ, typename TO>
__global__ void bn_bwd_dz_kernel(int64_t M, int C, const TZ *__restrict__ z, const float *__restrict__ mean,
                                 const float *__restrict__ invstd, const float *__restrict__ gamma,
                                 const float *__restrict__ beta, int relu, const float *dy0, const float *dy1,
                                 int cs, const float *__restrict__ dgamma, const float *__restrict__ dbeta,
                                 TO *__restrict__ dz) {
  const int64_t n = M * C;
  const float invM = 1.0f / (float)M;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t m = i / C;
    int c = (int)(i - m * C);
    float is = invstd[c];
    float xh = (ldv(z, i) - mean[c]) * is;
    float g = load_dy(dy0, dy1, cs, C, m, c);
    if (relu && !(fmaf(gamma[c], xh, beta[c]) > 0.f)) g = 0.f;
    float v = gamma[c] * is * (g - dbeta[c] * invM - xh * dgamma[c] * invM);
    stv(dz, i, v);
  }
}

inline unsigned ew_grid(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 8 * kNumSMs));
}

}  // namespace

size_t bn_partial_bytes(int64_t M, int C) { return (size_t)reduce_row_blocks(M, C) * C * 2 * sizeof(double); }

template <typename TZ>
void bn_stats(const TZ *z, int64_t M, int C, float eps, float *mean, float *invstd, float *rmean, float *rvar,
              float mom, double *part, cudaStream_t st) {
  int nrb = reduce_row_blocks(M, C);
  int64_t rpb = cdiv(M, nrb);
  nrb = (int)cdiv(M, rpb);
  dim3 grid(nrb, (unsigned)cdiv(C, 32));
  bn_stats_partial_kernel<TZ><<<grid, RT, 0, st>>>(z, M, C, rpb, part);
  PETRA_LAUNCH_CHECK();
  bn_stats_finalize_kernel<<<(unsigned)cdiv(C, 128), 128, 0, st>>>(part, nrb, C, M, eps, mean, invstd, rmean,
                                                                   rvar, mom);
  PETRA_LAUNCH_CHECK();
}
template void bn_stats<float>(const float *, int64_t, int, float, float *, float *, float *, float *, float,
                              double *, cudaStream_t);
template void bn_stats<__nv_bfloat16>(const __nv_bfloat16 *, int64_t, int, float, float *, float *, float *,
                                      float *, float, double *, cudaStream_t);

template <typename TZ, typename TO>
void bn_apply(int64_t M, int C, const TZ *z, int ldz, int zc0, const float *mean, const float *invstd,
              const float *gamma, const float *beta, int relu, float sign, const float *acc, TO *out,
              __nv_bfloat16 *out_bf16, cudaStream_t st) {
  bn_apply_kernel<TZ, TO><<<ew_grid(M * C), 256, 0, st>>>(M, C, z, ldz, zc0, mean, invstd, gamma, beta, relu,
                                                          sign, acc, out, out_bf16);
  PETRA_LAUNCH_CHECK();
}
template void bn_apply<float, float>(int64_t, int, const float *, int, int, const float *, const float *,
                                     const float *, const float *, int, float, const float *, float *,
                                     __nv_bfloat16 *, cudaStream_t);
template void bn_apply<__nv_bfloat16, float>(int64_t, int, const __nv_bfloat16 *, int, int, const float *,
                                             const float *, const float *, const float *, int, float,
                                             const float *, float *, __nv_bfloat16 *, cudaStream_t);
template void bn_apply<float, __nv_bfloat16>(int64_t, int, const float *, int, int, const float *,
                                             const float *, const float *, const float *, int, float,
                                             const float *, __nv_bfloat16 *, __nv_bfloat16 *, cudaStream_t);
template void bn_apply<__nv_bfloat16, __nv_bfloat16>(int64_t, int, const __nv_bfloat16 *, int, int,
                                                     const float *, const float *, const float *,
                                                     const float *, int, float, const float *,
                                                     __nv_bfloat16 *, __nv_bfloat16 *, cudaStream_t);

template <typename TZ>
void bn_bwd_reduce(const TZ *z, int64_t M, int C, const float *mean, const float *invstd, const float *gamma,
                   const float *beta, int relu, const float *dy0, const float *dy1, int cs, const float *dst_in,
                   float *dst_out, __nv_bfloat16 *dst_bf16, float *dgamma, float *dbeta, double *part,
                   cudaStream_t st) {
  int nrb = reduce_row_blocks(M, C);
  int64_t rpb = cdiv(M, nrb);
  nrb = (int)cdiv(M, rpb);
  dim3 grid(nrb, (unsigned)cdiv(C, 32));
  bn_bwd_reduce_kernel<TZ><<<grid, RT, 0, st>>>(z, M, C, mean, invstd, gamma, beta, relu, dy0, dy1, cs, dst_in,
                                                dst_out, dst_bf16, rpb, part);
  PETRA_LAUNCH_CHECK();
  bn_bwd_finalize_kernel<<<(unsigned)cdiv(C, 128), 128, 0, st>>>(part, nrb, C, dgamma, dbeta);
  PETRA_LAUNCH_CHECK();
}
template void bn_bwd_reduce<float>(const float *, int64_t, int, const float *, const float *, const float *,
                                   const float *, int, const float *, const float *, int, const float *, float *,
                                   __nv_bfloat16 *, float *, float *, double *, cudaStream_t);
template void bn_bwd_reduce<__nv_bfloat16>(const __nv_bfloat16 *, int64_t, int, const float *, const float *,
                                           const float *, const float *, int, const float *, const float *, int,
                                           const float *, float *, __nv_bfloat16 *, float *, float *, double *,
                                           cudaStream_t);

template <typename TZ, typename TO>
void bn_bwd_dz(int64_t M, int C, const TZ *z, const float *mean, const float *invstd, const float *gamma,
               const float *beta, int relu, const float *dy0, const float *dy1, int cs, const float *dgamma,
               const float *dbeta, TO *dz, cudaStream_t st) {
  bn_bwd_dz_kernel<TZ, TO><<<ew_grid(M * C), 256, 0, st>>>(M, C, z, mean, invstd, gamma, beta, relu, dy0, dy1,
                                                           cs, dgamma, dbeta, dz);
  PETRA_LAUNCH_CHECK();
}
template void bn_bwd_dz<float, float>(int64_t, int, const float *, const float *, const float *, const float *,
                                      const float *, int, const float *, const float *, int, const float *,
                                      const float *, float *, cudaStream_t);
template void bn_bwd_dz<__nv_bfloat16, __nv_bfloat16>(int64_t, int, const __nv_bfloat16 *, const float *,
                                                      const float *, const float *, const float *, int,
                                                      const float *, const float *, int, const float *,
                                                      const float *, __nv_bfloat16 *, cudaStream_t);
template void bn_bwd_dz<float, __nv_bfloat16>(int64_t, int, const float *, const float *, const float *,
                                              const float *, const float *, int, const float *, const float *,
                                              int, const float *, const float *, __nv_bfloat16 *, cudaStream_t);

}  // namespace petra

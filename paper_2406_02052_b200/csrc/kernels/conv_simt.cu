// conv_simt.cu -- fp32 SIMT implicit-GEMM convolutions (forward, dgrad, wgrad).
//
// The fp32 parity path (PETRA_FP32): TF32 tensor cores cannot meet rel 1e-4
// (10-bit mantissa), so these run on the FFMA pipe.  On the bf16 path they serve
// the geometries the tensor-core kernels do not take (channel counts that are not
// multiples of 64, the MLP's linear layers): there (RND = true) every operand is
// rounded to bf16 on load and the forward result z to bf16 on store, so every
// convolution pass of PETRA_BF16_TC follows one rule whichever engine runs it
// (reading c22).  NHWC activations, weights [Co][k][k][Ci].
//
//   forward : z[m][co]   = sum_{kh,kw,ci} x[b][ho*s+kh-p][wo*s+kw-p][ci] * w[co][kh][kw][ci]
//   dgrad   : dx[m'][ci] = sum_{kh,kw,co} dz[b][(h+p-kh)/s][(w+p-kw)/s][co] * w[co][kh][kw][ci]
//             (terms with non-integral or out-of-range output coordinates vanish)
//   wgrad   : dw[co][kh][kw][ci] = sum_{b,ho,wo} dz[b][ho][wo][co] * x[b][ho*s+kh-p][wo*s+kw-p][ci]
// (the VJP of the conv, Eqs. 2-3 applied per layer).  wgrad uses a
// deterministic split-K: per-split partial tiles, reduced in fixed order.
#include "../kernels.h"

namespace petra {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 256;
enum { FWD = 0, DGRAD = 1, WGRAD = 2 };

// round-to-nearest-even to bf16, kept in an fp32 register (reading c22)
template <bool RND>
__device__ __forceinline__ float opnd(float v) {
  return RND ? __bfloat162float(__float2bfloat16_rn(v)) : v;
}

template <int MODE, bool RND>
__global__ void __launch_bounds__(NT)
conv_simt_kernel(ConvGeom g, const float *__restrict__ asrc, const float *__restrict__ bsrc,
                 float *__restrict__ out, const float *__restrict__ addend,
                 int64_t M, int N, int64_t K, int64_t kchunk) {
  pdl_wait_trigger();
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int t = threadIdx.x;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  const int64_t kend = min(K, kbeg + kchunk);
  if (MODE == WGRAD) out += (int64_t)blockIdx.z * M * N;

  // per-thread fixed row decode for FWD / DGRAD A loads
  const int a_row = t >> 2, a_kq = (t & 3) * 4;
  int ab = 0, ah = 0, aw = 0;
  bool a_row_ok = false;
  if (MODE != WGRAD) {
    int64_t m = m0 + a_row;
    a_row_ok = m < M;
    if (a_row_ok) {
      int HW = (MODE == FWD) ? g.Ho * g.Wo : g.H * g.W;
      int Wd = (MODE == FWD) ? g.Wo : g.W;
      ab = (int)(m / HW);
      int r = (int)(m - (int64_t)ab * HW);
      ah = r / Wd;
      aw = r - ah * Wd;
    }
  }
  const int ty = t >> 4, tx = t & 15;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
    // ---------------- A tile -> As[kk][m]
    if (MODE == FWD) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int64_t kk = k0 + a_kq + i;
        float v = 0.f;
        if (a_row_ok && kk < kend) {
          int tap = (int)(kk / g.Ci), ci = (int)(kk - (int64_t)tap * g.Ci);
          int kh = tap / g.k, kw = tap - kh * g.k;
          int hi = ah * g.s + kh - g.p, wi = aw * g.s + kw - g.p;
          if (hi >= 0 && hi < g.H && wi >= 0 && wi < g.W)
            v = asrc[(((int64_t)ab * g.H + hi) * g.W + wi) * g.Ci + ci];
        }
        As[a_kq + i][a_row] = opnd<RND>(v);
      }
    } else if (MODE == DGRAD) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int64_t kk = k0 + a_kq + i;
        float v = 0.f;
        if (a_row_ok && kk < kend) {
          int tap = (int)(kk / g.Co), co = (int)(kk - (int64_t)tap * g.Co);
          int kh = tap / g.k, kw = tap - kh * g.k;
          int hh = ah + g.p - kh, ww = aw + g.p - kw;
          if (hh >= 0 && ww >= 0 && (hh % g.s) == 0 && (ww % g.s) == 0) {
            int ho = hh / g.s, wo = ww / g.s;
            if (ho < g.Ho && wo < g.Wo) v = asrc[(((int64_t)ab * g.Ho + ho) * g.Wo + wo) * g.Co + co];
          }
        }
        As[a_kq + i][a_row] = opnd<RND>(v);
      }
    } else {  // WGRAD: A[m=co][kk=pixel] = dz[pixel][co]
      const int kl = t >> 4, mq = (t & 15) * 4;
      int64_t kk = k0 + kl;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int64_t m = m0 + mq + i;
        As[kl][mq + i] = (kk < kend && m < M) ? opnd<RND>(asrc[kk * g.Co + m]) : 0.f;
      }
    }
    // ---------------- B tile -> Bs[kk][n]
    if (MODE == FWD) {
      const int nl = t >> 2, kq = (t & 3) * 4;
      int n = n0 + nl;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int64_t kk = k0 + kq + i;
        Bs[kq + i][nl] = (n < N && kk < kend) ? opnd<RND>(bsrc[(int64_t)n * K + kk]) : 0.f;
      }
    } else if (MODE == DGRAD) {
      const int kl = t >> 4, nq = (t & 15) * 4;
      int64_t kk = k0 + kl;
      int tap = 0, co = 0;
      if (kk < kend) { tap = (int)(kk / g.Co); co = (int)(kk - (int64_t)tap * g.Co); }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int n = n0 + nq + i;
        Bs[kl][nq + i] = (kk < kend && n < N)
                             ? opnd<RND>(bsrc[((int64_t)co * g.k * g.k + tap) * g.Ci + n]) : 0.f;
      }
    } else {  // WGRAD: B[kk=pixel][n=(kh,kw,ci)] = x[...]
      const int kl = t >> 4, nq = (t & 15) * 4;
      int64_t kk = k0 + kl;
      int b = 0, ho = 0, wo = 0;
      if (kk < kend) {
        int HW = g.Ho * g.Wo;
        b = (int)(kk / HW);
        int r = (int)(kk - (int64_t)b * HW);
        ho = r / g.Wo;
        wo = r - ho * g.Wo;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int n = n0 + nq + i;
        float v = 0.f;
        if (kk < kend && n < N) {
          int tap = n / g.Ci, ci = n - tap * g.Ci;
          int kh = tap / g.k, kw = tap - kh * g.k;
          int hi = ho * g.s + kh - g.p, wi = wo * g.s + kw - g.p;
          if (hi >= 0 && hi < g.H && wi >= 0 && wi < g.W)
            v = bsrc[(((int64_t)b * g.H + hi) * g.W + wi) * g.Ci + ci];
        }
        Bs[kl][nq + i] = opnd<RND>(v);
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t m = m0 + ty + 16 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + tx + 16 * j;
      if (n >= N) continue;
      float v = acc[i][j];
      if (addend) v += addend[m * N + n];
      out[m * N + n] = MODE == FWD ? opnd<RND>(v) : v;
    }
  }
}

__global__ void splitk_reduce_kernel(const float *__restrict__ part, int splits, int64_t n,
                                     float *__restrict__ out) {
  pdl_wait_trigger();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += part[(int64_t)z * n + i];  // fixed order
    out[i] = s;
  }
}

}  // namespace

void conv_fwd_simt(const ConvGeom &g, const float *x, const float *w, float *z, cudaStream_t st, bool bf16) {
  int64_t M = g.M();
  dim3 grid((unsigned)cdiv(M, BM), (unsigned)cdiv(g.Co, BN), 1);
  launch_k(bf16 ? conv_simt_kernel<FWD, true> : conv_simt_kernel<FWD, false>, grid, NT, 0, st, g, x, w, z, nullptr,
           M, g.Co, g.K(), g.K());
  PETRA_LAUNCH_CHECK();
}

void conv_dgrad_simt(const ConvGeom &g, const float *dz, const float *w, const float *addend,
                     float *dx, cudaStream_t st, bool bf16) {
  int64_t M = g.Min();
  int64_t K = (int64_t)g.k * g.k * g.Co;
  dim3 grid((unsigned)cdiv(M, BM), (unsigned)cdiv(g.Ci, BN), 1);
  launch_k(bf16 ? conv_simt_kernel<DGRAD, true> : conv_simt_kernel<DGRAD, false>, grid, NT, 0, st, g, dz, w, dx,
           addend, M, g.Ci, K, K);
  PETRA_LAUNCH_CHECK();
}

size_t conv_wgrad_simt_workspace(const ConvGeom &g) {
  int64_t M = g.Co, N = g.K();
  int64_t tiles = cdiv(M, BM) * cdiv(N, BN);
  int splits = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(2 * kNumSMs, tiles), cdiv(g.M(), 256)));
  return splits > 1 ? (size_t)splits * M * N * sizeof(float) : 0;
}

void conv_wgrad_simt(const ConvGeom &g, const float *dz, const float *x, float *dw, float *ws,
                     cudaStream_t st, bool bf16) {
  auto kern = bf16 ? conv_simt_kernel<WGRAD, true> : conv_simt_kernel<WGRAD, false>;
  int64_t M = g.Co, N = g.K(), K = g.M();
  int64_t tiles = cdiv(M, BM) * cdiv(N, BN);
  int splits = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(2 * kNumSMs, tiles), cdiv(K, 256)));
  int64_t kchunk = cdiv(cdiv(K, splits), BK) * BK;
  splits = (int)cdiv(K, kchunk);
  dim3 grid((unsigned)cdiv(M, BM), (unsigned)cdiv(N, BN), splits);
  if (splits == 1) {
    launch_k(kern, grid, NT, 0, st, g, dz, x, dw, nullptr, M, (int)N, K, kchunk);
    PETRA_LAUNCH_CHECK();
    return;
  }
  launch_k(kern, grid, NT, 0, st, g, dz, x, ws, nullptr, M, (int)N, K, kchunk);
  PETRA_LAUNCH_CHECK();
  int64_t n = M * N;
  launch_k(splitk_reduce_kernel, (unsigned)std::min<int64_t>(cdiv(n, 256), 4 * kNumSMs), 256, 0, st, 
      ws, splits, n, dw);
  PETRA_LAUNCH_CHECK();
}

}  // namespace petra

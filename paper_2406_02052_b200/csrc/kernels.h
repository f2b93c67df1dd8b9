// kernels.h -- launchers of the PETRA B200 kernels (internal C++ interface, not the ABI).
#pragma once
#include <algorithm>
#include <vector>
#include "common.cuh"

namespace petra {

// ---------------------------------------------------------------- SIMT fp32 convolutions
// bf16 = true: operands rounded to bf16 on load and the forward z on store (the
// bf16 path's rule for every convolution pass, reading c22)
void conv_fwd_simt(const ConvGeom &g, const float *x, const float *w, float *z, cudaStream_t st, bool bf16 = false);
void conv_dgrad_simt(const ConvGeom &g, const float *dz, const float *w, const float *addend, float *dx,
                     cudaStream_t st, bool bf16 = false);
size_t conv_wgrad_simt_workspace(const ConvGeom &g);
void conv_wgrad_simt(const ConvGeom &g, const float *dz, const float *x, float *dw, float *ws, cudaStream_t st,
                     bool bf16 = false);

// ---------------------------------------------------------------- tcgen05 bf16 convolutions
// bf16 activation operands are [B][H][W][C], or -- "padded" -- [B][H+2][W+2][C] with
// zero borders (the 3x3 / stride-1 layers: read by the halo kernel, conv_halo.cu;
// the other kernels read the interior of a padded buffer through strided TMA views).
bool conv_tc_supported(const ConvGeom &g, int mode);   // mode 0 fwd, 1 dgrad, 2 wgrad
void conv_tc_prepare();  // one-time kernel attributes (before any graph capture)
size_t conv_tc_workspace(const ConvGeom &g, int mode);  // split-K workspace bytes
void conv_tc_plan_info(const ConvGeom &g, int mode, int *out);  // {BN, splits, cluster size}
// BN partial statistics written by a conv epilogue: `rows` rows [rows][Co][2] of
// (mean, M2) over the CTA's valid output rows, one row per CTA, followed by the rows'
// counts (float[rows] at part + rows * Co * 2); with `groups` > 1 the CTAs each own one
// of `groups` column groups of Co/groups channels (CTA r: group r % groups) and write
// only those columns.  rows == 0: not fused (run bn_stats on z).
struct StatsRows {
  int rows = 0, groups = 1;
};
// z[m][co] = conv(x_bf16, w_bf16), stored fp32 or (z_bf16) bf16.  stats_part (nullable,
// >= 148*(Co*2+1) floats): the epilogue also writes BN partial statistics of z as stored.
StatsRows conv_fwd_tc(const ConvGeom &g, const __nv_bfloat16 *x, bool x_padded, const __nv_bfloat16 *w, void *z,
                bool z_bf16, float *ws, float *stats_part, cudaStream_t st);
void bn_stats_from_partials(const float *part, StatsRows rows, int N, int64_t M, float eps, float *mean,
                            float *invstd, float *rmean, float *rvar, float mom, cudaStream_t st);
// dx (fp32) = addend + conv^T(dz_bf16, wT_bf16)
void conv_dgrad_tc(const ConvGeom &g, const __nv_bfloat16 *dz, bool dz_padded, const __nv_bfloat16 *wt,
                   const float *addend, float *dx, float *ws, cudaStream_t st);
// dw (fp32) = sum_pixels dz (x) x
void conv_wgrad_tc(const ConvGeom &g, const __nv_bfloat16 *dz, bool dz_padded, const __nv_bfloat16 *x,
                   bool x_padded, float *dw, float *ws, cudaStream_t st);
// halo kernel (conv_halo.cu): 3x3 stride-1 pass on a padded operand
void conv_halo_prepare();
bool conv_halo_eligible(int B, int H, int W, int Cred, int N);
StatsRows conv_halo_run(int B, int H, int W, int Cred, int N, const __nv_bfloat16 *a_pad,
                        const __nv_bfloat16 *wmat, const float *addend, void *out, bool out16, float *stats,
                        cudaStream_t st);

// wgrad of a 3x3 stride-1 layer on zero-bordered operands: one x-halo load per pixel block
// serves all nine taps (conv_halo.cu)
bool wgrad_halo_eligible(const ConvGeom &g);
size_t wgrad_halo_workspace(const ConvGeom &g);
void wgrad_halo_run(const ConvGeom &g, const __nv_bfloat16 *dz_pad, const __nv_bfloat16 *x_pad, float *dw, float *ws,
                    cudaStream_t st);

// out[i] = sum over splits z of part[z * n + i], fixed order (deterministic)
void splitk_sum(const float *part, int splits, int64_t n, float *out, cudaStream_t st);

// ---------------------------------------------------------------- tcgen05 stem (small Ci)
// Convolutions whose input has few channels (the stem: Ci <= 4, k <= 8) run on the
// tensor cores with a GATHERING producer: warps build the im2col rows of each
// 128-pixel tile from a bf16 copy of the image padded to 4 channels (one 8-byte load
// per pixel and kernel tap) into the 128B-swizzled smem layout (no im2col tensor in
// HBM).  Forward and wgrad only (the stem input is data).
bool stem_tc_supported(const ConvGeom &g);
void stem_tc_prepare();  // kernel attributes (called by conv_tc_prepare)
size_t stem_tc_workspace(const ConvGeom &g);
size_t stem_operand_elems(const ConvGeom &g);  // bf16 elements of the 4-channel image copy
// xq[pixel][0..3] = bf16(x[pixel][c]) (0 for c >= Ci): the stem's tensor-core operand
void image_to_bf16x4(const float *x, __nv_bfloat16 *xq, const ConvGeom &g, cudaStream_t st);
// z = conv(xq, bf16(w)) stored fp32 or (z_bf16) bf16; w fp32 as stored; fused BN
// partials as conv_fwd_tc
StatsRows stem_fwd_tc(const ConvGeom &g, const __nv_bfloat16 *xq, const float *w, void *z, bool z_bf16,
                      float *stats_part, cudaStream_t st);
// dw (fp32) = sum_pixels dz_bf16 (x) xq
void stem_wgrad_tc(const ConvGeom &g, const __nv_bfloat16 *dz, const __nv_bfloat16 *xq, float *dw, float *ws,
                   cudaStream_t st);

// ---------------------------------------------------------------- batch norm / coupling
// BN statistics still to be merged from a conv epilogue's partial rows (StatsRows at
// `part`): the consuming BN pass (apply, backward reduce) merges the rows of its channel
// tile in its prologue instead of a separate stats_finalize launch.  Block 0 of each
// channel tile writes mean / invstd to global (for later passes) and, when rmean is set,
// applies the running-statistics update.  part == nullptr: mean / invstd are final.
struct StatsFold {
  const float *part = nullptr;
  int rows = 0, groups = 1, N = 0;  // partial rows, column groups, channels of the conv output
  int64_t M = 0;                    // valid output rows (the statistics' count)
  float eps = 1e-5f, mom = 0.1f;
  float *rmean = nullptr, *rvar = nullptr;
};
size_t bn_partial_bytes(int64_t M, int C);
size_t bn_counter_count(int C);  // zero-initialised unsigned counters a reduction needs
template <typename TZ>
void bn_stats(const TZ *z, int64_t M, int C, float eps, float *mean, float *invstd, float *rmean, float *rvar,
              float mom, double *part, unsigned *counter, cudaStream_t st);
// out_bf16 (nullable) is written padded when pH > 0: rows m = (b*pH + h)*pW + w go to the
// interior of a zero-bordered [B][pH+2][pW+2][C] buffer
// fold (nullable): statistics of z's columns [zc0, zc0 + C) still to be merged (StatsFold)
template <typename TZ, typename TO>
void bn_apply(int64_t M, int C, const TZ *z, int ldz, int zc0, const float *mean, const float *invstd,
              const float *gamma, const float *beta, int relu, float sign, const float *acc, TO *out,
              __nv_bfloat16 *out_bf16, int pH, int pW, cudaStream_t st, const StatsFold *fold = nullptr);
template <typename TZ>
void bn_bwd_reduce(const TZ *z, int64_t M, int C, const float *mean, const float *invstd, const float *gamma,
                   const float *beta, int relu, const float *dy0, const float *dy1, int cs, const float *dst_in,
                   float *dst_out, __nv_bfloat16 *dst_bf16, int pH, int pW, float *dgamma, float *dbeta,
                   double *part, unsigned *counter, cudaStream_t st, const StatsFold *fold = nullptr);
// dz (fp32, nullable) and/or its bf16 copy (nullable: the tensor-core operand; padded
// as in bn_apply when pH > 0)
template <typename TZ>
void bn_bwd_dz(int64_t M, int C, const TZ *z, const float *mean, const float *invstd, const float *gamma,
               const float *beta, int relu, const float *dy0, const float *dy1, int cs, const float *dgamma,
               const float *dbeta, float *dz, __nv_bfloat16 *dz_bf16, int pH, int pW, cudaStream_t st);

// ---------------------------------------------------------------- optimizer / tail / misc
struct SgdSeg {
  int64_t offset, count;
  int decay;
  int co, k, ci;                 // conv weights only (for the bf16 shadows)
  __nv_bfloat16 *w_bf16;         // nullable: bf16 shadow [Co][k][k][Ci]
  __nv_bfloat16 *wt_bf16;        // nullable: dgrad operand [Ci][k][k][Co], taps flipped
};
// work item of the update: a 32 x 32 tile (lo = tile index) of a conv weight with bf16
// shadows, or elements [lo, hi) of another tensor (built once per stage: sgd_chunks)
struct SgdChunk {
  int seg;
  int64_t lo, hi;
};
std::vector<SgdChunk> sgd_chunks(const std::vector<SgdSeg> &segs);
// lr_dev: device scalar (written per tick from pinned host memory, so a captured
// CUDA graph replays with the current learning rate)
enum { SGD_PLAIN = 0, SGD_ACCUMULATE = 1, SGD_ACC_UPDATE = 2 };
void sgd_update(const SgdSeg *segs_dev, int nseg, const SgdChunk *chunks_dev, int nchunks, float *theta, float *v,
                const float *grad, float *acc, int k, int mode, const float *lr_dev, float mom, float wd, int nesterov,
                cudaStream_t st, bool shadow_only, int *nonfinite);  // nonfinite: device flag set (2) by a NaN / Inf in Delta
void tail_forward_backward(const float *x1, const float *x2, int B, int HW, int C, const float *w,
                           const float *bias, int N, const int32_t *labels, float *feat, float *logits,
                           float *dlogits, float *loss_row, float *dfeat, float *dw, float *db, float *d1,
                           float *d2, float *loss, int *nonfinite, float *fc_ws, int64_t fc_ws_floats,
                           cudaStream_t st, int *correct = nullptr);  // correct: evaluation only (count += argmax == y)
// BN constants from the running statistics (evaluation): mean = rm, invstd = 1/sqrt(rv + eps)
void bn_running_constants(const float *rm, const float *rv, int C, float eps, float *mean, float *invstd,
                          cudaStream_t st);
void maxpool_fwd(const float *a, int B, int H, int W, int C, int Ho, int Wo, float *o1, float *o2, uint8_t *arg,
                 cudaStream_t st);
void maxpool_bwd(const float *d1, const float *d2, const uint8_t *arg, int B, int H, int W, int C, int Ho, int Wo,
                 float *da, cudaStream_t st);
void f32_to_bf16(const float *x, __nv_bfloat16 *y, int64_t n, cudaStream_t st);
void bf16_to_f32(const __nv_bfloat16 *x, float *y, int64_t n, cudaStream_t st);
// x = float(bf16_rn(x)): the pipeline's bf16 wire format (petra_pipeline_desc.wire)
void round_bf16_inplace(float *x, int64_t n, cudaStream_t st);
// y = bf16(x) into the interior of a zero-bordered [B][H+2][W+2][C] buffer
void f32_to_bf16_padded(const float *x, __nv_bfloat16 *y, int B, int H, int W, int C, cudaStream_t st);

}  // namespace petra

// convtest.cu -- petra_conv_run: one convolution pass on host buffers (kernel-level tests).
#include <cuda_runtime.h>

#include <cstring>
#include <functional>
#include <vector>

#include "../../include/petra.h"
#include "errors.h"
#include "kernels.h"
#include "stage.h"

namespace {
// one convolution pass on host buffers; iters > 0: also the mean device time of
// `iters` further passes (CUDA events; operands prepared once, outside the timing)
petra_status run(int mode, int engine, const petra_conv_geom *pg, const float *a, const float *b,
                 const float *addend, float *out, int iters = 0, float *ms = nullptr, bool out16 = false,
                 bool stats = false, float *mean_out = nullptr, float *var_out = nullptr,
                 bool direct_launches = false) {
  using namespace petra;
  ConvGeom g = make_geom(pg->batch, pg->h, pg->w, pg->cin, pg->cout, pg->ksize, pg->stride);
  int64_t nx = g.Min() * g.Ci, nz = g.M() * g.Co, nw = (int64_t)g.Co * g.K();
  int64_t na = mode == 0 ? nx : nz, nb = mode == 2 ? nx : nw, no = mode == 0 ? nz : (mode == 1 ? nx : nw);
  const bool padded = engine == 2;  // tcgen05 on zero-bordered operands (halo kernel where eligible)
  if (padded) engine = 1;
  const bool stem = engine == 1 && !padded && !conv_tc_supported(g, mode) && mode != 1 && stem_tc_supported(g);
  if (engine == 1 && !stem && !conv_tc_supported(g, mode)) return PETRA_E_UNSUPPORTED;
  if (engine == 1) conv_tc_prepare();
  DevPtr da = dalloc(na * 4), db = dalloc(nb * 4), dout = dalloc(no * 4), dadd;
  PETRA_CUDA(cudaMemcpy(da->p, a, na * 4, cudaMemcpyHostToDevice));
  PETRA_CUDA(cudaMemcpy(db->p, b, nb * 4, cudaMemcpyHostToDevice));
  if (addend) {
    dadd = dalloc(no * 4);
    PETRA_CUDA(cudaMemcpy(dadd->p, addend, no * 4, cudaMemcpyHostToDevice));
  }
  PETRA_CUDA(cudaDeviceSynchronize());  // pageable copies land before the non-blocking stream reads them
  // a capturable stream: the timed loop replays as one CUDA graph (no host encode / launch
  // time between the passes -- device time of back-to-back passes)
  cudaStream_t st = nullptr;
  PETRA_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } st_guard{st};
  DevPtr ab, bb, ws, part = dalloc((size_t)kNumSMs * 4 * (g.Co * 2 + 1) * sizeof(float));
  StatsRows rows;
  float *stats_part = stats ? part->as<float>() : nullptr;
  const bool a_pad = padded, b_pad = padded && mode == 2;
  std::function<void()> launch;
  if (stem) {  // gathered-im2col tensor-core stem: 4-channel bf16 copy of the image
    ws = dalloc(std::max<size_t>(16, stem_tc_workspace(g)));
    if (mode == 0) {
      ab = dalloc(stem_operand_elems(g) * 2);
      launch = [&] {
        image_to_bf16x4(da->as<float>(), ab->as<__nv_bfloat16>(), g, st);
        rows = stem_fwd_tc(g, ab->as<__nv_bfloat16>(), db->as<float>(), dout->p, out16, stats_part, st);
      };
    } else {
      ab = dalloc(na * 2);
      bb = dalloc(stem_operand_elems(g) * 2);
      f32_to_bf16(da->as<float>(), ab->as<__nv_bfloat16>(), na, st);
      image_to_bf16x4(db->as<float>(), bb->as<__nv_bfloat16>(), g, st);
      launch = [&] {
        stem_wgrad_tc(g, ab->as<__nv_bfloat16>(), bb->as<__nv_bfloat16>(), dout->as<float>(), ws->as<float>(), st);
      };
    }
  } else if (engine == 0) {
    ws = dalloc(std::max<size_t>(16, conv_wgrad_simt_workspace(g)));
    launch = [&] {
      if (mode == 0) conv_fwd_simt(g, da->as<float>(), db->as<float>(), dout->as<float>(), st);
      else if (mode == 1)
        conv_dgrad_simt(g, da->as<float>(), db->as<float>(), addend ? dadd->as<float>() : nullptr,
                        dout->as<float>(), st);
      else conv_wgrad_simt(g, da->as<float>(), db->as<float>(), dout->as<float>(), ws->as<float>(), st);
    };
  } else {
    // operand a (x or dz) and, for wgrad, b (= x) zero-bordered when padded
    const int aH = mode == 0 ? g.H : g.Ho, aW = mode == 0 ? g.W : g.Wo, aC = mode == 0 ? g.Ci : g.Co;
    const int64_t na_buf = a_pad ? (int64_t)g.B * (aH + 2) * (aW + 2) * aC : na;
    const int64_t nb_buf = b_pad ? (int64_t)g.B * (g.H + 2) * (g.W + 2) * g.Ci : nb;
    ab = dalloc(na_buf * 2);
    bb = dalloc(nb_buf * 2);
    PETRA_CUDA(cudaMemsetAsync(ab->p, 0, na_buf * 2, st));  // on st: it does not order with the legacy stream
    PETRA_CUDA(cudaMemsetAsync(bb->p, 0, nb_buf * 2, st));
    if (a_pad) f32_to_bf16_padded(da->as<float>(), ab->as<__nv_bfloat16>(), g.B, aH, aW, aC, st);
    else f32_to_bf16(da->as<float>(), ab->as<__nv_bfloat16>(), na, st);
    if (mode == 1) {  // flipped / transposed weights wT[ci][kh'][kw'][co] = w[co][k-1-kh'][k-1-kw'][ci]
      std::vector<float> wt(nw);
      int k = g.k;
      for (int co = 0; co < g.Co; ++co)
        for (int kh = 0; kh < k; ++kh)
          for (int kw = 0; kw < k; ++kw)
            for (int ci = 0; ci < g.Ci; ++ci)
              wt[(((int64_t)ci * k + (k - 1 - kh)) * k + (k - 1 - kw)) * g.Co + co] =
                  b[(((int64_t)co * k + kh) * k + kw) * g.Ci + ci];
      PETRA_CUDA(cudaMemcpy(db->p, wt.data(), nb * 4, cudaMemcpyHostToDevice));
      PETRA_CUDA(cudaDeviceSynchronize());
    }
    if (b_pad) f32_to_bf16_padded(db->as<float>(), bb->as<__nv_bfloat16>(), g.B, g.H, g.W, g.Ci, st);
    else f32_to_bf16(db->as<float>(), bb->as<__nv_bfloat16>(), nb, st);
    ws = dalloc(std::max<size_t>(16, conv_tc_workspace(g, mode)));
    launch = [&] {
      if (mode == 0)
        rows = conv_fwd_tc(g, ab->as<__nv_bfloat16>(), a_pad, bb->as<__nv_bfloat16>(), dout->p, out16,
                           ws->as<float>(), stats_part, st);
      else if (mode == 1)
        conv_dgrad_tc(g, ab->as<__nv_bfloat16>(), a_pad, bb->as<__nv_bfloat16>(),
                      addend ? dadd->as<float>() : nullptr, dout->as<float>(), ws->as<float>(), st);
      else
        conv_wgrad_tc(g, ab->as<__nv_bfloat16>(), a_pad, bb->as<__nv_bfloat16>(), b_pad, dout->as<float>(),
                      ws->as<float>(), st);
    };
  }
  launch();
  PETRA_CUDA(cudaDeviceSynchronize());
  if (iters > 0) {
    cudaEvent_t e0, e1;
    PETRA_CUDA(cudaEventCreate(&e0));
    PETRA_CUDA(cudaEventCreate(&e1));
    cudaGraphExec_t gx = nullptr;
    if (!direct_launches) {
      cudaGraph_t gr;
      PETRA_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      for (int i = 0; i < iters; ++i) launch();
      PETRA_CUDA(cudaStreamEndCapture(st, &gr));
      PETRA_CUDA(cudaGraphInstantiate(&gx, gr, 0));
      cudaGraphDestroy(gr);
      PETRA_CUDA(cudaGraphLaunch(gx, st));  // warm replay
      PETRA_CUDA(cudaStreamSynchronize(st));
    }
    PETRA_CUDA(cudaEventRecord(e0, st));
    if (gx) PETRA_CUDA(cudaGraphLaunch(gx, st));
    else
      for (int i = 0; i < iters; ++i) launch();
    PETRA_CUDA(cudaEventRecord(e1, st));
    PETRA_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    PETRA_CUDA(cudaEventElapsedTime(&t, e0, e1));
    *ms = t / iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (gx) cudaGraphExecDestroy(gx);
  }
  PETRA_CUDA(cudaStreamSynchronize(st));
  if (mean_out && var_out) {  // the library's BN batch statistics of z as stored (eps = 0: invstd^-2 = var)
    if (rows.rows == 0) throw PetraError(PETRA_E_UNSUPPORTED, "no fused statistics for this geometry");
    DevPtr dm = dalloc(g.Co * 4), di = dalloc(g.Co * 4);
    bn_stats_from_partials(part->as<float>(), rows, g.Co, g.M(), 0.f, dm->as<float>(), di->as<float>(), nullptr,
                           nullptr, 0.1f, st);
    std::vector<float> inv(g.Co);
    PETRA_CUDA(cudaStreamSynchronize(st));
    PETRA_CUDA(cudaMemcpy(mean_out, dm->p, g.Co * 4, cudaMemcpyDeviceToHost));
    PETRA_CUDA(cudaMemcpy(inv.data(), di->p, g.Co * 4, cudaMemcpyDeviceToHost));
    for (int c = 0; c < g.Co; ++c) var_out[c] = 1.f / (inv[c] * inv[c]);
  }
  if (out && out16) {  // bf16 z -> fp32
    std::vector<uint16_t> h(no);
    PETRA_CUDA(cudaMemcpy(h.data(), dout->p, no * 2, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < no; ++i) {
      const uint32_t u = (uint32_t)h[i] << 16;
      std::memcpy(out + i, &u, 4);
    }
  } else if (out) {
    PETRA_CUDA(cudaMemcpy(out, dout->p, no * 4, cudaMemcpyDeviceToHost));
  }
  return PETRA_OK;
}
}  // namespace

extern "C" petra_status petra_conv_run(int32_t mode, int32_t engine, const petra_conv_geom *g, const float *a,
                                       const float *b, const float *addend, float *out) {
  if (!g || !a || !b || !out || mode < 0 || mode > 2 || engine < 0 || engine > 2) return PETRA_E_ARG;
  try {
    return run(mode, engine, g, a, b, addend, out);
  } catch (const petra::PetraError &e) {
    return e.status;
  } catch (...) {
    cudaGetLastError();
    return PETRA_E_CUDA;
  }
}

extern "C" petra_status petra_conv_bn_stats(const petra_conv_geom *g, int32_t engine, const float *x,
                                            const float *w, float *z, float *mean, float *var) {
  if (!g || !x || !w || !z || !mean || !var || engine < 1 || engine > 2) return PETRA_E_ARG;
  try {
    return run(0, engine, g, x, w, nullptr, z, 0, nullptr, true, true, mean, var);
  } catch (const petra::PetraError &e) {
    return e.status;
  } catch (...) {
    cudaGetLastError();
    return PETRA_E_CUDA;
  }
}

extern "C" petra_status petra_conv_bench(int32_t mode, int32_t engine, const petra_conv_geom *g, int32_t flags,
                                         int32_t iters, float *avg_ms) {
  if (!g || !avg_ms || iters < 1 || mode < 0 || mode > 2 || engine < 0 || engine > 2) return PETRA_E_ARG;
  try {
    petra::ConvGeom cg = petra::make_geom(g->batch, g->h, g->w, g->cin, g->cout, g->ksize, g->stride);
    const int64_t nx = cg.Min() * cg.Ci, nz = cg.M() * cg.Co, nw = (int64_t)cg.Co * cg.K();
    const int64_t na = mode == 0 ? nx : nz, nb = mode == 2 ? nx : nw;
    std::vector<float> a(na), b(nb);
    uint32_t r = 12345u;
    auto rnd = [&r]() {
      r = r * 1664525u + 1013904223u;
      return (float)((r >> 9) & 0xFFFF) / 32768.f - 1.f;
    };
    for (auto &v : a) v = rnd();
    for (auto &v : b) v = rnd() * 0.05f;
    return run(mode, engine, g, a.data(), b.data(), nullptr, nullptr, iters, avg_ms, (flags & 1) != 0,
               (flags & 2) != 0, nullptr, nullptr, (flags & 4) != 0);
  } catch (const petra::PetraError &e) {
    return e.status;
  } catch (...) {
    cudaGetLastError();
    return PETRA_E_CUDA;
  }
}

extern "C" int32_t petra_conv_engine(const petra_conv_geom *pg, int32_t mode, int32_t precision) {
  if (!pg || precision != PETRA_BF16_TC) return 0;
  petra::ConvGeom g = petra::make_geom(pg->batch, pg->h, pg->w, pg->cin, pg->cout, pg->ksize, pg->stride);
  if (petra::conv_tc_supported(g, mode)) return 1;
  return (mode != 1 && petra::stem_tc_supported(g)) ? 1 : 0;
}

extern "C" petra_status petra_conv_plan(const petra_conv_geom *pg, int32_t mode, int32_t *plan) {
  if (!pg || !plan || (mode != 0 && mode != 1)) return PETRA_E_ARG;
  petra::ConvGeom g = petra::make_geom(pg->batch, pg->h, pg->w, pg->cin, pg->cout, pg->ksize, pg->stride);
  if (!petra::conv_tc_supported(g, mode) || (mode == 1 && g.s != 1)) return PETRA_E_UNSUPPORTED;
  int out[3];
  petra::conv_tc_plan_info(g, mode, out);
  for (int i = 0; i < 3; ++i) plan[i] = out[i];
  return PETRA_OK;
}

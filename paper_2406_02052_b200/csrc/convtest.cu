// convtest.cu -- petra_conv_run: one convolution pass on host buffers (kernel-level tests).
#include <cuda_runtime.h>

#include <vector>

#include "../../include/petra.h"
#include "errors.h"
#include "kernels.h"
#include "stage.h"

namespace {
petra_status run(int mode, int engine, const petra_conv_geom *pg, const float *a, const float *b,
                 const float *addend, float *out) {
  using namespace petra;
  ConvGeom g = make_geom(pg->batch, pg->h, pg->w, pg->cin, pg->cout, pg->ksize, pg->stride);
  int64_t nx = g.Min() * g.Ci, nz = g.M() * g.Co, nw = (int64_t)g.Co * g.K();
  int64_t na = mode == 0 ? nx : nz, nb = mode == 2 ? nx : nw, no = mode == 0 ? nz : (mode == 1 ? nx : nw);
  const bool stem = engine == 1 && !conv_tc_supported(g, mode) && mode != 1 && stem_tc_supported(g);
  if (engine == 1 && !stem && !conv_tc_supported(g, mode)) return PETRA_E_UNSUPPORTED;
  if (engine == 1) conv_tc_prepare();
  DevPtr da = dalloc(na * 4), db = dalloc(nb * 4), dout = dalloc(no * 4), dadd;
  PETRA_CUDA(cudaMemcpy(da->p, a, na * 4, cudaMemcpyHostToDevice));
  PETRA_CUDA(cudaMemcpy(db->p, b, nb * 4, cudaMemcpyHostToDevice));
  if (addend) {
    dadd = dalloc(no * 4);
    PETRA_CUDA(cudaMemcpy(dadd->p, addend, no * 4, cudaMemcpyHostToDevice));
  }
  cudaStream_t st = nullptr;
  if (stem) {  // gathered-im2col tensor-core stem: fp32 image (and fp32 weights) read directly
    DevPtr ws = dalloc(std::max<size_t>(16, stem_tc_workspace(g)));
    if (mode == 0) {
      stem_fwd_tc(g, da->as<float>(), db->as<float>(), dout->p, false, nullptr, st);
    } else {
      DevPtr ab = dalloc(na * 2);
      f32_to_bf16(da->as<float>(), ab->as<__nv_bfloat16>(), na, st);
      stem_wgrad_tc(g, ab->as<__nv_bfloat16>(), db->as<float>(), dout->as<float>(), ws->as<float>(), st);
    }
    PETRA_CUDA(cudaDeviceSynchronize());
  } else if (engine == 0) {
    DevPtr ws = dalloc(std::max<size_t>(16, conv_wgrad_simt_workspace(g)));
    if (mode == 0) conv_fwd_simt(g, da->as<float>(), db->as<float>(), dout->as<float>(), st);
    else if (mode == 1)
      conv_dgrad_simt(g, da->as<float>(), db->as<float>(), addend ? dadd->as<float>() : nullptr,
                      dout->as<float>(), st);
    else conv_wgrad_simt(g, da->as<float>(), db->as<float>(), dout->as<float>(), ws->as<float>(), st);
    PETRA_CUDA(cudaDeviceSynchronize());
  } else {
    DevPtr ab = dalloc(na * 2), bb = dalloc(nb * 2);
    f32_to_bf16(da->as<float>(), ab->as<__nv_bfloat16>(), na, st);
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
    }
    f32_to_bf16(db->as<float>(), bb->as<__nv_bfloat16>(), nb, st);
    DevPtr ws = dalloc(std::max<size_t>(16, conv_tc_workspace(g, mode)));
    if (mode == 0) conv_fwd_tc(g, ab->as<__nv_bfloat16>(), bb->as<__nv_bfloat16>(), dout->p, false, ws->as<float>(),
                            nullptr, st);
    else if (mode == 1)
      conv_dgrad_tc(g, ab->as<__nv_bfloat16>(), bb->as<__nv_bfloat16>(), addend ? dadd->as<float>() : nullptr,
                    dout->as<float>(), ws->as<float>(), st);
    else conv_wgrad_tc(g, ab->as<__nv_bfloat16>(), bb->as<__nv_bfloat16>(), dout->as<float>(), ws->as<float>(), st);
    PETRA_CUDA(cudaDeviceSynchronize());
  }
  PETRA_CUDA(cudaMemcpy(out, dout->p, no * 4, cudaMemcpyDeviceToHost));
  return PETRA_OK;
}
}  // namespace

extern "C" petra_status petra_conv_run(int32_t mode, int32_t engine, const petra_conv_geom *g, const float *a,
                                       const float *b, const float *addend, float *out) {
  if (!g || !a || !b || !out || mode < 0 || mode > 2 || engine < 0 || engine > 1) return PETRA_E_ARG;
  try {
    return run(mode, engine, g, a, b, addend, out);
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

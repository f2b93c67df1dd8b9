// api.cpp -- the C ABI of libpetra.so (include/petra.h): argument checks,
// exception -> petra_status translation, thread-local error strings.
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "../../include/petra.h"
#include "errors.h"
#include "pipeline.h"

struct petra_stage {
  std::unique_ptr<petra::Stage> owned;  // null for handles borrowed from a pipeline
  petra::Stage *s = nullptr;
};
struct petra_pipeline {
  std::unique_ptr<petra::Pipeline> p;
  std::vector<std::unique_ptr<petra_stage>> borrowed;  // non-owning stage handles
};
struct petra_schedule {
  std::unique_ptr<petra::Schedule> s;
};

namespace {
thread_local std::string g_err;

petra_status fail(petra_status s, const std::string &m) {
  g_err = m;
  return s;
}

template <typename F>
petra_status guard(F &&f) {
  try {
    f();
    g_err.clear();
    return PETRA_OK;
  } catch (const petra::PetraError &e) {
    return fail(e.status, e.what());
  } catch (const petra::CudaError &e) {
    cudaGetLastError();
    return fail(PETRA_E_CUDA, e.what());
  } catch (const std::bad_alloc &e) {
    return fail(PETRA_E_OOM, e.what());
  } catch (const std::exception &e) {
    return fail(PETRA_E_ARG, e.what());
  } catch (...) {
    return fail(PETRA_E_ARG, "unknown error");
  }
}

void need_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw petra::PetraError(PETRA_E_CUDA, "no CUDA device available (libpetra has no CPU fallback)");
  }
}
}  // namespace

extern "C" {

const char *petra_status_str(int s) {
  switch (s) {
    case PETRA_OK: return "ok";
    case PETRA_E_ARG: return "invalid argument";
    case PETRA_E_SHAPE: return "shape mismatch";
    case PETRA_E_ODD_CHANNELS: return "odd channel count";
    case PETRA_E_EMPTY_BUFFER: return "empty FIFO on non-reversible backward";
    case PETRA_E_ORDER: return "micro-batch order violation";
    case PETRA_E_NONFINITE: return "non-finite loss";
    case PETRA_E_CUDA: return "CUDA error";
    case PETRA_E_NCCL: return "NCCL error";
    case PETRA_E_OOM: return "out of device memory";
    case PETRA_E_UNSUPPORTED: return "unsupported configuration";
    default: return "unknown status";
  }
}

const char *petra_last_error(void) { return g_err.c_str(); }
const char *petra_version(void) { return "petra-b200 0.1 sm_100a"; }

petra_status petra_stage_create(const petra_stage_desc *desc, uint64_t seed, petra_stage **out) {
  if (!desc || !out) return fail(PETRA_E_ARG, "NULL desc/out");
  return guard([&] {
    need_device();
    std::unique_ptr<petra_stage> h(new petra_stage);
    h->owned.reset(new petra::Stage(*desc, seed));
    h->s = h->owned.get();
    *out = h.release();
  });
}

petra_status petra_stage_destroy(petra_stage *s) {
  if (s && !s->owned) return fail(PETRA_E_ARG, "stage handle is owned by a pipeline");
  return guard([&] { delete s; });
}

petra_status petra_stage_output_shape(const petra_stage *s, int32_t *b, int32_t *h, int32_t *w, int32_t *c) {
  if (!s) return fail(PETRA_E_ARG, "NULL stage");
  const auto &o = s->s->out_shape();
  if (b) *b = o.B;
  if (h) *h = o.H;
  if (w) *w = o.W;
  if (c) *c = o.C;
  return PETRA_OK;
}

petra_status petra_stage_param_count(const petra_stage *s, size_t *np, size_t *nb) {
  if (!s) return fail(PETRA_E_ARG, "NULL stage");
  if (np) *np = s->s->n_params();
  if (nb) *nb = s->s->n_buffers();
  return PETRA_OK;
}

petra_status petra_stage_memory(const petra_stage *s, petra_memory_report *out) {
  if (!s || !out) return fail(PETRA_E_ARG, "NULL argument");
  s->s->memory(out);
  return PETRA_OK;
}

petra_status petra_stage_num_tensors(const petra_stage *s, int32_t *n) {
  if (!s || !n) return fail(PETRA_E_ARG, "NULL argument");
  *n = (int32_t)s->s->tensors().size();
  return PETRA_OK;
}

petra_status petra_stage_tensor_info(const petra_stage *s, int32_t i, petra_tensor_info *info) {
  if (!s || !info) return fail(PETRA_E_ARG, "NULL argument");
  if (i < 0 || i >= (int32_t)s->s->tensors().size()) return fail(PETRA_E_ARG, "tensor index out of range");
  *info = s->s->tensors()[i];
  return PETRA_OK;
}

petra_status petra_stage_get_params(petra_stage *s, float *theta, float *v, float *bufs) {
  if (!s) return fail(PETRA_E_ARG, "NULL stage");
  petra_status st = guard([&] { s->s->get_params(theta, v, bufs); });
  if (st != PETRA_OK) return st;
  int nf = 0;
  st = guard([&] { nf = s->s->nonfinite(); });
  if (st != PETRA_OK) return st;
  if (nf) return fail(PETRA_E_NONFINITE, std::string("non-finite ") + ((nf & 1) ? "loss " : "") +
                                             ((nf & 2) ? "Delta (a gradient fed to the update) " : "") +
                                             "was produced");
  return PETRA_OK;
}

petra_status petra_stage_set_params(petra_stage *s, const float *theta, const float *v, const float *bufs) {
  if (!s) return fail(PETRA_E_ARG, "NULL stage");
  return guard([&] { s->s->set_params(theta, v, bufs); });
}

petra_status petra_stage_get_grads(petra_stage *s, float *delta) {
  if (!s || !delta) return fail(PETRA_E_ARG, "NULL argument");
  return guard([&] { s->s->get_grads(delta); });
}

petra_status petra_stage_forward(petra_stage *s, uint64_t mb, const float *x1, const float *x2, float *o1,
                                 float *o2, void *stream) {
  if (!s) return fail(PETRA_E_ARG, "NULL stage");
  return guard([&] { s->s->forward(mb, x1, x2, o1, o2, (cudaStream_t)stream); });
}

petra_status petra_stage_backward(petra_stage *s, uint64_t mb, const float *xt1, const float *xt2,
                                  const float *d1, const float *d2, float *oxt1, float *oxt2, float *od1,
                                  float *od2, float lr, void *stream) {
  if (!s) return fail(PETRA_E_ARG, "NULL stage");
  return guard([&] { s->s->backward(mb, xt1, xt2, d1, d2, oxt1, oxt2, od1, od2, lr, (cudaStream_t)stream); });
}

petra_status petra_stage_tail(petra_stage *s, uint64_t mb, const float *x1, const float *x2, const int32_t *labels,
                              float lr, float *oxt1, float *oxt2, float *od1, float *od2, float *loss,
                              void *stream) {
  if (!s) return fail(PETRA_E_ARG, "NULL stage");
  return guard([&] { s->s->tail(mb, x1, x2, labels, lr, oxt1, oxt2, od1, od2, loss, (cudaStream_t)stream); });
}

petra_status petra_stage_eval(petra_stage *s, const float *x1, const float *x2, float *o1, float *o2, void *stream) {
  if (!s) return fail(PETRA_E_ARG, "NULL stage");
  return guard([&] { s->s->eval(x1, x2, o1, o2, (cudaStream_t)stream); });
}

petra_status petra_stage_eval_tail(petra_stage *s, const float *x1, const float *x2, const int32_t *labels,
                                   int32_t *correct, float *loss, void *stream) {
  if (!s) return fail(PETRA_E_ARG, "NULL stage");
  return guard([&] { s->s->eval_tail(x1, x2, labels, correct, loss, (cudaStream_t)stream); });
}

petra_status petra_pipeline_create(const petra_pipeline_desc *d, petra_pipeline **out) {
  if (!d || !out || !d->stages || !d->stage_rank) return fail(PETRA_E_ARG, "NULL argument");
  return guard([&] {
    need_device();
    std::unique_ptr<petra_pipeline> h(new petra_pipeline);
    h->p.reset(new petra::Pipeline(*d));
    h->borrowed.resize(d->n_stages + 1);
    for (int j = 1; j <= d->n_stages; ++j) {
      if (petra::Stage *st = h->p->stage(j)) {
        h->borrowed[j].reset(new petra_stage);
        h->borrowed[j]->s = st;
      }
    }
    *out = h.release();
  });
}

petra_status petra_set_allocator(void *(*alloc)(size_t bytes, int32_t device, void *ctx),
                                 void (*release)(void *ptr, int32_t device, void *ctx), void *ctx) {
  if ((alloc == nullptr) != (release == nullptr)) return fail(PETRA_E_ARG, "alloc and release go together");
  petra::Allocator &a = petra::allocator();
  a.alloc = reinterpret_cast<void *(*)(size_t, int, void *)>(alloc);
  a.release = reinterpret_cast<void (*)(void *, int, void *)>(release);
  a.ctx = ctx;
  return PETRA_OK;
}

petra_status petra_nccl_unique_id(unsigned char out[128]) {
  if (!out) return fail(PETRA_E_ARG, "NULL argument");
  return guard([&] {
    ncclUniqueId id;
    PETRA_NCCL(petra::nccl().GetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out, &id, sizeof(id));
  });
}

petra_status petra_pipeline_destroy(petra_pipeline *p) {
  return guard([&] { delete p; });
}

petra_status petra_pipeline_stage(petra_pipeline *p, int32_t j, petra_stage **out) {
  if (!p || !out) return fail(PETRA_E_ARG, "NULL argument");
  *out = (j >= 1 && j < (int32_t)p->borrowed.size() && p->borrowed[j]) ? p->borrowed[j].get() : nullptr;
  return PETRA_OK;
}

petra_status petra_pipeline_tick(petra_pipeline *p, int64_t t, int32_t inject, const float *x0,
                                 const int32_t *labels, float lr, float *loss, void *stream, petra_tick_report *rep) {
  if (!p) return fail(PETRA_E_ARG, "NULL pipeline");
  return guard([&] { p->p->tick(t, inject != 0, x0, labels, lr, loss, (cudaStream_t)stream, rep); });
}

petra_status petra_pipeline_comm(petra_pipeline *p, int64_t t, petra_comm_plan *plan) {
  if (!p || !plan) return fail(PETRA_E_ARG, "NULL argument");
  return guard([&] { p->p->comm(t, plan); });
}

petra_status petra_pipeline_timing(petra_pipeline *p, int32_t enable) {
  if (!p) return fail(PETRA_E_ARG, "NULL pipeline");
  return guard([&] { p->p->timing(enable != 0); });
}

petra_status petra_pipeline_stage_ms(petra_pipeline *p, float *ms, int32_t n, int32_t *ticks) {
  if (!p || !ms) return fail(PETRA_E_ARG, "NULL argument");
  return guard([&] {
    int t = p->p->stage_ms(ms, n);
    if (ticks) *ticks = t;
  });
}

petra_status petra_schedule_create(int32_t n, const int32_t *stage_rank, const int32_t *nonrev,
                                   const int32_t *accum_k, int32_t rank, petra_schedule **out) {
  if (!stage_rank || !nonrev || !out || n < 1) return fail(PETRA_E_ARG, "bad schedule arguments");
  return guard([&] {
    auto *h = new petra_schedule;
    h->s.reset(new petra::Schedule(n, std::vector<int>(stage_rank, stage_rank + n),
                                   std::vector<int>(nonrev, nonrev + n), rank,
                                   accum_k ? std::vector<int>(accum_k, accum_k + n) : std::vector<int>()));
    *out = h;
  });
}

petra_status petra_schedule_tick(petra_schedule *s, int64_t t, int32_t inject, petra_tick_report *rep,
                                 petra_sched_msgs *msgs) {
  if (!s) return fail(PETRA_E_ARG, "NULL schedule");
  return guard([&] {
    std::vector<int64_t> ver, fifo;
    auto steps = s->s->tick(t, inject != 0, &ver, &fifo);
    int J = s->s->J();
    if (J > PETRA_MAX_STAGES) throw petra::PetraError(PETRA_E_ARG, "too many stages for the report");
    if (rep) {
      rep->tick = t;
      rep->n_stages = J;
      for (int j = 1; j <= J; ++j) {
        rep->fwd_mb[j - 1] = steps[j].fwd_mb;
        rep->bwd_mb[j - 1] = steps[j].bwd_mb;
        rep->param_version[j - 1] = ver[j];
        rep->fifo_depth[j - 1] = fifo[j];
      }
    }
    if (msgs) {
      auto c = s->s->comm(t);
      msgs->n = (int32_t)c.size();
      for (size_t i = 0; i < c.size(); ++i) {
        msgs->m[i].peer = c[i].peer;
        msgs->m[i].send = c[i].send;
        msgs->m[i].kind = c[i].kind;
        msgs->m[i].stage = c[i].stage;
        msgs->m[i].mb = c[i].mb;
      }
    }
  });
}

petra_status petra_schedule_destroy(petra_schedule *s) {
  return guard([&] { delete s; });
}

}  // extern "C"

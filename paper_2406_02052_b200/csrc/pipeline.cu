// pipeline.cu -- the stages of one rank, their double-buffered mailboxes and the
// per-tick driver (product code).  Cross-rank bytes are moved by the caller
// (NCCL send/recv through torch.distributed) from the plan of petra_pipeline_comm.
#include "pipeline.h"

#include <cstdlib>

namespace petra {

static bool has_stem(const petra_stage_desc &d) { return d.n_units > 0 && d.units[0].kind == PETRA_UNIT_STEM; }

static std::vector<int> nonrev_counts(const petra_pipeline_desc &d) {
  std::vector<int> v(d.n_stages, 0);
  for (int j = 0; j < d.n_stages; ++j)
    for (int u = 0; u < d.stages[j].n_units; ++u) {
      int k = d.stages[j].units[u].kind;
      if (k == PETRA_UNIT_DS || k == PETRA_UNIT_STEM) v[j] += 1;
    }
  return v;
}

static std::vector<int> accum_ks(const petra_pipeline_desc &d) {
  std::vector<int> k(d.n_stages, 1);
  for (int j = 0; j < d.n_stages; ++j) k[j] = d.stages[j].accumulation_k;
  return k;
}

Pipeline::Pipeline(const petra_pipeline_desc &d)
    : J_(d.n_stages),
      rank_(d.rank),
      sched_(d.n_stages, std::vector<int>(d.stage_rank, d.stage_rank + d.n_stages), nonrev_counts(d), d.rank,
             accum_ks(d)) {
  if (J_ < 1 || J_ > PETRA_MAX_STAGES) throw PetraError(PETRA_E_ARG, "n_stages out of range");
  stages_.resize(J_ + 2);
  fwd_.resize(J_ + 2);
  bwd_.resize(J_ + 2);
  descs_.assign(d.stages, d.stages + J_);
  for (int j = 1; j <= J_; ++j) {
    if (!sched_.local(j)) continue;
    petra_stage_desc sd = d.stages[j - 1];
    sd.fifo_capacity = 2 * (J_ - j) + 1;  // Table 1: at most 2(J-j)+1 inputs in flight
    stages_[j].reset(new Stage(sd, d.seed + (uint64_t)j));
    Stage &s = *stages_[j];
    if ((j == J_) != s.is_last()) throw PetraError(PETRA_E_SHAPE, "exactly the last stage must hold the tail");
    for (int p = 0; p < 2; ++p) {
      if (j < J_) {
        fwd_[j][p].x[0] = dalloc(s.out_shape().numel() * sizeof(float));
        fwd_[j][p].x[1] = dalloc(s.out_shape().numel() * sizeof(float));
        fwd_[j][p].labels = dalloc((size_t)s.out_shape().B * sizeof(int32_t));
      }
      if (!has_stem(d.stages[j - 1])) {
        for (int k = 0; k < 4; ++k) bwd_[j][p].x[k] = dalloc(s.in_shape().numel() * sizeof(float));
      }
    }
  }
  int j0 = sched_.first_local(), j1 = sched_.last_local();
  if (j1 < 1) throw PetraError(PETRA_E_ARG, "rank owns no stage");
  streams_.assign(J_ + 2, nullptr);
  done_.assign(J_ + 2, nullptr);
  for (int j = j0; j <= j1; ++j) {
    PETRA_CUDA(cudaStreamCreateWithFlags(&streams_[j], cudaStreamNonBlocking));
    PETRA_CUDA(cudaEventCreateWithFlags(&done_[j], cudaEventDisableTiming));
  }
  PETRA_CUDA(cudaEventCreateWithFlags(&start_, cudaEventDisableTiming));
  if (sched_.local(1)) {
    const Shape &in = stages_[1]->in_shape();
    int64_t n = in.numel() * (has_stem(d.stages[0]) ? 1 : 2);
    for (int p = 0; p < 2; ++p) {
      x0_stage_[p] = dalloc(n * sizeof(float));
      lab_stage_[p] = dalloc((size_t)in.B * sizeof(int32_t));
    }
  }
  const char *g = getenv("PETRA_GRAPHS");
  graphs_ = !(g && g[0] == '0');
  for (int p = 0; p < 2; ++p) {
    if (j0 > 1) {
      const Shape &in = stages_[j0]->in_shape();
      ghost_fwd_[p].x[0] = dalloc(in.numel() * sizeof(float));
      ghost_fwd_[p].x[1] = dalloc(in.numel() * sizeof(float));
      ghost_fwd_[p].labels = dalloc((size_t)in.B * sizeof(int32_t));
    }
    if (j1 < J_) {
      const Shape &out = stages_[j1]->out_shape();
      for (int k = 0; k < 4; ++k) ghost_bwd_[p].x[k] = dalloc(out.numel() * sizeof(float));
    }
  }
}

cudaEvent_t Pipeline::ev() {
  if (ev_next_ == ev_pool_.size()) {
    cudaEvent_t e;
    PETRA_CUDA(cudaEventCreate(&e));
    ev_pool_.push_back(e);
  }
  return ev_pool_[ev_next_++];
}

void Pipeline::timing(bool on) {
  PETRA_CUDA(cudaDeviceSynchronize());
  for (auto &v : tev_) v.clear();
  ev_next_ = 0;
  timed_ticks_ = 0;
  timing_ = on;
}

int Pipeline::stage_ms(float *ms, int n) {
  PETRA_CUDA(cudaDeviceSynchronize());
  for (int j = 1; j <= J_ && j <= n; ++j) {
    double acc = 0;
    for (auto &pr : tev_[j]) {
      float x = 0.f;
      PETRA_CUDA(cudaEventElapsedTime(&x, pr.first, pr.second));
      acc += x;
    }
    ms[j - 1] = (float)acc;
  }
  return timed_ticks_;
}

Pipeline::~Pipeline() {
  for (auto e : ev_pool_) cudaEventDestroy(e);
  for (auto s : streams_)
    if (s) cudaStreamDestroy(s);
  for (auto e : done_)
    if (e) cudaEventDestroy(e);
  if (start_) cudaEventDestroy(start_);
}

static float *fp(const DevPtr &p) { return p ? p->as<float>() : nullptr; }

void Pipeline::tick(int64_t t, bool inject, const float *x0, const int32_t *labels, float lr, float *loss,
                    cudaStream_t st, petra_tick_report *rep) {
  std::vector<int64_t> ver, fifo;
  std::vector<Schedule::Step> steps = sched_.tick(t, inject, &ver, &fifo);
  const int p = (int)(t & 1), q = p ^ 1;
  const cudaStream_t caller = st;
  PETRA_CUDA(cudaEventRecord(start_, caller));  // fork: everything before this tick is visible
  for (int j = 1; j <= J_; ++j) {
    if (!sched_.local(j)) continue;
    Stage &s = *stages_[j];
    st = Prof::enabled ? caller : streams_[j];  // profiled replay: one stream, kernels timed alone
    PETRA_CUDA(cudaStreamWaitEvent(st, start_, 0));
    const Schedule::Step &sp = steps[j];
    TickArgs a;
    a.fwd = sp.fwd_mb >= 0;
    a.bwd = sp.bwd_mb >= 0;
    a.fmb = (uint64_t)std::max<int64_t>(sp.fwd_mb, 0);
    a.bmb = (uint64_t)std::max<int64_t>(sp.bwd_mb, 0);
    // ---- forward input message
    if (a.fwd) {
      if (j == 1) {
        if (!x0 || !labels) throw PetraError(PETRA_E_ARG, "inject on the rank of stage 1 needs x0 and labels");
        // copy into fixed staging buffers: the captured graph reads fixed addresses
        PETRA_CUDA(cudaMemcpyAsync(x0_stage_[p]->p, x0, x0_stage_[p]->bytes, cudaMemcpyDeviceToDevice, st));
        PETRA_CUDA(cudaMemcpyAsync(lab_stage_[p]->p, labels, lab_stage_[p]->bytes, cudaMemcpyDeviceToDevice, st));
        a.x1 = x0_stage_[p]->as<float>();
        a.x2 = has_stem(descs_[0]) ? nullptr : a.x1 + s.in_shape().numel();
        a.labels = lab_stage_[p]->as<int32_t>();
      } else {
        Msg &m = sched_.local(j - 1) ? fwd_[j - 1][q] : ghost_fwd_[q];
        a.x1 = fp(m.x[0]);
        a.x2 = fp(m.x[1]);
        a.labels = m.labels->as<int32_t>();
      }
    }
    if (j < J_) {
      if (a.fwd) {
        Msg &o = fwd_[j][p];
        a.o[0] = fp(o.x[0]);
        a.o[1] = fp(o.x[1]);
        PETRA_CUDA(cudaMemcpyAsync(o.labels->p, a.labels, (size_t)s.out_shape().B * sizeof(int32_t),
                                   cudaMemcpyDeviceToDevice, st));
      }
      if (a.bwd) {
        Msg &m = sched_.local(j + 1) ? bwd_[j + 1][q] : ghost_bwd_[q];
        for (int k = 0; k < 2; ++k) {
          a.xt[k] = fp(m.x[k]);
          a.d[k] = fp(m.x[2 + k]);
        }
      }
    }
    if (a.bwd || (j == J_ && a.fwd)) {
      Msg &o = bwd_[j][p];
      for (int k = 0; k < 2; ++k) {
        a.oxt[k] = fp(o.x[k]);
        a.od[k] = fp(o.x[2 + k]);
      }
    }
    if (j == J_) a.loss = loss;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timing_) {
      e0 = ev();
      e1 = ev();
      PETRA_CUDA(cudaEventRecord(e0, st));
    }
    s.tick(a, lr, st, graphs_);
    if (timing_) {
      PETRA_CUDA(cudaEventRecord(e1, st));
      tev_[j].push_back({e0, e1});
    }
    PETRA_CUDA(cudaEventRecord(done_[j], st));
  }
  if (timing_) ++timed_ticks_;
  for (int j = 1; j <= J_; ++j)  // join: the caller's stream sees the whole tick
    if (sched_.local(j)) PETRA_CUDA(cudaStreamWaitEvent(caller, done_[j], 0));
  if (rep) {
    rep->tick = t;
    rep->n_stages = J_;
    for (int j = 1; j <= J_; ++j) {
      rep->fwd_mb[j - 1] = steps[j].fwd_mb;
      rep->bwd_mb[j - 1] = steps[j].bwd_mb;
      rep->param_version[j - 1] = ver[j];
      rep->fifo_depth[j - 1] = fifo[j];
    }
  }
}

void Pipeline::comm(int64_t t, petra_comm_plan *plan) {
  plan->n = 0;
  const int p = (int)(t & 1);
  auto add = [&](int peer, int send, const DevPtr &buf) {
    if (plan->n >= PETRA_MAX_COMM) throw PetraError(PETRA_E_ARG, "comm plan overflow");
    petra_comm_entry &e = plan->e[plan->n++];
    e.peer = peer;
    e.send = send;
    e.ptr = buf->p;
    e.bytes = (int64_t)buf->bytes;
  };
  for (const Schedule::Comm &c : sched_.comm(t)) {
    if (c.kind == Schedule::MSG_FWD) {
      Msg &m = c.send ? fwd_[c.stage][p] : ghost_fwd_[p];
      add(c.peer, c.send, m.x[0]);
      add(c.peer, c.send, m.x[1]);
      add(c.peer, c.send, m.labels);
    } else {
      Msg &m = c.send ? bwd_[c.stage][p] : ghost_bwd_[p];
      for (int k = 0; k < 4; ++k) add(c.peer, c.send, m.x[k]);
    }
  }
}

}  // namespace petra

// pipeline.cu -- the stages of one rank, their double-buffered mailboxes, the
// per-tick driver and the neighbour exchange (product code).
//
// Exchange (library transports, include/petra.h "pipeline"): two comm streams, one
// per direction.  Tick t (parity p, q = p ^ 1):
//   stage j0 (first local, j0 > 1) forward  waits  recv_done(FWD, q)  (message of tick t-1)
//   stage j1 (last local,  j1 < J) forward  waits  cdone[FWD][p]      (its send of t-2 released
//                                                                      fwd_[j1][p])
//   stage j1 backward                       waits  recv_done(BWD, q)
//   stage j0 backward                       waits  cdone[BWD][p]      (bwd_[j0][p] released)
// and every stage records fdone / bdone (its forward / backward part) and tdone (its
// whole tick) per parity.  After enqueuing the stages, the FWD comm stream waits for
// fdone[j1][p] (the message is final) and tdone[j0][q] (ghost_fwd[p] was last read at
// t-1), moves the forward messages, records cdone[FWD][p]; the BWD stream likewise
// with bdone[j0][p] and tdone[j1][q].  So the forward exchange of tick t runs under
// that tick's backwards, and at tick t+1 only the stages that consume a received
// message wait for it.
#include "pipeline.h"

#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

namespace petra {

// LOCAL transport: the pipelines of one process that form one group, by rank
static std::mutex g_hub_mu;
static std::map<int64_t, std::vector<Pipeline *>> g_hub;

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
      world_(d.world),
      transport_(d.transport),
      group_(d.local_group),
      join_comm_(d.join_comm != 0),
      wire_(d.wire),
      sched_(d.n_stages, std::vector<int>(d.stage_rank, d.stage_rank + d.n_stages), nonrev_counts(d), d.rank,
             accum_ks(d)) {
  if (J_ < 1 || J_ > PETRA_MAX_STAGES) throw PetraError(PETRA_E_ARG, "n_stages out of range");
  if (world_ < 1 || rank_ < 0 || rank_ >= world_) throw PetraError(PETRA_E_ARG, "rank / world out of range");
  if (transport_ < PETRA_TRANSPORT_NONE || transport_ > PETRA_TRANSPORT_LOCAL)
    throw PetraError(PETRA_E_ARG, "unknown transport");
  if (transport_ == PETRA_TRANSPORT_NCCL && !d.nccl_id) throw PetraError(PETRA_E_ARG, "NCCL transport needs nccl_id");
  if (transport_ == PETRA_TRANSPORT_LOCAL && group_ == 0) throw PetraError(PETRA_E_ARG, "LOCAL transport needs local_group");
  if (wire_ != PETRA_WIRE_FP32 && wire_ != PETRA_WIRE_BF16) throw PetraError(PETRA_E_ARG, "unknown wire format");
  {  // persistent-grid caps for the stages sharing this GPU (prof.cu; PETRA_STAGES_PER_GPU pins it)
    int n = 0;
    for (int j = 1; j <= J_; ++j) n += sched_.local(j) ? 1 : 0;
    const int pin = env_int("PETRA_STAGES_PER_GPU", 0);
    set_stages_per_gpu(pin > 0 ? pin : n);
  }
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
  // stage streams rank between a stage's backward stream (highest) and its wgrad stream
  // (lowest) when stream priorities are on (stage.cu, PETRA_STREAM_PRIO)
  int prio_lo = 0, prio_hi = 0;
  PETRA_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  const bool prio_on = env_int("PETRA_STREAM_PRIO", 1) != 0;
  // the final stage runs forward, loss and backward as ONE chain on its stage stream (no
  // backward side stream): PETRA_TAIL_PRIO=1 gives that stream the backward streams' rank
  // (2: one rank below the backward streams)
  const int tail_p = env_int("PETRA_TAIL_PRIO", 1);  // R18 +2.4 % (profiles/r02/tuning/tail_priority.txt)
  const int tail_rank = tail_p == 1 ? prio_hi : (tail_p == 2 ? std::min(prio_lo, prio_hi + 1) : (prio_lo + prio_hi) / 2);
  // PETRA_FWD_PRIO (experiment): ranks above the middle for the other stages' streams
  const int fwd_up = env_int("PETRA_FWD_PRIO", 0);
  const int mid = std::max(prio_hi, (prio_lo + prio_hi) / 2 - fwd_up);
  for (int j = j0; j <= j1; ++j) {
    if (prio_on)
      PETRA_CUDA(cudaStreamCreateWithPriority(&streams_[j], cudaStreamNonBlocking, j == J_ ? tail_rank : mid));
    else PETRA_CUDA(cudaStreamCreateWithFlags(&streams_[j], cudaStreamNonBlocking));
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
  if (lib_transport() && wire_ == PETRA_WIRE_BF16) {  // 2-byte images of the cross-rank messages
    for (int p = 0; p < 2; ++p) {
      if (j1 < J_) {  // forward send of j1, backward receive for j1
        const int64_t n = stages_[j1]->out_shape().numel();
        for (int k = 0; k < 2; ++k) wsend_[DIR_FWD][p].x[k] = dalloc(n * sizeof(__nv_bfloat16));
        for (int k = 0; k < 4; ++k) wrecv_[DIR_BWD][p].x[k] = dalloc(n * sizeof(__nv_bfloat16));
      }
      if (j0 > 1) {  // forward receive for j0, backward send of j0
        const int64_t n = stages_[j0]->in_shape().numel();
        for (int k = 0; k < 2; ++k) wrecv_[DIR_FWD][p].x[k] = dalloc(n * sizeof(__nv_bfloat16));
        for (int k = 0; k < 4; ++k) wsend_[DIR_BWD][p].x[k] = dalloc(n * sizeof(__nv_bfloat16));
      }
    }
  }
  if (lib_transport()) {
    fdone_.assign(J_ + 2, {nullptr, nullptr});
    bdone_.assign(J_ + 2, {nullptr, nullptr});
    tdone_.assign(J_ + 2, {nullptr, nullptr});
    for (int j = j0; j <= j1; ++j)
      for (int p = 0; p < 2; ++p) {
        PETRA_CUDA(cudaEventCreateWithFlags(&fdone_[j][p], cudaEventDisableTiming));
        PETRA_CUDA(cudaEventCreateWithFlags(&bdone_[j][p], cudaEventDisableTiming));
        PETRA_CUDA(cudaEventCreateWithFlags(&tdone_[j][p], cudaEventDisableTiming));
      }
    for (int dir = 0; dir < 2; ++dir) {
      PETRA_CUDA(cudaStreamCreateWithFlags(&cs_[dir], cudaStreamNonBlocking));
      for (int p = 0; p < 2; ++p) PETRA_CUDA(cudaEventCreateWithFlags(&cdone_[dir][p], cudaEventDisableTiming));
    }
  }
  if (transport_ == PETRA_TRANSPORT_NCCL) {
    ncclUniqueId id;
    std::memcpy(&id, d.nccl_id, sizeof(id));
    PETRA_NCCL(nccl().CommInitRank(&nccl_comm_, world_, id, rank_));
  } else if (transport_ == PETRA_TRANSPORT_LOCAL) {
    std::lock_guard<std::mutex> lk(g_hub_mu);
    auto &v = g_hub[group_];
    if ((int)v.size() < world_) v.resize(world_, nullptr);
    if (v[rank_]) throw PetraError(PETRA_E_ARG, "LOCAL transport: rank already registered in this group");
    v[rank_] = this;
  }
}

Pipeline *Pipeline::peer(int rank) const {
  std::lock_guard<std::mutex> lk(g_hub_mu);
  auto it = g_hub.find(group_);
  if (it == g_hub.end() || rank >= (int)it->second.size() || !it->second[rank])
    throw PetraError(PETRA_E_ARG, "LOCAL transport: rank " + std::to_string(rank) + " has no pipeline in the group");
  return it->second[rank];
}

// the event that completes when the message of direction `dir` produced at a tick of
// parity `parity` has arrived in this rank's ghost buffer
cudaEvent_t Pipeline::recv_done(int dir, int parity) const {
  if (transport_ == PETRA_TRANSPORT_NCCL) return cdone_[dir][parity];  // this rank's own receive
  // LOCAL: the sender pushed it on its comm stream
  const int src = dir == DIR_FWD ? sched_.rank_of(sched_.first_local() - 1) : sched_.rank_of(sched_.last_local() + 1);
  return peer(src)->cdone_[dir][parity];
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
  cudaDeviceSynchronize();  // mailboxes and ghost buffers may still be in use (see ~Stage)
  if (transport_ == PETRA_TRANSPORT_LOCAL) {
    std::lock_guard<std::mutex> lk(g_hub_mu);
    auto it = g_hub.find(group_);
    if (it != g_hub.end()) {
      if (rank_ < (int)it->second.size() && it->second[rank_] == this) it->second[rank_] = nullptr;
      bool empty = true;
      for (auto *q : it->second) empty &= q == nullptr;
      if (empty) g_hub.erase(it);
    }
  }
  for (int dir = 0; dir < 2; ++dir)
    if (cs_[dir]) cudaStreamSynchronize(cs_[dir]);
  if (nccl_comm_) nccl().CommDestroy(nccl_comm_);
  for (int dir = 0; dir < 2; ++dir) {
    if (cs_[dir]) cudaStreamDestroy(cs_[dir]);
    for (int p = 0; p < 2; ++p)
      if (cdone_[dir][p]) cudaEventDestroy(cdone_[dir][p]);
  }
  for (auto *v : {&fdone_, &bdone_, &tdone_})
    for (auto &pr : *v)
      for (cudaEvent_t e : pr)
        if (e) cudaEventDestroy(e);
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
  NvtxRange tick_range("petra tick %lld (rank %d)", (long long)t, rank_);
  std::vector<int64_t> ver, fifo;
  std::vector<Schedule::Step> steps = sched_.tick(t, inject, &ver, &fifo);
  const int p = (int)(t & 1), q = p ^ 1;
  const cudaStream_t caller = st;
  PETRA_CUDA(cudaEventRecord(start_, caller));  // fork: everything before this tick is visible
  for (int j = 1; j <= J_; ++j) {
    if (!sched_.local(j)) continue;
    Stage &s = *stages_[j];
    // profiled replay: every local stage on ONE of the pipeline's (capturable, non-blocking)
    // streams, so kernels run and are timed alone
    int jl = 1;
    while (!sched_.local(jl)) ++jl;
    st = Prof::enabled ? streams_[jl] : streams_[j];
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
    a.round_msgs = wire_ == PETRA_WIRE_BF16;
    if (lib_transport()) {  // cross-rank synchronisation points (header comment)
      const int j0 = sched_.first_local(), j1 = sched_.last_local();
      if (a.fwd) {
        if (j == j0 && j > 1) a.wait_f[0] = recv_done(DIR_FWD, q);
        if (j == j1 && j < J_) a.wait_f[1] = cdone_[DIR_FWD][p];
        a.done_f = fdone_[j][p];
      }
      if (a.bwd) {
        if (j == j1 && j < J_) a.wait_b[0] = recv_done(DIR_BWD, q);
        if (j == j0 && j > 1) a.wait_b[1] = cdone_[DIR_BWD][p];
        a.done_b = bdone_[j][p];
      }
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timing_) {
      e0 = ev();
      e1 = ev();
      PETRA_CUDA(cudaEventRecord(e0, st));
    }
    {
      NvtxRange r("stage %d: fwd mb %lld, bwd mb %lld", j, (long long)sp.fwd_mb, (long long)sp.bwd_mb);
      s.tick(a, lr, st, graphs_);
    }
    if (timing_) {
      PETRA_CUDA(cudaEventRecord(e1, st));
      tev_[j].push_back({e0, e1});
    }
    PETRA_CUDA(cudaEventRecord(done_[j], st));
    if (lib_transport()) PETRA_CUDA(cudaEventRecord(tdone_[j][p], st));
  }
  if (timing_) ++timed_ticks_;
  std::vector<bool> used(2, false);
  if (lib_transport()) exchange(t, used);
  for (int j = 1; j <= J_; ++j)  // join: the caller's stream sees the whole tick
    if (sched_.local(j)) PETRA_CUDA(cudaStreamWaitEvent(caller, done_[j], 0));
  if (join_comm_)
    for (int dir = 0; dir < 2; ++dir)
      if (used[dir]) PETRA_CUDA(cudaStreamWaitEvent(caller, cdone_[dir][p], 0));
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

void Pipeline::exchange(int64_t t, std::vector<bool> &used) {
  const int p = (int)(t & 1), q = p ^ 1;
  const int j0 = sched_.first_local(), j1 = sched_.last_local();
  std::vector<Schedule::Comm> msgs = sched_.comm(t);
  for (int dir = 0; dir < 2; ++dir) {
    std::vector<const Schedule::Comm *> ops;
    for (const Schedule::Comm &c : msgs)
      if (c.kind == (dir == DIR_FWD ? Schedule::MSG_FWD : Schedule::MSG_BWD)) ops.push_back(&c);
    if (ops.empty()) continue;
    used[dir] = true;
    cudaStream_t cs = cs_[dir];
    for (const Schedule::Comm *c : ops) {
      if (c->send) {  // the message is final when the sending part of the stage is done
        PETRA_CUDA(cudaStreamWaitEvent(cs, dir == DIR_FWD ? fdone_[j1][p] : bdone_[j0][p], 0));
      } else {        // this rank's ghost buffer of parity p was last read at tick t-1
        PETRA_CUDA(cudaStreamWaitEvent(cs, dir == DIR_FWD ? tdone_[j0][q] : tdone_[j1][q], 0));
      }
    }
    NvtxRange nr(dir == DIR_FWD ? "exchange fwd (x1, x2, labels -> rank+1)" : "exchange bwd (x~, delta -> rank-1)");
    ProfScope ps(dir == DIR_FWD ? "exchange_fwd" : "exchange_bwd", cs, 0.0, 0.0);
    const bool w16 = wire_ == PETRA_WIRE_BF16;
    const int nt = dir == DIR_FWD ? 2 : 4;  // message tensors (labels travel as int32)
    if (transport_ == PETRA_TRANSPORT_NCCL) {
      const NcclApi &nc = nccl();
      if (w16)  // pack: the values are bf16-exact (rounded by the producing stage)
        for (const Schedule::Comm *c : ops)
          if (c->send) {
            Msg &m = dir == DIR_FWD ? fwd_[j1][p] : bwd_[j0][p];
            for (int k = 0; k < nt; ++k)
              f32_to_bf16(m.x[k]->as<float>(), wsend_[dir][p].x[k]->as<__nv_bfloat16>(),
                          (int64_t)(m.x[k]->bytes / sizeof(float)), cs);
          }
      PETRA_NCCL(nc.GroupStart());
      for (const Schedule::Comm *c : ops) {
        Msg &m = dir == DIR_FWD ? (c->send ? fwd_[j1][p] : ghost_fwd_[p]) : (c->send ? bwd_[j0][p] : ghost_bwd_[p]);
        Msg &wm = c->send ? wsend_[dir][p] : wrecv_[dir][p];
        for (int k = 0; k <= nt; ++k) {
          const DevPtr &b = k < nt ? (w16 ? wm.x[k] : m.x[k]) : m.labels;
          if (!b) continue;
          if (c->send) PETRA_NCCL(nc.Send(b->p, b->bytes, ncclUint8, c->peer, nccl_comm_, cs));
          else PETRA_NCCL(nc.Recv(b->p, b->bytes, ncclUint8, c->peer, nccl_comm_, cs));
        }
      }
      PETRA_NCCL(nc.GroupEnd());
      if (w16)  // unpack into the fp32 ghost buffers (exact widening)
        for (const Schedule::Comm *c : ops)
          if (!c->send) {
            Msg &g = dir == DIR_FWD ? ghost_fwd_[p] : ghost_bwd_[p];
            for (int k = 0; k < nt; ++k)
              bf16_to_f32(wrecv_[dir][p].x[k]->as<__nv_bfloat16>(), g.x[k]->as<float>(),
                          (int64_t)(g.x[k]->bytes / sizeof(float)), cs);
          }
    } else {  // LOCAL: push into the receiver's ghost buffer once it released it
      for (const Schedule::Comm *c : ops) {
        if (!c->send) continue;
        Pipeline *pr = peer(c->peer);
        const int rj = dir == DIR_FWD ? pr->sched_.first_local() : pr->sched_.last_local();
        PETRA_CUDA(cudaStreamWaitEvent(cs, pr->tdone_[rj][q], 0));
        Msg &src = dir == DIR_FWD ? fwd_[j1][p] : bwd_[j0][p];
        Msg &dst = dir == DIR_FWD ? pr->ghost_fwd_[p] : pr->ghost_bwd_[p];
        for (int k = 0; k <= nt; ++k) {
          const DevPtr &a = k < nt ? src.x[k] : src.labels;
          const DevPtr &b = k < nt ? dst.x[k] : dst.labels;
          if (!a || !b) continue;
          if (a->bytes != b->bytes) throw PetraError(PETRA_E_SHAPE, "LOCAL transport: message sizes differ");
          if (w16 && k < nt) {  // the same 2-byte wire as NCCL: pack, move, widen
            const DevPtr &ws = wsend_[dir][p].x[k], &wr = pr->wrecv_[dir][p].x[k];
            const int64_t n = (int64_t)(a->bytes / sizeof(float));
            f32_to_bf16(a->as<float>(), ws->as<__nv_bfloat16>(), n, cs);
            PETRA_CUDA(cudaMemcpyAsync(wr->p, ws->p, ws->bytes, cudaMemcpyDeviceToDevice, cs));
            bf16_to_f32(wr->as<__nv_bfloat16>(), b->as<float>(), n, cs);
            continue;
          }
          PETRA_CUDA(cudaMemcpyAsync(b->p, a->p, a->bytes, cudaMemcpyDeviceToDevice, cs));
        }
      }
    }
    PETRA_CUDA(cudaEventRecord(cdone_[dir][p], cs));
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

// stage.cu -- PETRA stage engine (product code): builds the unit list of a stage,
// owns theta / v / Delta / running stats / FIFOs / workspace, and enqueues the
// kernel sequence of a forward tick, a backward tick (approximate inversion +
// VJP + immediate update) and the final-stage step.
//
// Paper map:
//   forward                PAPER.md:131, Alg. 1 lines 3-10
//   backward, reversible   PAPER.md:132-135, Alg. 1 lines 12-21; "a reconstruction step
//                          and a backward step": the recomputed conv
//                          outputs z of the reconstruction ARE the graph of the VJP
//   backward, non-rev      Alg. 1 lines 15-17 (buffer + recompute), reading c5/c6
//   final stage            Alg. 1 lines 26-35, readings c7/c10
//   BN running stats       PAPER.md:259 (updated only when recomputing)
//   update                 PAPER.md:135, 256 (Nesterov 0.9, wd exclusions)
#include "stage.h"

#include <algorithm>

#include <cstdlib>

#include <cmath>
#include <cstring>

#include "errors.h"

namespace petra {

// bytes allocated by the stage under construction (Stage::memory)
static thread_local size_t *g_alloc_acc = nullptr;

// device allocator (petra_set_allocator): cudaMalloc / cudaFree unless the caller installed
// its own (e.g. PyTorch's caching allocator); a buffer remembers who allocated it
Allocator &allocator() {
  static Allocator a;
  return a;
}

DevBuf::DevBuf(size_t n) : bytes(n) {
  if (n == 0) return;
  if (g_alloc_acc) *g_alloc_acc += n;
  const Allocator a = allocator();
  if (a.alloc) {
    int dev = 0;
    PETRA_CUDA(cudaGetDevice(&dev));
    p = a.alloc(n, dev, a.ctx);
    if (!p) throw PetraError(PETRA_E_OOM, "installed allocator returned NULL for " + std::to_string(n) + " bytes");
    release = a.release;
    ctx = a.ctx;
    device = dev;
    return;
  }
  cudaError_t e = cudaMalloc(&p, n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw PetraError(PETRA_E_OOM, "cudaMalloc(" + std::to_string(n) + "): " + cudaGetErrorString(e));
  }
}
DevBuf::~DevBuf() {
  if (!p) return;
  if (release) release(p, device, ctx);
  else cudaFree(p);
}
DevPtr dalloc(size_t bytes) { return DevPtr(new DevBuf(bytes)); }

namespace {

uint64_t splitmix(uint64_t &s) {
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void check_conv(const petra_conv &c) {
  if (c.cin <= 0 || c.cout <= 0 || c.ksize <= 0 || c.stride <= 0 || (c.ksize % 2) == 0)
    throw PetraError(PETRA_E_ARG, "invalid conv (cin/cout/ksize/stride must be positive, ksize odd)");
}

}  // namespace

// ------------------------------------------------------------------ construction
Stage::Stage(const petra_stage_desc &desc, uint64_t seed) : desc_(desc) {
  if (desc.n_units <= 0 || !desc.units) throw PetraError(PETRA_E_ARG, "stage needs at least one unit");
  if (desc.batch <= 0 || desc.in_h <= 0 || desc.in_w <= 0 || desc.in_c <= 0)
    throw PetraError(PETRA_E_ARG, "non-positive stage input shape");
  if (desc.precision != PETRA_FP32 && desc.precision != PETRA_BF16_TC)
    throw PetraError(PETRA_E_ARG, "unknown precision");
  if (desc.accumulation_k < 1) throw PetraError(PETRA_E_ARG, "accumulation_k must be >= 1");
  if (!(desc.momentum >= 0.f) || !(desc.weight_decay >= 0.f) || !(desc.bn_eps > 0.f))
    throw PetraError(PETRA_E_ARG, "bad optimizer / BN hyper-parameters");
  tc_ = desc.precision == PETRA_BF16_TC;
  int dev = 0;
  PETRA_CUDA(cudaGetDevice(&dev));
  units_.resize(desc.n_units);
  for (int i = 0; i < desc.n_units; ++i) units_[i].d = desc.units[i];
  struct AccGuard {
    explicit AccGuard(size_t *p) { g_alloc_acc = p; }
    ~AccGuard() { g_alloc_acc = nullptr; }
  } guard(&alloc_bytes_);
  build();
  init_params(seed);
}

Stage::~Stage() {
  // the device may still run this stage's work; its buffers go back to an allocator
  // (cudaFree, or a caller's caching pool that would hand them out again at once)
  cudaDeviceSynchronize();
  for (auto &kv : graphs_) cudaGraphExecDestroy(kv.second.exec);
  for (auto ex : prof_execs_) cudaGraphExecDestroy(ex);
  if (side_) cudaStreamDestroy(side_);
  if (fork_) cudaEventDestroy(fork_);
  if (join_) cudaEventDestroy(join_);
  if (eu_b_) cudaEventDestroy(eu_b_);
  if (fwd_done_) cudaEventDestroy(fwd_done_);
  if (wg_) cudaStreamDestroy(wg_);
  if (wg_fork_) cudaEventDestroy(wg_fork_);
  if (wg_join_) cudaEventDestroy(wg_join_);
  if (lr_host_) cudaFreeHost(lr_host_);
}

int64_t Stage::add_tensor(int unit, int part, int kind, int decay, std::vector<int> shape, bool buffer) {
  petra_tensor_info t{};
  t.unit = unit;
  t.part = part;
  t.kind = kind;
  t.decay = decay;
  t.ndim = (int)shape.size();
  int64_t cnt = 1;
  for (int i = 0; i < t.ndim; ++i) {
    t.shape[i] = shape[i];
    cnt *= shape[i];
  }
  t.count = cnt;
  if (buffer) {
    t.offset = n_buffers_;
    n_buffers_ += cnt;
  } else {
    t.offset = n_params_;
    n_params_ += cnt;
  }
  tensors_.push_back(t);
  return t.offset;
}

void Stage::alloc_layer(Layer &L, bool inner) {
  int64_t n = L.g.M() * L.g.Co;
  L.ctx = &ctx_;
  L.z16 = tc_ && (conv_tc_supported(L.g, 0) || stem_tc_supported(L.g));
  for (int c = 0; c < 2; ++c) {
    L.z_[c] = dalloc(n * (L.z16 ? sizeof(__nv_bfloat16) : sizeof(float)));
    L.mean_[c] = dalloc(L.g.Co * sizeof(float));
    L.invstd_[c] = dalloc(L.g.Co * sizeof(float));
    if (inner) L.a_[c] = dalloc(n * sizeof(float));
  }
  L.dz = dalloc(n * sizeof(float));
  if (inner) L.da = dalloc(n * sizeof(float));
  if (tc_) {
    L.w_bf16 = dalloc((int64_t)L.g.Co * L.g.K() * sizeof(__nv_bfloat16));
    L.wt_bf16 = dalloc((int64_t)L.g.Co * L.g.K() * sizeof(__nv_bfloat16));
    // 3x3 stride-1 layers keep their bf16 operands zero-bordered for the halo kernel
    // (on by default; PETRA_HALO=0 keeps every layer on the per-tap im2col kernel)
    static const bool halo = [] {
      const char *e = getenv("PETRA_HALO");
      return !(e && e[0] == '0');
    }();
    const bool s1k3 = halo && !L.is_stem && L.g.k == 3 && L.g.s == 1;
    L.xpad = s1k3 && conv_tc_supported(L.g, 0) && conv_halo_eligible(L.g.B, L.g.H, L.g.W, L.g.Ci, L.g.Co);
    L.dzpad = s1k3 && conv_tc_supported(L.g, 1) && conv_halo_eligible(L.g.B, L.g.Ho, L.g.Wo, L.g.Co, L.g.Ci);
    const int64_t nxb = L.xpad ? (int64_t)L.g.B * (L.g.H + 2) * (L.g.W + 2) * L.g.Ci
                        : (L.is_stem && stem_tc_supported(L.g)) ? (int64_t)stem_operand_elems(L.g)
                                                                 : L.g.Min() * L.g.Ci;
    const int64_t ndz = L.dzpad ? (int64_t)L.g.B * (L.g.Ho + 2) * (L.g.Wo + 2) * L.g.Co : n;
    L.dzb = dalloc(ndz * sizeof(__nv_bfloat16));
    if (L.dzpad) PETRA_CUDA(cudaMemset(L.dzb->p, 0, ndz * sizeof(__nv_bfloat16)));  // borders stay zero
    for (int c = 0; c < 2 && !L.operand_of && !L.fifo_backed; ++c) {
      L.xb_[c] = dalloc(nxb * sizeof(__nv_bfloat16));
      if (L.xpad) PETRA_CUDA(cudaMemset(L.xb_[c]->p, 0, nxb * sizeof(__nv_bfloat16)));
    }
  }
}

void Stage::build() {
  const int B = desc_.batch;
  Shape cur{B, desc_.in_h, desc_.in_w, desc_.in_c};
  in_ = cur;
  size_t max_part = 0, max_spart = 0, max_ws = 0;
  std::vector<std::vector<Layer *>> unit_layers(units_.size());
  struct Pending {
    Layer *L;
    int unit, part;
  };
  std::vector<Pending> layers;
  for (size_t ui = 0; ui < units_.size(); ++ui) {
    Unit &u = units_[ui];
    const petra_unit &d = u.d;
    u.in = cur;
    if (d.kind == PETRA_UNIT_TAIL && ui + 1 != units_.size())
      throw PetraError(PETRA_E_SHAPE, "the tail must be the last unit of its stage");
    if (d.kind == PETRA_UNIT_STEM && ui != 0) throw PetraError(PETRA_E_SHAPE, "the stem must be the first unit");
    switch (d.kind) {
      case PETRA_UNIT_STEM: {
        check_conv(d.layer[0]);
        if (d.layer[0].cin != cur.C) throw PetraError(PETRA_E_SHAPE, "stem cin != image channels");
        if (d.layer[0].cout % 2) throw PetraError(PETRA_E_ODD_CHANNELS, "stem output channels must be even");
        u.phi.resize(1);
        Layer &L = u.phi[0];
        L.g = make_geom(B, cur.H, cur.W, cur.C, d.layer[0].cout, d.layer[0].ksize, d.layer[0].stride);
        L.relu = true;
        L.is_stem = true;
        layers.push_back({&L, (int)ui, 0});
        int Ho = L.g.Ho, Wo = L.g.Wo;
        if (d.maxpool) {
          u.ctx = &ctx_;
          for (int c = 0; c < 2; ++c) u.pool_a_[c] = dalloc(L.g.M() * L.g.Co * sizeof(float));
          Ho = (Ho + 2 - 3) / 2 + 1;
          Wo = (Wo + 2 - 3) / 2 + 1;
          for (int c = 0; c < 2; ++c) u.pool_arg_[c] = dalloc((int64_t)B * Ho * Wo * L.g.Co);
        }
        cur = Shape{B, Ho, Wo, d.layer[0].cout / 2};
        break;
      }
      case PETRA_UNIT_REV:
      case PETRA_UNIT_DS: {
        if (d.dst_half != 0 && d.dst_half != 1) throw PetraError(PETRA_E_ARG, "dst_half must be 0 or 1");
        if (d.n_layers < 1 || d.n_layers > 3) throw PetraError(PETRA_E_ARG, "n_layers must be 1..3");
        u.phi.resize(d.n_layers);
        Shape s = cur;
        for (int l = 0; l < d.n_layers; ++l) {
          check_conv(d.layer[l]);
          if (d.layer[l].cin != s.C)
            throw PetraError(PETRA_E_SHAPE, "unit " + std::to_string(ui) + " layer " + std::to_string(l) +
                                                ": cin " + std::to_string(d.layer[l].cin) + " != " +
                                                std::to_string(s.C));
          Layer &L = u.phi[l];
          L.g = make_geom(B, s.H, s.W, s.C, d.layer[l].cout, d.layer[l].ksize, d.layer[l].stride);
          L.relu = true;
          layers.push_back({&L, (int)ui, l});
          s = Shape{B, L.g.Ho, L.g.Wo, L.g.Co};
        }
        if (d.kind == PETRA_UNIT_REV) {
          if (s != cur) throw PetraError(PETRA_E_SHAPE, "reversible unit must preserve the half shape");
        } else {
          for (int k = 0; k < 2; ++k) {
            check_conv(d.proj[k]);
            if (d.proj[k].cin != cur.C || d.proj[k].cout != s.C)
              throw PetraError(PETRA_E_SHAPE, "DS projection channels do not match");
            Layer &P = k == 0 ? u.pa : u.pb;
            P.g = make_geom(B, cur.H, cur.W, cur.C, d.proj[k].cout, d.proj[k].ksize, d.proj[k].stride);
            P.relu = false;
            if (P.g.Ho != s.H || P.g.Wo != s.W) throw PetraError(PETRA_E_SHAPE, "DS projection stride mismatch");
            layers.push_back({&P, (int)ui, 3 + k});
          }
          cur = s;
        }
        break;
      }
      case PETRA_UNIT_TAIL: {
        if (d.classes <= 0) throw PetraError(PETRA_E_ARG, "classes must be positive");
        is_last_ = true;
        break;
      }
      default:
        throw PetraError(PETRA_E_ARG, "unknown unit kind");
    }
    u.out = cur;
  }
  out_ = is_last_ ? Shape{B, 1, 1, units_.back().d.classes} : cur;

  // ---- parameter layout: per unit, per layer (W, gamma, beta); tail (W, b); then buffers
  for (auto &p : layers) {
    Layer &L = *p.L;
    L.w_off = add_tensor(p.unit, p.part, PETRA_T_CONV_W, 1, {L.g.Co, L.g.k, L.g.k, L.g.Ci}, false);
    L.g_off = add_tensor(p.unit, p.part, PETRA_T_BN_GAMMA, 0, {L.g.Co}, false);
    L.b_off = add_tensor(p.unit, p.part, PETRA_T_BN_BETA, 0, {L.g.Co}, false);
  }
  if (is_last_) {
    Unit &t = units_.back();
    t.fc_w = add_tensor((int)units_.size() - 1, 0, PETRA_T_FC_W, 1, {t.d.classes, 2 * t.in.C}, false);
    t.fc_b = add_tensor((int)units_.size() - 1, 0, PETRA_T_FC_B, 0, {t.d.classes}, false);
  }
  for (auto &p : layers) {
    Layer &L = *p.L;
    L.rm_off = add_tensor(p.unit, p.part, PETRA_T_BN_RMEAN, 0, {L.g.Co}, true);
    L.rv_off = add_tensor(p.unit, p.part, PETRA_T_BN_RVAR, 0, {L.g.Co}, true);
  }
  theta_ = dalloc(n_params_ * sizeof(float));
  v_ = dalloc(n_params_ * sizeof(float));
  grad_ = dalloc(n_params_ * sizeof(float));
  if (desc_.accumulation_k > 1) {  // Delta_j of Alg. 1: the running average of k backwards
    acc_ = dalloc(n_params_ * sizeof(float));
    PETRA_CUDA(cudaMemset(acc_->p, 0, n_params_ * sizeof(float)));
  }
  bufs_ = dalloc(std::max<int64_t>(1, n_buffers_) * sizeof(float));
  PETRA_CUDA(cudaMemset(grad_->p, 0, n_params_ * sizeof(float)));

  // ---- bf16 operands of non-reversible units live in their FIFO slots (tensor-core
  // path, plain layouts): converted once in the forward, reused by the recomputation
  if (tc_ && desc_.precision == PETRA_BF16_TC) {
    for (auto &u : units_) {
      auto plain = [&](const Layer &L) { return conv_tc_supported(L.g, 0) && !(L.g.k == 3 && L.g.s == 1); };
      if (u.d.kind == PETRA_UNIT_DS && plain(u.pa) && plain(u.phi[0]))
        u.pa.fifo_backed = u.phi[0].fifo_backed = true;
      if (u.d.kind == PETRA_UNIT_STEM && stem_tc_supported(u.phi[0].g)) u.phi[0].fifo_backed = true;
    }
  }
  // ---- workspace
  for (auto &u : units_) {
    for (size_t l = 0; l < u.phi.size(); ++l) alloc_layer(u.phi[l], l + 1 < u.phi.size());
    if (u.d.kind == PETRA_UNIT_DS) {
      alloc_layer(u.pa, false);
      // P_b reads the same tensor as the branch's first conv (x[src]): one bf16 operand
      // for both when neither uses the zero-bordered layout (written by the branch first)
      Layer &f = u.phi[0];
      if (tc_ && conv_tc_supported(u.pb.g, 0) && conv_tc_supported(f.g, 0) && !f.xpad && !f.is_stem &&
          f.g.H == u.pb.g.H && f.g.W == u.pb.g.W && f.g.Ci == u.pb.g.Ci)
        u.pb.operand_of = &f;
      alloc_layer(u.pb, false);
    }
  }
  for (auto &p : layers) {
    max_part = std::max(max_part, bn_partial_bytes(p.L->g.M(), p.L->g.Co));
    max_spart = std::max(max_spart, (size_t)kNumSMs * 4 * (p.L->g.Co * 2 + 1) * sizeof(float));  // fused conv stats
    max_ws = std::max(max_ws, conv_wgrad_simt_workspace(p.L->g));
    if (tc_)
      for (int mode = 0; mode < 3; ++mode) max_ws = std::max(max_ws, conv_tc_workspace(p.L->g, mode));
    if (tc_) max_ws = std::max(max_ws, stem_tc_workspace(p.L->g));
  }
  size_t max_ctr = 1;
  for (auto &p : layers) max_ctr = std::max(max_ctr, bn_counter_count(p.L->g.Co));
  for (int c = 0; c < 2; ++c) {
    part_[c] = dalloc(std::max<size_t>(max_part, 16));
    spart_[c] = dalloc(std::max<size_t>(max_spart, 16));
    counters_[c] = dalloc(max_ctr * sizeof(unsigned));
    PETRA_CUDA(cudaMemset(counters_[c]->p, 0, max_ctr * sizeof(unsigned)));
    wgrad_ws_[c] = dalloc(std::max<size_t>(max_ws, 16));
  }
  // stream priorities (PETRA_STREAM_PRIO=1): the backward -- a stage's longer half, on the
  // tick's critical path -- outranks the forward; the wgrads (needed only by the update)
  // rank lowest; the block scheduler then hands freed SMs to the critical work first
  static const bool prio_on = env_int("PETRA_STREAM_PRIO", 1) != 0;
  int prio_lo = 0, prio_hi = 0;
  PETRA_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  if (prio_on) PETRA_CUDA(cudaStreamCreateWithPriority(&side_, cudaStreamNonBlocking, prio_hi));
  else PETRA_CUDA(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
  PETRA_CUDA(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming));
  PETRA_CUDA(cudaEventCreateWithFlags(&join_, cudaEventDisableTiming));
  PETRA_CUDA(cudaEventCreateWithFlags(&eu_b_, cudaEventDisableTiming));
  PETRA_CUDA(cudaEventCreateWithFlags(&fwd_done_, cudaEventDisableTiming));
  if (tc_ && env_int("PETRA_WGRAD_STREAM", 1)) {
    // PETRA_WGRAD_PRIO: 0 lowest (default), 1 the forward's rank, 2 the backward's
    static const int wprio = env_int("PETRA_WGRAD_PRIO", 0);
    const int wp = wprio >= 2 ? prio_hi : (wprio == 1 ? (prio_lo + prio_hi) / 2 : prio_lo);
    if (prio_on) PETRA_CUDA(cudaStreamCreateWithPriority(&wg_, cudaStreamNonBlocking, wp));
    else PETRA_CUDA(cudaStreamCreateWithFlags(&wg_, cudaStreamNonBlocking));
    PETRA_CUDA(cudaEventCreateWithFlags(&wg_fork_, cudaEventDisableTiming));
    PETRA_CUDA(cudaEventCreateWithFlags(&wg_join_, cudaEventDisableTiming));
    wg_ws_ = dalloc(std::max<size_t>(max_ws, 16));
  }
  // Table 3 comparison buffers (memory measurement; numerics unchanged)
  if (desc_.compare_buffers & PETRA_CMP_INPUTS) {
    const bool own_fifo = !units_.empty() && units_[0].d.kind != PETRA_UNIT_REV;  // PETRA buffers these already
    if (!own_fifo)
      for (int s = 0; s < std::max(1, desc_.fifo_capacity); ++s)
        for (int h = 0; h < 2; ++h) cmp_in_[h].push_back(dalloc(in_.numel() * sizeof(float)));
  }
  if (desc_.compare_buffers & PETRA_CMP_STASH)
    for (int s = 0; s < desc_.fifo_capacity - 1; ++s) cmp_stash_.push_back(dalloc(theta_->bytes));
  lr_dev_ = dalloc(sizeof(float));
  PETRA_CUDA(cudaMallocHost(&lr_host_, kLrRing * sizeof(float)));
  if (tc_) conv_tc_prepare();
  nonfinite_ = dalloc(sizeof(int));
  evalflag_ = dalloc(sizeof(int));  // the evaluation tail's non-finite flag (not latched)
  PETRA_CUDA(cudaMemset(evalflag_->p, 0, sizeof(int)));
  PETRA_CUDA(cudaMemset(nonfinite_->p, 0, sizeof(int)));

  // ---- output-target planning (see header of forward/backward)
  const int n = (int)units_.size();
  int cap = std::max(1, desc_.fifo_capacity);
  for (int i = 0; i < n; ++i) {
    Unit &u = units_[i];
    bool later_nonrev = false, earlier_nonrev = false;
    for (int k = i + 1; k < n; ++k)
      if (units_[k].d.kind == PETRA_UNIT_DS || units_[k].d.kind == PETRA_UNIT_STEM) later_nonrev = true;
    for (int k = 0; k < i; ++k)
      if (units_[k].d.kind == PETRA_UNIT_DS || units_[k].d.kind == PETRA_UNIT_STEM) earlier_nonrev = true;
    if (u.d.kind == PETRA_UNIT_TAIL) continue;
    bool need_fout = later_nonrev || is_last_;
    if (need_fout)
      for (int h = 0; h < 2; ++h) u.fout[h] = dalloc(u.out.numel() * sizeof(float));
    // a reversible unit reconstructs into its own buffer when the half it receives is
    // read-only FIFO memory of an earlier unit's input or, in the final stage, of a
    // later non-reversible unit (the tail has no caller output to reconstruct into)
    if (earlier_nonrev || (is_last_ && later_nonrev)) {
      for (int h = 0; h < 2; ++h) {
        if (u.d.kind == PETRA_UNIT_REV) u.bx[h] = dalloc(u.in.numel() * sizeof(float));
        if (u.d.kind != PETRA_UNIT_STEM) u.bd[h] = dalloc(u.in.numel() * sizeof(float));
      }
    } else if (u.d.kind == PETRA_UNIT_DS && is_last_) {
      for (int h = 0; h < 2; ++h) u.bd[h] = dalloc(u.in.numel() * sizeof(float));
    }
    if (u.d.kind == PETRA_UNIT_DS || u.d.kind == PETRA_UNIT_STEM) {
      u.fifo.cap = is_last_ ? 1 : cap;
      for (int s = 0; s < u.fifo.cap; ++s) {
        // the stem's fp32 input is needed only by SIMT passes: with its bf16 operand in the
        // slot (tensor cores) and no backward message (stage 1 sends none), it is not kept
        if (!(u.d.kind == PETRA_UNIT_STEM && u.phi[0].fifo_backed))
          u.fifo.slot0.push_back(dalloc(u.in.numel() * sizeof(float)));
        if (u.d.kind == PETRA_UNIT_DS) u.fifo.slot1.push_back(dalloc(u.in.numel() * sizeof(float)));
        if (u.d.kind == PETRA_UNIT_DS && u.pa.fifo_backed) {
          u.fifo.bslot0.push_back(dalloc(u.in.numel() * sizeof(__nv_bfloat16)));
          u.fifo.bslot1.push_back(dalloc(u.in.numel() * sizeof(__nv_bfloat16)));
        } else if (u.d.kind == PETRA_UNIT_STEM && u.phi[0].fifo_backed) {
          u.fifo.bslot0.push_back(dalloc(stem_operand_elems(u.phi[0].g) * sizeof(__nv_bfloat16)));
        }
      }
    }
  }
  if (is_last_) {
    Unit &t = units_.back();
    int Cin = 2 * t.in.C;
    feat_ = dalloc((int64_t)B * Cin * sizeof(float));
    logits_ = dalloc((int64_t)B * t.d.classes * sizeof(float));
    dlogits_ = dalloc((int64_t)B * t.d.classes * sizeof(float));
    lossrow_ = dalloc((int64_t)B * sizeof(float));
    dfeat_ = dalloc((int64_t)B * Cin * sizeof(float));
    fc_ws_floats_ = 16 * (int64_t)B * std::max(Cin, t.d.classes);  // split-K partials of the FC GEMMs
    fc_ws_ = dalloc(fc_ws_floats_ * sizeof(float));
    for (int h = 0; h < 2; ++h) tail_d_[h] = dalloc(t.in.numel() * sizeof(float));
  }

  // ---- optimizer segments
  for (auto &t : tensors_) {
    if (t.kind > PETRA_T_FC_B) continue;
    SgdSeg s{};
    s.offset = t.offset;
    s.count = t.count;
    s.decay = t.decay;
    segs_.push_back(s);
    max_seg_ = std::max<int64_t>(max_seg_, t.count);
  }
  if (tc_) {
    for (auto &p : layers) {
      for (auto &s : segs_)
        if (s.offset == p.L->w_off) {
          s.co = p.L->g.Co;
          s.k = p.L->g.k;
          s.ci = p.L->g.Ci;
          s.w_bf16 = p.L->w_bf16->as<__nv_bfloat16>();
          s.wt_bf16 = p.L->wt_bf16->as<__nv_bfloat16>();
        }
    }
  }
  segs_dev_ = dalloc(segs_.size() * sizeof(SgdSeg));
  PETRA_CUDA(cudaMemcpy(segs_dev_->p, segs_.data(), segs_.size() * sizeof(SgdSeg), cudaMemcpyHostToDevice));
  const std::vector<SgdChunk> chunks = sgd_chunks(segs_);
  n_chunks_ = (int)chunks.size();
  {  // per-unit chunk ranges (segments follow tensors_ order; chunks follow segments)
    std::vector<int> seg_unit;
    for (auto &t : tensors_)
      if (t.kind <= PETRA_T_FC_B) seg_unit.push_back(t.unit);
    const int nu = (int)units_.size();
    unit_chunk_lo_.assign(nu, 0);
    unit_chunk_hi_.assign(nu, 0);
    std::vector<int> seen(nu, 0);
    early_ok_ = (int)seg_unit.size() == (int)segs_.size();
    int prev = -1;
    for (int c = 0; c < n_chunks_ && early_ok_; ++c) {
      const int u = seg_unit[chunks[c].seg];
      if (u < 0 || u >= nu) { early_ok_ = false; break; }
      if (u != prev) {
        if (seen[u]) early_ok_ = false;  // a unit's items must be one contiguous range
        seen[u] = 1;
        unit_chunk_lo_[u] = c;
        prev = u;
      }
      unit_chunk_hi_[u] = c + 1;
    }
  }
  chunks_dev_ = dalloc(std::max<size_t>(1, chunks.size()) * sizeof(SgdChunk));
  PETRA_CUDA(cudaMemcpy(chunks_dev_->p, chunks.data(), chunks.size() * sizeof(SgdChunk), cudaMemcpyHostToDevice));
}

void Stage::init_params(uint64_t seed) {
  std::vector<float> th(n_params_, 0.f), bufs(std::max<int64_t>(1, n_buffers_), 0.f);
  uint64_t s = seed * 0x2545F4914F6CDD1Dull + 1;
  for (auto &t : tensors_) {
    float *dst = (t.kind >= PETRA_T_BN_RMEAN ? bufs.data() : th.data()) + t.offset;
    if (t.kind == PETRA_T_CONV_W || t.kind == PETRA_T_FC_W) {
      int64_t fan_in = t.count / t.shape[0];
      double b = std::sqrt(6.0 / (double)fan_in);
      for (int64_t i = 0; i < t.count; ++i) {
        double u = (double)(splitmix(s) >> 11) * (1.0 / 9007199254740992.0);
        dst[i] = (float)((2.0 * u - 1.0) * b);
      }
    } else if (t.kind == PETRA_T_BN_GAMMA || t.kind == PETRA_T_BN_RVAR) {
      for (int64_t i = 0; i < t.count; ++i) dst[i] = 1.f;
    }
  }
  std::vector<float> zeros(n_params_, 0.f);
  set_params(th.data(), zeros.data(), bufs.data());
}

// ------------------------------------------------------------------ params
void Stage::set_params(const float *theta, const float *v, const float *bufs) {
  if (theta) PETRA_CUDA(cudaMemcpy(theta_->p, theta, n_params_ * sizeof(float), cudaMemcpyHostToDevice));
  if (v) PETRA_CUDA(cudaMemcpy(v_->p, v, n_params_ * sizeof(float), cudaMemcpyHostToDevice));
  if (bufs && n_buffers_)
    PETRA_CUDA(cudaMemcpy(bufs_->p, bufs, n_buffers_ * sizeof(float), cudaMemcpyHostToDevice));
  if (tc_ && theta) {
    sgd_update(segs_dev_->as<SgdSeg>(), (int)segs_.size(), chunks_dev_->as<SgdChunk>(), n_chunks_, theta_->as<float>(),
               v_->as<float>(),
               grad_->as<float>(), nullptr, 1, SGD_PLAIN, nullptr, 0.f, 0.f, 1, nullptr, /*shadow_only=*/true,
               nonfinite_->as<int>());
    PETRA_CUDA(cudaDeviceSynchronize());
  }
}

void Stage::get_params(float *theta, float *v, float *bufs) {
  PETRA_CUDA(cudaDeviceSynchronize());
  if (theta) PETRA_CUDA(cudaMemcpy(theta, theta_->p, n_params_ * sizeof(float), cudaMemcpyDeviceToHost));
  if (v) PETRA_CUDA(cudaMemcpy(v, v_->p, n_params_ * sizeof(float), cudaMemcpyDeviceToHost));
  if (bufs && n_buffers_)
    PETRA_CUDA(cudaMemcpy(bufs, bufs_->p, n_buffers_ * sizeof(float), cudaMemcpyDeviceToHost));
}

void Stage::get_grads(float *delta) {
  PETRA_CUDA(cudaDeviceSynchronize());
  PETRA_CUDA(cudaMemcpy(delta, grad_->p, n_params_ * sizeof(float), cudaMemcpyDeviceToHost));
}

int Stage::nonfinite() {
  int h = 0;
  PETRA_CUDA(cudaDeviceSynchronize());
  PETRA_CUDA(cudaMemcpy(&h, nonfinite_->p, sizeof(int), cudaMemcpyDeviceToHost));
  return h;
}

void Stage::memory(petra_memory_report *r) const {
  auto b = [](const DevPtr &p) -> uint64_t { return p ? p->bytes : 0; };
  *r = petra_memory_report{};
  r->params = b(theta_) + (n_buffers_ ? b(bufs_) : 0);
  r->optimizer = b(v_) + b(grad_) + b(acc_);
  auto layer = [&](const Layer &L) { r->shadows += b(L.w_bf16) + b(L.wt_bf16); };
  for (auto &u : units_) {
    for (auto &L : u.phi) layer(L);
    if (u.d.kind == PETRA_UNIT_DS) {
      layer(u.pa);
      layer(u.pb);
    }
    uint64_t slot = 0, all = 0;
    for (size_t s = 0; s < (size_t)u.fifo.cap; ++s) {
      uint64_t one = (s < u.fifo.slot0.size() ? b(u.fifo.slot0[s]) : 0) +
                     (s < u.fifo.slot1.size() ? b(u.fifo.slot1[s]) : 0) +
                     (s < u.fifo.bslot0.size() ? b(u.fifo.bslot0[s]) : 0) +
                     (s < u.fifo.bslot1.size() ? b(u.fifo.bslot1[s]) : 0);
      all += one;
      slot = one;
    }
    r->fifo += all;
    r->fifo_live += slot * (uint64_t)u.fifo.size;
  }
  for (int h = 0; h < 2; ++h)
    for (auto &p : cmp_in_[h]) r->cmp_inputs += b(p);
  for (auto &p : cmp_stash_) r->cmp_stash += b(p);
  r->total = alloc_bytes_;
  r->workspace = r->total - r->params - r->optimizer - r->shadows - r->fifo - r->cmp_inputs - r->cmp_stash;
}

int Stage::fifo_depth() const {
  int d = 0;
  for (auto &u : units_) d += u.fifo.size;
  return d;
}

// the tick's learning rate -> device scalar (pinned ring: the async copy's source
// stays valid while up to kLrRing ticks are in flight)
void Stage::upload_lr(float lr, cudaStream_t st) {
  float *h = lr_host_ + (lr_next_++ % kLrRing);
  *h = lr;
  PETRA_CUDA(cudaMemcpyAsync(lr_dev_->p, h, sizeof(float), cudaMemcpyHostToDevice, st));
}

// the optimizer mode of the backward about to be enqueued (Alg. 1 lines 19-23:
// Delta += Delta_mb / k every backward, update and reset when t mod k == 0, t from 1)
int Stage::next_update_mode() const {
  const int k = desc_.accumulation_k;
  if (k == 1) return SGD_PLAIN;
  return (t_ % k == 0) ? SGD_ACC_UPDATE : SGD_ACCUMULATE;
}

void Stage::advance_step(int mode) {
  ++t_;
  if (mode != SGD_ACCUMULATE) ++version_;
}

void Stage::enqueue_update(int mode, cudaStream_t st) {
  ProfScope ps("sgd_update", st, 0.0,
               (mode == SGD_PLAIN ? 20.0 : mode == SGD_ACCUMULATE ? 12.0 : 28.0) * (double)n_params_);
  sgd_update(segs_dev_->as<SgdSeg>(), (int)segs_.size(), chunks_dev_->as<SgdChunk>(), n_chunks_, theta_->as<float>(),
               v_->as<float>(),
             grad_->as<float>(), acc_ ? acc_->as<float>() : nullptr, desc_.accumulation_k, mode, lr_dev_->as<float>(),
             desc_.momentum, desc_.weight_decay, desc_.nesterov, st, false, nonfinite_->as<int>());
}

// unit `u`'s update on the wgrad stream, ordered after everything `st` (the backward
// stream) has enqueued so far -- the unit's dgrad, BN-backward sums and SIMT wgrads -- its
// tensor-core wgrads (already on the wgrad stream) and, once, this tick's forward
void Stage::early_update(int u, cudaStream_t st) {
  if (!eu_.active || u < 0 || u >= (int)eu_.done.size() || unit_chunk_hi_[u] <= unit_chunk_lo_[u]) return;
  PETRA_CUDA(cudaEventRecord(eu_b_, st));
  PETRA_CUDA(cudaStreamWaitEvent(wg_, eu_b_, 0));
  if (eu_.fwd_pending) {
    PETRA_CUDA(cudaStreamWaitEvent(wg_, fwd_done_, 0));
    eu_.fwd_pending = false;
  }
  const int lo = unit_chunk_lo_[u], n = unit_chunk_hi_[u] - lo;
  ProfScope ps("sgd_update", wg_, 0.0, 0.0);
  sgd_update(segs_dev_->as<SgdSeg>(), (int)segs_.size(), chunks_dev_->as<SgdChunk>() + lo, n, theta_->as<float>(),
             v_->as<float>(), grad_->as<float>(), acc_ ? acc_->as<float>() : nullptr, desc_.accumulation_k, eu_.mode,
             lr_dev_->as<float>(), desc_.momentum, desc_.weight_decay, desc_.nesterov, wg_, false,
             nonfinite_->as<int>());
  wg_active_ = true;
  eu_.done[u] = 1;
}

// the tick's update of every unit not updated early (all of them when early updates are off)
void Stage::enqueue_update_rest(int mode, cudaStream_t st) {
  const bool any = eu_.active && std::any_of(eu_.done.begin(), eu_.done.end(), [](char c) { return c != 0; });
  eu_.active = false;
  if (!any) {
    enqueue_update(mode, st);
    return;
  }
  for (int u = 0; u < (int)eu_.done.size(); ++u) {
    if (eu_.done[u] || unit_chunk_hi_[u] <= unit_chunk_lo_[u]) continue;
    const int lo = unit_chunk_lo_[u], n = unit_chunk_hi_[u] - lo;
    ProfScope ps("sgd_update", st, 0.0, 0.0);
    sgd_update(segs_dev_->as<SgdSeg>(), (int)segs_.size(), chunks_dev_->as<SgdChunk>() + lo, n, theta_->as<float>(),
               v_->as<float>(), grad_->as<float>(), acc_ ? acc_->as<float>() : nullptr, desc_.accumulation_k, mode,
               lr_dev_->as<float>(), desc_.momentum, desc_.weight_decay, desc_.nesterov, st, false,
               nonfinite_->as<int>());
  }
}

// ------------------------------------------------------------------ layer kernels
static void apply_bn(int64_t M, int C, const void *z, bool z16, int ldz, int zc0, const float *mean,
                     const float *invstd, const float *gamma, const float *beta, int relu, float sign,
                     const float *acc, float *out, __nv_bfloat16 *out_bf16, cudaStream_t st, int pH = 0,
                     int pW = 0, const StatsFold *fold = nullptr) {
  ProfScope ps("bn_apply", st, 0.0,
               (double)M * C * ((z16 ? 2.0 : 4.0) + (acc ? 4.0 : 0.0) + (out ? 4.0 : 0.0) + (out_bf16 ? 2.0 : 0.0)));
  if (z16)
    bn_apply<__nv_bfloat16, float>(M, C, static_cast<const __nv_bfloat16 *>(z), ldz, zc0, mean, invstd, gamma, beta,
                                   relu, sign, acc, out, out_bf16, pH, pW, st, fold);
  else
    bn_apply<float, float>(M, C, static_cast<const float *>(z), ldz, zc0, mean, invstd, gamma, beta, relu, sign, acc,
                           out, out_bf16, pH, pW, st, fold);
}

static double conv_flops(const ConvGeom &g) { return 2.0 * (double)g.M() * g.Co * g.K(); }
// algorithmic HBM bytes of one convolution pass: operands once (elements of size esz),
// the result once (out_es bytes per element) and the addend once (dgrad)
enum { PASS_FWD = 0, PASS_DGRAD = 1, PASS_WGRAD = 2 };
static double conv_bytes(const ConvGeom &g, int esz, int pass, int out_es, bool addend = false) {
  const double x = (double)g.Min() * g.Ci, w = (double)g.Co * g.K(), z = (double)g.M() * g.Co;
  if (pass == PASS_FWD) return esz * (x + w) + out_es * z;
  if (pass == PASS_DGRAD) return esz * (z + w) + (out_es + (addend ? 4.0 : 0.0)) * x;
  return esz * (x + z) + out_es * w;
}

void Stage::conv_fwd(Layer &L, const float *x, cudaStream_t st, bool x_bf16_ready, bool running) {
  flush_fold(st);  // this conv's epilogue rewrites the context's partial rows
  const float *w = theta_->as<float>() + L.w_off;
  if (tc_ && stem_tc_supported(L.g)) {  // few input channels: gathered im2col from a 4-channel bf16 copy
    if (!x_bf16_ready) {
      ProfScope pc("cvt_bf16", st, 0.0, (4.0 * L.g.Ci + 8.0) * (double)L.g.Min());
      image_to_bf16x4(x, L.xbp(), L.g, st);
    }
    ProfScope ps("conv_fwd_stem_tc", st, conv_flops(L.g), conv_bytes(L.g, 2, PASS_FWD, L.z16 ? 2 : 4));
    L.stats_rows() = stem_fwd_tc(L.g, L.xbp(), w, L.z()->p, L.z16,
                                 reinterpret_cast<float *>(spart()->p), st);
    return;
  }
  bool tc = tc_ && conv_tc_supported(L.g, 0);
  if (tc && !x_bf16_ready) {  // bf16 operand of a stream input (also read by the TC wgrad)
    ProfScope pc("cvt_bf16", st, 0.0, 6.0 * (double)L.g.Min() * L.g.Ci);
    if (L.xpad) f32_to_bf16_padded(x, L.xbp(), L.g.B, L.g.H, L.g.W, L.g.Ci, st);
    else f32_to_bf16(x, L.xbp(), L.g.Min() * L.g.Ci, st);
  }
  ProfScope ps(tc ? "conv_fwd_tc" : "conv_fwd_simt", st, conv_flops(L.g),
               conv_bytes(L.g, tc ? 2 : 4, PASS_FWD, L.z16 ? 2 : 4));
  if (tc) {
    L.stats_rows() = conv_fwd_tc(L.g, L.xbp(), L.xpad, L.w_bf16->as<__nv_bfloat16>(), L.z()->p, L.z16,
                                 wgrad_ws()->as<float>(), reinterpret_cast<float *>(spart()->p), st);
  } else {
    conv_fwd_simt(L.g, x, w, L.z()->as<float>(), st, tc_);
  }
}

// the wgrads' stream back into `st` (before the update reads Delta)
void Stage::join_wgrads(cudaStream_t st) {
  if (!wg_active_) return;
  PETRA_CUDA(cudaEventRecord(wg_join_, wg_));
  PETRA_CUDA(cudaStreamWaitEvent(st, wg_join_, 0));
  wg_active_ = false;
}

void Stage::conv_wgrad(Layer &L, const float *x, cudaStream_t st) {
  float *dw = grad_->as<float>() + L.w_off;
  const bool stem = tc_ && stem_tc_supported(L.g);
  bool tc = tc_ && conv_tc_supported(L.g, 2);
  float *ws = wgrad_ws()->as<float>();
  // tensor-core wgrads read only the bf16 operands (L.xbp, L.dzb), which nothing later in
  // the walk rewrites: off the critical path onto the wgrad stream (not in a profiled,
  // serialised replay; SIMT wgrads read the fp32 input, which a later reconstruction may
  // overwrite in place, and stay on `st`)
  if ((stem || tc) && wg_ && !Prof::enabled) {
    PETRA_CUDA(cudaEventRecord(wg_fork_, st));
    PETRA_CUDA(cudaStreamWaitEvent(wg_, wg_fork_, 0));
    st = wg_;
    ws = wg_ws_->as<float>();
    wg_active_ = true;
  }
  if (stem) {
    ProfScope ps("conv_wgrad_stem_tc", st, conv_flops(L.g), conv_bytes(L.g, 2, PASS_WGRAD, 4));
    stem_wgrad_tc(L.g, L.dzb->as<__nv_bfloat16>(), L.xbp(), dw, ws, st);
    return;
  }
  ProfScope ps(tc ? "conv_wgrad_tc" : "conv_wgrad_simt", st, conv_flops(L.g),
               conv_bytes(L.g, tc ? 2 : 4, PASS_WGRAD, 4));
  if (tc) {
    // L.xb holds bf16(x) from the conv_fwd of this tick (forward or recomputation);
    // L.dzb was written in bf16 by bn_bwd_dz
    conv_wgrad_tc(L.g, L.dzb->as<__nv_bfloat16>(), L.dzpad, L.xbp(), L.xpad, dw, ws, st);
  } else {
    conv_wgrad_simt(L.g, L.dz->as<float>(), x, dw, wgrad_ws()->as<float>(), st, tc_);
  }
}

void Stage::conv_dgrad(Layer &L, const float *addend, float *out, cudaStream_t st) {
  bool tc = tc_ && conv_tc_supported(L.g, 1);
  ProfScope ps(tc ? "conv_dgrad_tc" : "conv_dgrad_simt", st, conv_flops(L.g),
               conv_bytes(L.g, tc ? 2 : 4, PASS_DGRAD, 4, addend != nullptr));
  if (tc) {
    conv_dgrad_tc(L.g, L.dzb->as<__nv_bfloat16>(), L.dzpad, L.wt_bf16->as<__nv_bfloat16>(), addend, out,
                  wgrad_ws()->as<float>(), st);
  } else {
    conv_dgrad_simt(L.g, L.dz->as<float>(), theta_->as<float>() + L.w_off, addend, out, st, tc_);
  }
}

// Statistics of a conv output whose epilogue wrote partial rows are merged by the BN
// pass that consumes them (StatsFold, the pass's prologue); a fold not consumed before
// the next conv epilogue of the context rewrites the rows is launched on its own.
void Stage::flush_fold(cudaStream_t st) {
  Layer *L = pending_[ctx_];
  if (!L) return;
  pending_[ctx_] = nullptr;
  StatsFold &f = L->fold();
  if (!f.part) return;
  ProfScope ps("bn_stats_merge", st, 0.0, 8.0 * f.rows * L->g.Co / f.groups);
  StatsRows r;
  r.rows = f.rows;
  r.groups = f.groups;
  bn_stats_from_partials(f.part, r, f.N, f.M, f.eps, L->mean()->as<float>(), L->invstd()->as<float>(), f.rmean,
                         f.rvar, f.mom, st);
  f = StatsFold{};
}

const StatsFold *Stage::take_fold(Layer &L) {
  if (pending_[ctx_] != &L || !L.fold().part) return nullptr;
  pending_[ctx_] = nullptr;
  fold_tmp_[ctx_] = L.fold();
  L.fold() = StatsFold{};
  return &fold_tmp_[ctx_];
}

void Stage::layer_stats(Layer &L, bool running, cudaStream_t st) {
  float *b = bufs_->as<float>();
  if (eval_) {  // evaluation: normalise by the running statistics
    L.stats_rows() = StatsRows{};
    bn_running_constants(b + L.rm_off, b + L.rv_off, L.g.Co, desc_.bn_eps, L.mean()->as<float>(),
                         L.invstd()->as<float>(), st);
    return;
  }
  if (L.stats_rows().rows > 0) {  // sums already produced by the tensor-core conv epilogue
    flush_fold(st);
    StatsFold f;
    f.part = reinterpret_cast<const float *>(spart()->p);
    f.rows = L.stats_rows().rows;
    f.groups = L.stats_rows().groups;
    f.N = L.g.Co;
    f.M = L.g.M();
    f.eps = desc_.bn_eps;
    f.mom = desc_.bn_momentum;
    f.rmean = running ? b + L.rm_off : nullptr;
    f.rvar = running ? b + L.rv_off : nullptr;
    L.fold() = f;
    L.stats_rows() = StatsRows{};
    pending_[ctx_] = &L;
    // off by default: every block of the consuming pass merging the partial rows of its
    // channel tile costs more than the launch it saves (measured)
    static const bool fold_on = env_int("PETRA_STATS_FOLD", 0) != 0;
    if (!fold_on) flush_fold(st);
    return;
  }
  ProfScope ps("bn_stats", st, 0.0, 4.0 * (double)L.g.M() * L.g.Co);
  if (L.z16)
    bn_stats<__nv_bfloat16>(L.z()->as<__nv_bfloat16>(), L.g.M(), L.g.Co, desc_.bn_eps, L.mean()->as<float>(),
                            L.invstd()->as<float>(), running ? b + L.rm_off : nullptr,
                            running ? b + L.rv_off : nullptr, desc_.bn_momentum, part()->as<double>(),
                            counters()->as<unsigned>(), st);
  else
    bn_stats<float>(L.z()->as<float>(), L.g.M(), L.g.Co, desc_.bn_eps, L.mean()->as<float>(), L.invstd()->as<float>(),
                    running ? b + L.rm_off : nullptr, running ? b + L.rv_off : nullptr, desc_.bn_momentum,
                    part()->as<double>(), counters()->as<unsigned>(), st);
}

// forward of a conv-BN-ReLU chain on x; inner activations into L.a; the last
// layer's z / stats are left for the caller's fused epilogue.
void Stage::branch_forward(std::vector<Layer> &phi, const float *x, bool running, cudaStream_t st, bool ready0) {
  const float *th = theta_->as<float>();
  bool ready = ready0;
  for (size_t l = 0; l < phi.size(); ++l) {
    Layer &L = phi[l];
    conv_fwd(L, x, st, ready, running);
    layer_stats(L, running, st);
    if (l + 1 < phi.size()) {
      // inner activation; its bf16 copy is written straight into the next layer's operand
      Layer &N = phi[l + 1];
      ready = tc_ && conv_tc_supported(N.g, 0);
      // the fp32 copy only feeds SIMT passes of the next layer (forward or wgrad)
      const bool need32 = !ready || !conv_tc_supported(N.g, 2);
      apply_bn(L.g.M(), L.g.Co, L.z()->p, L.z16, L.g.Co, 0, L.mean()->as<float>(), L.invstd()->as<float>(),
               th + L.g_off, th + L.b_off, 1, 1.f, nullptr, need32 ? L.a()->as<float>() : nullptr,
               ready ? N.xbp() : nullptr, st, N.xpad ? N.g.H : 0, N.g.W, take_fold(L));
      x = L.a()->as<float>();
    }
  }
}

// BN(+ReLU) backward of one layer given dy (gradient wrt the layer output);
// optional fused reconstruction dst_out = dst_in - act(bn(z)); writes dgamma,
// dbeta into Delta and dz into L.dz.
void Stage::layer_bwd(Layer &L, const float *dy0, const float *dy1, int cs, const float *dst_in, float *dst_out,
                      cudaStream_t st, Bf16Out ob) {
  const float *th = theta_->as<float>();
  float *gr = grad_->as<float>();
  double n = (double)L.g.M() * L.g.Co;
  const StatsFold *fold = take_fold(L);
  {
  ProfScope ps("bn_bwd_reduce", st, 0.0, n * ((L.z16 ? 2.0 : 4.0) + 4.0 + (dst_out ? 8.0 : 0.0) + (ob.p ? 2.0 : 0.0)));
  if (L.z16)
    bn_bwd_reduce<__nv_bfloat16>(L.z()->as<__nv_bfloat16>(), L.g.M(), L.g.Co, L.mean()->as<float>(),
                                 L.invstd()->as<float>(), th + L.g_off, th + L.b_off, L.relu ? 1 : 0, dy0, dy1, cs,
                                 dst_in, dst_out, ob.p, ob.pH, ob.pW, gr + L.g_off, gr + L.b_off,
                                 part()->as<double>(), counters()->as<unsigned>(), st, fold);
  else
    bn_bwd_reduce<float>(L.z()->as<float>(), L.g.M(), L.g.Co, L.mean()->as<float>(), L.invstd()->as<float>(),
                         th + L.g_off, th + L.b_off, L.relu ? 1 : 0, dy0, dy1, cs, dst_in, dst_out, ob.p, ob.pH,
                         ob.pW, gr + L.g_off, gr + L.b_off, part()->as<double>(), counters()->as<unsigned>(), st,
                         fold);
  }
  // dz in bf16 for tensor-core dgrad / wgrad, in fp32 only if a SIMT pass consumes it
  // (the stem has no dgrad: its input is data)
  const bool tc_d = tc_ && (L.is_stem || conv_tc_supported(L.g, 1));
  const bool tc_w = tc_ && (conv_tc_supported(L.g, 2) || stem_tc_supported(L.g));
  float *dz32 = (!tc_d || !tc_w) ? L.dz->as<float>() : nullptr;
  __nv_bfloat16 *dz16 = (tc_d || tc_w) ? L.dzb->as<__nv_bfloat16>() : nullptr;
  ProfScope ps("bn_bwd_dz", st, 0.0, n * ((L.z16 ? 2.0 : 4.0) + 4.0 + (dz32 ? 4.0 : 0.0) + (dz16 ? 2.0 : 0.0)));
  if (L.z16)
    bn_bwd_dz<__nv_bfloat16>(L.g.M(), L.g.Co, L.z()->as<__nv_bfloat16>(), L.mean()->as<float>(), L.invstd()->as<float>(),
                             th + L.g_off, th + L.b_off, L.relu ? 1 : 0, dy0, dy1, cs, gr + L.g_off, gr + L.b_off,
                             dz32, dz16, L.dzpad ? L.g.Ho : 0, L.g.Wo, st);
  else
    bn_bwd_dz<float>(L.g.M(), L.g.Co, L.z()->as<float>(), L.mean()->as<float>(), L.invstd()->as<float>(), th + L.g_off,
                     th + L.b_off, L.relu ? 1 : 0, dy0, dy1, cs, gr + L.g_off, gr + L.b_off, dz32, dz16,
                     L.dzpad ? L.g.Ho : 0, L.g.Wo, st);
}

// VJP through a branch whose last layer receives dy (reconstruction fused when
// dst_out != null).  dx_out = addend + d(branch)/dx^T dy  (dx_out may be null).
void Stage::branch_backward(std::vector<Layer> &phi, const float *x, const float *dy, const float *dst_in,
                            float *dst_out, const float *addend, float *dx_out, cudaStream_t st, Bf16Out ob) {
  int n = (int)phi.size();
  layer_bwd(phi[n - 1], dy, nullptr, 0, dst_in, dst_out, st, dst_out ? ob : Bf16Out{});
  for (int l = n - 1; l >= 0; --l) {
    Layer &L = phi[l];
    const float *xl = l == 0 ? x : phi[l - 1].a()->as<float>();
    conv_wgrad(L, xl, st);
    if (l > 0) {
      conv_dgrad(L, nullptr, phi[l - 1].da->as<float>(), st);
      layer_bwd(phi[l - 1], phi[l - 1].da->as<float>(), nullptr, 0, nullptr, nullptr, st);
    } else if (dx_out) {
      conv_dgrad(L, addend, dx_out, st);
    }
  }
}

// ------------------------------------------------------------------ units
// forward of one unit: cur[] = current halves (inputs), out[] = where the unit's
// outputs go (REV: only out[dst] is written; may equal cur[dst] for in place).
// The bf16 operand of the next unit's first convolution (when that unit reads the
// half this one writes): written by the producing kernel instead of a separate
// conversion pass.
Bf16Out Stage::src_operand(Unit &n) {
  if (!tc_ || n.d.kind != PETRA_UNIT_REV) return {};
  Layer &L = n.phi[0];
  if (!conv_tc_supported(L.g, 0)) return {};
  return Bf16Out{L.xbp(), L.xpad ? L.g.H : 0, L.g.W};
}

// point the FIFO-backed layers of a non-reversible unit at the bf16 slots of `slot`
void Stage::bind_fifo_operands(Unit &u, int slot) {
  if (u.fifo.bslot0.empty()) return;
  if (u.d.kind == PETRA_UNIT_STEM) {
    u.phi[0].xb_ext = u.fifo.bslot0[slot]->as<__nv_bfloat16>();
    return;
  }
  DevPtr *b[2] = {&u.fifo.bslot0[slot], &u.fifo.bslot1[slot]};
  u.pa.xb_ext = (*b[u.dst()])->as<__nv_bfloat16>();      // P_a reads x[dst]
  u.phi[0].xb_ext = (*b[u.src()])->as<__nv_bfloat16>();  // the branch (and P_b) read x[src]
}

void Stage::unit_forward(Unit &u, const float *cur[2], float *out[2], bool keep, cudaStream_t st, Bf16Out ob,
                         bool src_ready, int ob_half) {
  const float *th = theta_->as<float>();
  switch (u.d.kind) {
    case PETRA_UNIT_REV: {
      // x[dst] += Phi(x[src])  (north_star y1 = x1 + F(x2), y2 = x2 + G(y1))
      branch_forward(u.phi, cur[u.src()], keep, st, src_ready);
      Layer &L = u.phi.back();
      apply_bn(L.g.M(), L.g.Co, L.z()->p, L.z16, L.g.Co, 0, L.mean()->as<float>(), L.invstd()->as<float>(),
               th + L.g_off, th + L.b_off, 1, 1.f, cur[u.dst()], out[u.dst()], ob.p, st, ob.pH, ob.pW, take_fold(L));
      break;
    }
    case PETRA_UNIT_DS: {
      // y[dst] = P_a(x[dst]) + Phi_s(x[src]);  y[src] = P_b(x[src])
      const float *xd = cur[u.dst()], *xs = cur[u.src()];
      branch_forward(u.phi, xs, keep, st);
      conv_fwd(u.pa, xd, st, false, keep);
      layer_stats(u.pa, keep, st);
      conv_fwd(u.pb, xs, st, u.pb.operand_of != nullptr, keep);  // operand shared with the branch's first conv
      layer_stats(u.pb, keep, st);
      Layer &L = u.phi.back();
      int64_t M = L.g.M();
      int C = L.g.Co;
      const Bf16Out od = ob_half == u.dst() ? ob : Bf16Out{}, os = ob_half == u.src() ? ob : Bf16Out{};
      apply_bn(M, C, u.pa.z()->p, u.pa.z16, C, 0, u.pa.mean()->as<float>(), u.pa.invstd()->as<float>(),
                             th + u.pa.g_off, th + u.pa.b_off, 0, 1.f, nullptr, out[u.dst()], nullptr, st, 0, 0,
                             take_fold(u.pa));
      apply_bn(M, C, L.z()->p, L.z16, C, 0, L.mean()->as<float>(), L.invstd()->as<float>(), th + L.g_off,
               th + L.b_off, 1, 1.f, out[u.dst()], out[u.dst()], od.p, st, od.pH, od.pW, take_fold(L));
      apply_bn(M, C, u.pb.z()->p, u.pb.z16, C, 0, u.pb.mean()->as<float>(), u.pb.invstd()->as<float>(),
               th + u.pb.g_off, th + u.pb.b_off, 0, 1.f, nullptr, out[u.src()], os.p, st, os.pH, os.pW,
               take_fold(u.pb));
      break;
    }
    case PETRA_UNIT_STEM: {
      Layer &L = u.phi[0];
      conv_fwd(L, cur[0], st, false, keep);
      layer_stats(L, keep, st);
      int Ch = L.g.Co / 2;
      if (u.d.maxpool) {
        apply_bn(L.g.M(), L.g.Co, L.z()->p, L.z16, L.g.Co, 0, L.mean()->as<float>(),
                               L.invstd()->as<float>(), th + L.g_off, th + L.b_off, 1, 1.f, nullptr,
                               u.pool_a()->as<float>(), nullptr, st, 0, 0, take_fold(L));
        ProfScope ps("maxpool", st, 0.0, 4.0 * (double)L.g.M() * L.g.Co * 1.25);
        maxpool_fwd(u.pool_a()->as<float>(), L.g.B, L.g.Ho, L.g.Wo, L.g.Co, u.out.H, u.out.W, out[0], out[1],
                    u.pool_arg()->as<uint8_t>(), st);
      } else {
        flush_fold(st);  // two passes over halves of the channels: final statistics first
        for (int h = 0; h < 2; ++h)
          apply_bn(L.g.M(), Ch, L.z()->p, L.z16, L.g.Co, h * Ch, L.mean()->as<float>(),
                                 L.invstd()->as<float>(), th + L.g_off, th + L.b_off, 1, 1.f, nullptr, out[h],
                                 nullptr, st);
      }
      break;
    }
    default:
      throw PetraError(PETRA_E_ARG, "unit_forward: bad kind");
  }
}

// backward of one unit.  cur_x = unit output (reconstructed or current), xin =
// the unit input for non-reversible units (FIFO slot), cur_d = gradient wrt the
// unit output; out_x / out_d = targets (REV: out_x[dst], out_d[src]; DS: out_d[both]).
void Stage::unit_backward(Unit &u, bool recompute, const float *xin[2], const float *cur_x[2], float *out_x[2],
                          const float *cur_d[2], float *out_d[2], cudaStream_t st, Bf16Out ob, bool src_ready) {
  switch (u.d.kind) {
    case PETRA_UNIT_REV: {
      // approximate inversion with the current theta: recompute the
      // graph of Phi on x[src] (src is unchanged by the unit), subtract, VJP.
      const float *src = cur_x[u.src()];
      if (recompute) branch_forward(u.phi, src, true, st, src_ready);
      branch_backward(u.phi, src, cur_d[u.dst()], cur_x[u.dst()], out_x[u.dst()], cur_d[u.src()],
                      out_d[u.src()], st, ob);
      break;
    }
    case PETRA_UNIT_DS: {
      const float *xd = xin[u.dst()], *xs = xin[u.src()];
      if (recompute) {
        branch_forward(u.phi, xs, true, st, src_ready);
        conv_fwd(u.pa, xd, st, src_ready, true);
        layer_stats(u.pa, true, st);
        conv_fwd(u.pb, xs, st, u.pb.operand_of != nullptr, true);
        layer_stats(u.pb, true, st);
      }
      const float *dyd = cur_d[u.dst()], *dys = cur_d[u.src()];
      // P_a: dx[dst] = P_a^T dy[dst]
      layer_bwd(u.pa, dyd, nullptr, 0, nullptr, nullptr, st);
      conv_wgrad(u.pa, xd, st);
      if (out_d[u.dst()]) conv_dgrad(u.pa, nullptr, out_d[u.dst()], st);
      // Phi_s: dx[src] = Phi_s^T dy[dst]
      branch_backward(u.phi, xs, dyd, nullptr, nullptr, nullptr, out_d[u.src()], st);
      // P_b: dx[src] += P_b^T dy[src]
      layer_bwd(u.pb, dys, nullptr, 0, nullptr, nullptr, st);
      conv_wgrad(u.pb, xs, st);
      if (out_d[u.src()]) conv_dgrad(u.pb, out_d[u.src()], out_d[u.src()], st);
      break;
    }
    case PETRA_UNIT_STEM: {
      Layer &L = u.phi[0];
      const float *th = theta_->as<float>();
      if (recompute) {
        conv_fwd(L, xin[0], st, src_ready, true);
        layer_stats(L, true, st);
        if (u.d.maxpool) {
          // recompute the pre-pool activation and argmax (outputs go to scratch)
          apply_bn(L.g.M(), L.g.Co, L.z()->p, L.z16, L.g.Co, 0, L.mean()->as<float>(),
                                 L.invstd()->as<float>(), th + L.g_off, th + L.b_off, 1, 1.f, nullptr,
                                 u.pool_a()->as<float>(), nullptr, st, 0, 0, take_fold(L));
          maxpool_fwd(u.pool_a()->as<float>(), L.g.B, L.g.Ho, L.g.Wo, L.g.Co, u.out.H, u.out.W, L.dz->as<float>(),
                      L.dz->as<float>() + u.out.numel(), u.pool_arg()->as<uint8_t>(), st);
        }
      }
      if (u.d.maxpool) {
        maxpool_bwd(cur_d[0], cur_d[1], u.pool_arg()->as<uint8_t>(), L.g.B, L.g.Ho, L.g.Wo, L.g.Co, u.out.H,
                    u.out.W, u.pool_a()->as<float>(), st);
        layer_bwd(L, u.pool_a()->as<float>(), nullptr, 0, nullptr, nullptr, st);
      } else {
        layer_bwd(L, cur_d[0], cur_d[1], L.g.Co / 2, nullptr, nullptr, st);
      }
      conv_wgrad(L, xin[0], st);  // no dgrad: the stem input is data
      break;
    }
    default:
      throw PetraError(PETRA_E_ARG, "unit_backward: bad kind");
  }
}

// ------------------------------------------------------------------ ticks
// Host bookkeeping (FIFO slots, id order, counters) is kept apart from the device
// enqueue functions, so that the device work of a tick can be captured once into a
// CUDA graph and replayed: its pointers depend only on the mailbox parity and the
// FIFO slots, both fixed per graph key.
static void copy_d2d(float *dst, const float *src, int64_t n, cudaStream_t st) {
  if (dst && src && dst != src) {
    ProfScope ps("copy", st, 0.0, 8.0 * (double)n);
    PETRA_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(float), cudaMemcpyDeviceToDevice, st));
  }
}

// reserve the FIFO slot a forward pushes its input into (reading c5)
static int fifo_reserve(Fifo &f, uint64_t mb) {
  if (f.size >= f.cap) throw PetraError(PETRA_E_ARG, "FIFO overflow: capacity below 2(J-j)+1");
  int slot = (f.head + f.size) % f.cap;
  f.ids.push_back(mb);
  ++f.size;
  f.peak = std::max(f.peak, f.size);
  return slot;
}

// the slot a backward pops (must be the FIFO head, Alg. 1 line 16)
static int fifo_take(Fifo &f, uint64_t mb) {
  if (f.size == 0) throw PetraError(PETRA_E_EMPTY_BUFFER, "non-reversible backward with an empty FIFO");
  if (f.ids.front() != mb)
    throw PetraError(PETRA_E_ORDER, "backward mb " + std::to_string(mb) + " != FIFO head " +
                                        std::to_string(f.ids.front()));
  int slot = f.head;
  f.head = (f.head + 1) % f.cap;
  --f.size;
  f.ids.pop_front();
  return slot;
}

std::vector<int> Stage::reserve_push(uint64_t mb) {
  std::vector<int> slots(units_.size(), -1);
  for (size_t i = 0; i < units_.size(); ++i)
    if (units_[i].d.kind == PETRA_UNIT_DS || units_[i].d.kind == PETRA_UNIT_STEM) slots[i] = fifo_reserve(units_[i].fifo, mb);
  return slots;
}

std::vector<int> Stage::take_pop(uint64_t mb) {
  std::vector<int> slots(units_.size(), -1);
  for (int i = (int)units_.size() - 1; i >= 0; --i)
    if (units_[i].d.kind == PETRA_UNIT_DS || units_[i].d.kind == PETRA_UNIT_STEM) slots[i] = fifo_take(units_[i].fifo, mb);
  return slots;
}

// Forward.  Targets: a unit that first writes a half writes into the
// stage output buffer if no non-reversible unit follows, else into its own buffer;
// later units work in place.  Caller inputs are never written.  keep = final stage
// (running stats updated in this single forward, reading c10; outputs stay in the
// stage's buffers for its own backward).
// comparison buffers of this forward (slot n_fwd_ of each ring): the received input and
// theta^t, as a delayed-gradient method with weight stashing would keep them
void Stage::enqueue_compare(const float *x1, const float *x2, cudaStream_t st) {
  if (eval_) return;
  if (!cmp_in_[0].empty()) {
    const size_t s = (size_t)(n_fwd_ % (int64_t)cmp_in_[0].size());
    copy_d2d(cmp_in_[0][s]->as<float>(), x1, in_.numel(), st);
    copy_d2d(cmp_in_[1][s]->as<float>(), x2, in_.numel(), st);
  }
  if (!cmp_stash_.empty()) {
    const size_t s = (size_t)(n_fwd_ % (int64_t)cmp_stash_.size());
    copy_d2d(cmp_stash_[s]->as<float>(), theta_->as<float>(), (int64_t)(theta_->bytes / sizeof(float)), st);
  }
}

void Stage::enqueue_forward(const float *x1, const float *x2, float *o1, float *o2, const std::vector<int> &push,
                            bool keep, const float **fin, cudaStream_t st) {
  enqueue_compare(x1, x2, st);
  const float *cur[2] = {x1, x2};
  bool ro[2] = {true, true};
  float *outs[2] = {o1, o2};
  const int n = (int)units_.size() - (is_last_ ? 1 : 0);
  bool ready = false;  // bf16 operand of this unit's src already written by its producer
  static const bool in_place_push = env_int("PETRA_PUSH_IN_PLACE", 1) != 0;
  for (int i = 0; i < n; ++i) {
    Unit &u = units_[i];
    float *tgt[2];
    for (int h = 0; h < 2; ++h) tgt[h] = u.fout[h] ? u.fout[h]->as<float>() : outs[h];
    // the units before a DS unit write its input straight into the DS's FIFO slot of this
    // micro-batch (the slot the DS forward would copy it into: the copy becomes a no-op)
    int nx = i + 1;
    while (nx < n && units_[nx].d.kind == PETRA_UNIT_REV) ++nx;
    if (in_place_push && nx < n && units_[nx].d.kind == PETRA_UNIT_DS && push[nx] >= 0) {
      tgt[0] = units_[nx].fifo.slot0[push[nx]]->as<float>();
      tgt[1] = units_[nx].fifo.slot1[push[nx]]->as<float>();
    }
    if (u.d.kind == PETRA_UNIT_REV) {
      float *o[2] = {nullptr, nullptr};
      int d = u.dst();
      o[d] = ro[d] ? tgt[d] : const_cast<float *>(cur[d]);
      Bf16Out ob = (i + 1 < n && units_[i + 1].d.kind == PETRA_UNIT_REV && units_[i + 1].src() == d)
                       ? src_operand(units_[i + 1]) : Bf16Out{};
      unit_forward(u, cur, o, keep, st, ob, ready);
      ready = ob.p != nullptr;
      cur[d] = o[d];
      ro[d] = false;
    } else {
      ready = false;
      int slot = push[i];
      if (!eval_ && !u.fifo.slot0.empty()) {  // an evaluation forward keeps nothing for a backward
        copy_d2d(u.fifo.slot0[slot]->as<float>(), cur[0], u.in.numel(), st);
        if (u.d.kind == PETRA_UNIT_DS) copy_d2d(u.fifo.slot1[slot]->as<float>(), cur[1], u.in.numel(), st);
      }
      // a DS unit writes the bf16 operand of the next reversible unit's src half too
      Bf16Out ob = (u.d.kind == PETRA_UNIT_DS && i + 1 < n && units_[i + 1].d.kind == PETRA_UNIT_REV)
                       ? src_operand(units_[i + 1]) : Bf16Out{};
      const int obh = ob.p ? units_[i + 1].src() : -1;
      bind_fifo_operands(u, slot);
      unit_forward(u, cur, tgt, keep, st, ob, false, obh);
      ready = ob.p != nullptr;
      cur[0] = tgt[0];
      cur[1] = tgt[1];
      ro[0] = ro[1] = false;
    }
  }
  flush_fold(st);
  if (fin) {
    fin[0] = cur[0];
    fin[1] = cur[1];
    return;
  }
  for (int h = 0; h < 2; ++h)
    if (cur[h] != outs[h]) copy_d2d(outs[h], cur[h], out_.numel(), st);
}

// Backward walk over units (reverse order): reversible units reconstruct their
// input with the current theta and run the VJP; non-reversible
// units recompute from their FIFO slot (Alg. 1 lines 16-17).  recompute = false
// in the final stage (plain backprop through the graph kept by its forward).
void Stage::enqueue_backward_walk(int last_unit, bool recompute, const float *cx[2], const float *cd[2],
                                  bool rox[2], bool rod[2], float *ox[2], float *od[2], const std::vector<int> &pop,
                                  cudaStream_t st) {
  bool ready = false;  // bf16 operand of this unit's src written by the previous reconstruction
  for (int i = last_unit; i >= 0; --i) {
    Unit &u = units_[i];
    if (u.d.kind == PETRA_UNIT_REV) {
      int d = u.dst(), s = u.src();
      float *tx[2] = {nullptr, nullptr}, *td[2] = {nullptr, nullptr};
      tx[d] = rox[d] ? (u.bx[d] ? u.bx[d]->as<float>() : ox[d]) : const_cast<float *>(cx[d]);
      td[s] = rod[s] ? (u.bd[s] ? u.bd[s]->as<float>() : od[s]) : const_cast<float *>(cd[s]);
      if (!tx[d] || !td[s])
        throw PetraError(PETRA_E_ARG, "NULL backward output for reversible unit " + std::to_string(i) + " of " +
                                          std::to_string(units_.size()) + (is_last_ ? " (final stage)" : "") +
                                          (tx[d] ? "" : ": no x~ target") + (td[s] ? "" : ": no delta target"));
      const float *nox[2] = {nullptr, nullptr};
      // the reconstructed dst half is the src of the unit processed next (recomputed
      // from it): its bf16 operand comes out of the reconstruction kernel
      Bf16Out ob = (recompute && i > 0 && units_[i - 1].d.kind == PETRA_UNIT_REV && units_[i - 1].src() == d)
                       ? src_operand(units_[i - 1]) : Bf16Out{};
      unit_backward(u, recompute, nox, cx, tx, cd, td, st, ob, ready && recompute);
      early_update(i, st);
      ready = ob.p != nullptr;
      cx[d] = tx[d];
      rox[d] = false;
      cd[s] = td[s];
      rod[s] = false;
    } else {
      ready = false;
      int slot = pop[i];
      const float *xin[2] = {u.fifo.slot0.empty() ? nullptr : u.fifo.slot0[slot]->as<float>(),
                             u.d.kind == PETRA_UNIT_DS ? u.fifo.slot1[slot]->as<float>() : nullptr};
      float *td[2] = {nullptr, nullptr};
      if (u.d.kind == PETRA_UNIT_DS)
        for (int h = 0; h < 2; ++h) td[h] = u.bd[h] ? u.bd[h]->as<float>() : od[h];
      bind_fifo_operands(u, slot);  // the forward converted this micro-batch's input into the slot
      unit_backward(u, recompute, xin, cx, nullptr, cd, td, st, Bf16Out{}, !u.fifo.bslot0.empty());
      early_update(i, st);
      cx[0] = xin[0];
      cx[1] = xin[1];
      rox[0] = rox[1] = true;  // FIFO memory: copied out at the end, never written
      cd[0] = td[0];
      cd[1] = td[1];
      rod[0] = rod[1] = false;
    }
  }
}

void Stage::enqueue_backward(const float *xt1, const float *xt2, const float *d1, const float *d2, float *oxt1,
                             float *oxt2, float *od1, float *od2, const std::vector<int> &pop, cudaStream_t st) {
  const float *cx[2] = {xt1, xt2}, *cd[2] = {d1, d2};
  bool rox[2] = {true, true}, rod[2] = {true, true};
  float *ox[2] = {oxt1, oxt2}, *od[2] = {od1, od2};
  enqueue_backward_walk((int)units_.size() - 1, true, cx, cd, rox, rod, ox, od, pop, st);
  flush_fold(st);
  join_wgrads(st);
  if (!stem_first())
    for (int h = 0; h < 2; ++h) {
      if (ox[h]) copy_d2d(ox[h], cx[h], in_.numel(), st);
      if (od[h]) copy_d2d(od[h], cd[h], in_.numel(), st);
    }
}

// Final stage (Alg. 1 lines 26-35): forward keeping the graph, loss, backprop, and
// the received input returned unchanged with delta_J wrt it (reading c7).
void Stage::enqueue_tail(const float *x1, const float *x2, const int32_t *labels, float *oxt1, float *oxt2,
                         float *od1, float *od2, float *loss, const std::vector<int> &push,
                         const std::vector<int> &pop, cudaStream_t st) {
  const float *cur[2];
  enqueue_forward(x1, x2, nullptr, nullptr, push, true, cur, st);
  Unit &t = units_.back();
  const float *th = theta_->as<float>();
  float *gr = grad_->as<float>();
  {
    ProfScope pst("tail_loss", st, 6.0 * desc_.batch * 2.0 * t.in.C * t.d.classes, 12.0 * (double)t.in.numel());
    tail_forward_backward(cur[0], cur[1], desc_.batch, t.in.H * t.in.W, t.in.C, th + t.fc_w, th + t.fc_b,
                          t.d.classes, labels, feat_->as<float>(), logits_->as<float>(), dlogits_->as<float>(),
                          lossrow_->as<float>(), dfeat_->as<float>(), gr + t.fc_w, gr + t.fc_b,
                          tail_d_[0]->as<float>(), tail_d_[1]->as<float>(), loss, nonfinite_->as<int>(),
                          fc_ws_->as<float>(), fc_ws_floats_, st);
  }
  // the stage's own forward buffers and gradient buffers are written in place
  const float *cx[2] = {cur[0], cur[1]}, *cd[2] = {tail_d_[0]->as<float>(), tail_d_[1]->as<float>()};
  bool rox[2] = {false, false}, rod[2] = {false, false};
  float *ox[2] = {nullptr, nullptr}, *od[2] = {nullptr, nullptr};
  enqueue_backward_walk((int)units_.size() - 2, false, cx, cd, rox, rod, ox, od, pop, st);
  join_wgrads(st);
  if (!stem_first()) {
    copy_d2d(oxt1, x1, in_.numel(), st);
    copy_d2d(oxt2, x2, in_.numel(), st);
    copy_d2d(od1, cd[0], in_.numel(), st);
    copy_d2d(od2, cd[1], in_.numel(), st);
  }
}

// ---- evaluation (the running statistics of batch normalisation "are then
// used during model evaluation"): the forward of every unit with BN on the running
// statistics; nothing is pushed, updated or counted.  Non-reversible units stage their
// bf16 operand in the next free FIFO slot (peeked, not reserved).
std::vector<int> Stage::peek_push() const {
  std::vector<int> slots(units_.size(), -1);
  for (size_t i = 0; i < units_.size(); ++i) {
    const Fifo &f = units_[i].fifo;
    if (units_[i].d.kind == PETRA_UNIT_DS || units_[i].d.kind == PETRA_UNIT_STEM) {
      if (f.size >= f.cap) throw PetraError(PETRA_E_ARG, "evaluation needs a free FIFO slot (drain the pipeline)");
      slots[i] = (f.head + f.size) % f.cap;
    }
  }
  return slots;
}

void Stage::eval(const float *x1, const float *x2, float *o1, float *o2, cudaStream_t st) {
  NvtxRange nr("stage eval");
  if (is_last_) throw PetraError(PETRA_E_ARG, "the final stage runs petra_stage_eval_tail");
  if (!x1 || (!stem_first() && !x2) || !o1 || !o2) throw PetraError(PETRA_E_ARG, "NULL activation pointer");
  std::vector<int> push = peek_push();
  ctx_ = 0;
  eval_ = true;
  try {
    enqueue_forward(x1, x2, o1, o2, push, false, nullptr, st);
  } catch (...) {
    eval_ = false;
    throw;
  }
  eval_ = false;
}

void Stage::eval_tail(const float *x1, const float *x2, const int32_t *labels, int *correct, float *loss,
                      cudaStream_t st) {
  NvtxRange nr("stage eval tail");
  if (!is_last_) throw PetraError(PETRA_E_ARG, "petra_stage_eval_tail on a stage without a tail unit");
  if (!x1 || (!stem_first() && !x2) || !labels || !correct || !loss) throw PetraError(PETRA_E_ARG, "NULL argument");
  std::vector<int> push = peek_push();
  ctx_ = 0;
  eval_ = true;
  try {
    const float *cur[2];
    enqueue_forward(x1, x2, nullptr, nullptr, push, false, cur, st);
    Unit &t = units_.back();
    const float *th = theta_->as<float>();
    tail_forward_backward(cur[0], cur[1], desc_.batch, t.in.H * t.in.W, t.in.C, th + t.fc_w, th + t.fc_b,
                          t.d.classes, labels, feat_->as<float>(), logits_->as<float>(), dlogits_->as<float>(),
                          lossrow_->as<float>(), nullptr, nullptr, nullptr, nullptr, nullptr, loss,
                          evalflag_->as<int>(), fc_ws_->as<float>(), fc_ws_floats_, st, correct);
  } catch (...) {
    eval_ = false;
    throw;
  }
  eval_ = false;
}

// ---- public entry points (standalone stages: direct enqueue)
void Stage::check_fwd(uint64_t mb, const float *x1, const float *x2) {
  if (!x1 || (!stem_first() && !x2)) throw PetraError(PETRA_E_ARG, "NULL activation pointer");
  if (have_last_fwd_ && mb <= last_fwd_mb_) throw PetraError(PETRA_E_ORDER, "forward mb ids must increase");
}

static void check_lr(float lr) {
  if (!std::isfinite(lr) || lr < 0.f) throw PetraError(PETRA_E_ARG, "lr must be finite and >= 0");
}

void Stage::forward(uint64_t mb, const float *x1, const float *x2, float *o1, float *o2, cudaStream_t st) {
  NvtxRange nr("stage forward mb %llu", (unsigned long long)mb);
  if (is_last_) throw PetraError(PETRA_E_ARG, "the final stage runs petra_stage_tail");
  check_fwd(mb, x1, x2);
  if (!o1 || !o2) throw PetraError(PETRA_E_ARG, "NULL output pointer");
  std::vector<int> push = reserve_push(mb);
  ctx_ = 0;
  enqueue_forward(x1, x2, o1, o2, push, false, nullptr, st);
  have_last_fwd_ = true;
  last_fwd_mb_ = mb;
  ++n_fwd_;
  last_stream_ = st;
}

void Stage::backward(uint64_t mb, const float *xt1, const float *xt2, const float *d1, const float *d2,
                     float *oxt1, float *oxt2, float *od1, float *od2, float lr, cudaStream_t st) {
  NvtxRange nr("stage backward mb %llu", (unsigned long long)mb);
  if (is_last_) throw PetraError(PETRA_E_ARG, "the final stage runs petra_stage_tail");
  if (!xt1 || !xt2 || !d1 || !d2) throw PetraError(PETRA_E_ARG, "NULL backward input");
  check_lr(lr);
  std::vector<int> pop = take_pop(mb);
  upload_lr(lr, st);
  ctx_ = 1;
  enqueue_backward(xt1, xt2, d1, d2, oxt1, oxt2, od1, od2, pop, st);
  ctx_ = 0;
  const int mode = next_update_mode();
  enqueue_update(mode, st);
  advance_step(mode);
  ++n_bwd_;
  last_stream_ = st;
}

void Stage::tail(uint64_t mb, const float *x1, const float *x2, const int32_t *labels, float lr, float *oxt1,
                 float *oxt2, float *od1, float *od2, float *loss, cudaStream_t st) {
  NvtxRange nr("stage tail mb %llu", (unsigned long long)mb);
  if (!is_last_) throw PetraError(PETRA_E_ARG, "petra_stage_tail on a stage without a tail unit");
  if (!labels) throw PetraError(PETRA_E_ARG, "NULL labels");
  check_fwd(mb, x1, x2);
  check_lr(lr);
  std::vector<int> push = reserve_push(mb), pop = take_pop(mb);
  upload_lr(lr, st);
  ctx_ = 0;
  enqueue_tail(x1, x2, labels, oxt1, oxt2, od1, od2, loss, push, pop, st);
  const int mode = next_update_mode();
  enqueue_update(mode, st);
  advance_step(mode);
  have_last_fwd_ = true;
  last_fwd_mb_ = mb;
  ++n_fwd_;
  ++n_bwd_;
  last_stream_ = st;
}

// ---- pipeline entry point: forward and/or backward (or the tail step) of one
// tick, replayed from a cached CUDA graph when graphs are enabled.
void Stage::tick(const TickArgs &a, float lr, cudaStream_t st, bool use_graph) {
  const bool fwd = a.fwd, bwd = a.bwd;
  if (is_last_ && fwd != bwd) throw PetraError(PETRA_E_ARG, "the final stage runs forward and backward together");
  std::vector<int> push, pop;
  if (fwd) {
    check_fwd(a.fmb, a.x1, a.x2);
    if (is_last_ && !a.labels) throw PetraError(PETRA_E_ARG, "NULL labels");
    push = reserve_push(a.fmb);
  }
  if (bwd) {
    check_lr(lr);
    pop = take_pop(is_last_ ? a.fmb : a.bmb);
  }
  if (!fwd && !bwd) return;
  if (bwd) upload_lr(lr, st);
  const int mode = bwd ? next_update_mode() : SGD_PLAIN;
  bool capturing = false;
  // external synchronisation points (TickArgs::wait_* / done_*): plain event waits and
  // records when enqueued directly, external event nodes when captured into the graph
  auto wait_on = [&](cudaStream_t s, const cudaEvent_t (&evs)[2]) {
    for (cudaEvent_t e : evs)
      if (e) PETRA_CUDA(cudaStreamWaitEvent(s, e, capturing ? cudaEventWaitExternal : cudaEventWaitDefault));
  };
  auto record = [&](cudaEvent_t e, cudaStream_t s) {
    if (e) PETRA_CUDA(cudaEventRecordWithFlags(e, s, capturing ? cudaEventRecordExternal : cudaEventRecordDefault));
  };
  // bf16 wire format: round the messages of this tick before they are declared final
  auto round_fwd = [&](cudaStream_t s) {
    if (!a.round_msgs) return;
    for (int h = 0; h < 2; ++h)
      if (a.o[h]) round_bf16_inplace(a.o[h], out_.numel(), s);
  };
  auto round_bwd = [&](cudaStream_t s) {
    if (!a.round_msgs || stem_first()) return;
    for (int h = 0; h < 2; ++h) {
      if (a.oxt[h]) round_bf16_inplace(a.oxt[h], in_.numel(), s);
      if (a.od[h]) round_bf16_inplace(a.od[h], in_.numel(), s);
    }
  };
  static const bool early_env = env_int("PETRA_EARLY_UPDATE", 1) != 0;
  auto enqueue = [&](cudaStream_t s) {
    // early per-unit updates: on the wgrad stream, in a direct or captured (not profiled) tick
    eu_.active = bwd && early_env && early_ok_ && wg_ && !Prof::enabled;
    eu_.mode = mode;
    eu_.fwd_pending = false;
    eu_.done.assign(units_.size(), 0);
    if (is_last_) {
      ctx_ = 0;
      wait_on(s, a.wait_f);
      wait_on(s, a.wait_b);
      enqueue_tail(a.x1, a.x2, a.labels, a.oxt[0], a.oxt[1], a.od[0], a.od[1], a.loss, push, pop, s);
      round_bwd(s);
      record(a.done_f, s);
      record(a.done_b, s);
    } else if (fwd && bwd && !Prof::enabled) {
      // forward (theta^t, context 0) and backward (context 1) of different micro-batches
      // are independent until the update: run them on two streams, join, then update
      // (a profiled replay serialises them so that each kernel's events time it alone)
      PETRA_CUDA(cudaEventRecord(fork_, s));
      PETRA_CUDA(cudaStreamWaitEvent(side_, fork_, 0));
      ctx_ = 0;
      wait_on(s, a.wait_f);
      enqueue_forward(a.x1, a.x2, a.o[0], a.o[1], push, false, nullptr, s);
      round_fwd(s);
      record(a.done_f, s);
      if (eu_.active) {  // the early updates wait for this forward's reads of theta^t
        PETRA_CUDA(cudaEventRecord(fwd_done_, s));
        eu_.fwd_pending = true;
      }
      ctx_ = 1;
      wait_on(side_, a.wait_b);
      enqueue_backward(a.xt[0], a.xt[1], a.d[0], a.d[1], a.oxt[0], a.oxt[1], a.od[0], a.od[1], pop, side_);
      round_bwd(side_);
      record(a.done_b, side_);
      PETRA_CUDA(cudaEventRecord(join_, side_));
      PETRA_CUDA(cudaStreamWaitEvent(s, join_, 0));
      ctx_ = 0;
    } else {
      if (fwd) {
        ctx_ = 0;
        wait_on(s, a.wait_f);
        enqueue_forward(a.x1, a.x2, a.o[0], a.o[1], push, false, nullptr, s);
        round_fwd(s);
        record(a.done_f, s);
      }
      if (bwd) {
        ctx_ = 1;
        wait_on(s, a.wait_b);
        enqueue_backward(a.xt[0], a.xt[1], a.d[0], a.d[1], a.oxt[0], a.oxt[1], a.od[0], a.od[1], pop, s);
        round_bwd(s);
        record(a.done_b, s);
      }
      ctx_ = 0;
    }
    if (bwd) enqueue_update_rest(mode, s);
  };
  if (!use_graph) {
    enqueue(st);
  } else if (Prof::enabled) {
    // profiled replay: this tick as a one-off graph (its kernels and the ProfScope event
    // nodes), so each kernel's event pair brackets device work only, not the host's tensor-map
    // encoding and launch calls (a kernel shorter than its host enqueue would otherwise be
    // timed at the host's pace)
    cudaGraph_t g = nullptr;
    PETRA_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
    capturing = true;
    try {
      enqueue(st);
      capturing = false;
    } catch (...) {
      capturing = false;
      cudaStreamEndCapture(st, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    PETRA_CUDA(cudaStreamEndCapture(st, &g));
    cudaGraphExec_t ex = nullptr;
    cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    PETRA_CUDA(e);
    PETRA_CUDA(cudaGraphLaunch(ex, st));
    prof_execs_.push_back(ex);  // released by the destructor (after its device sync)
  } else {
    std::vector<uintptr_t> key = {(uintptr_t)fwd, (uintptr_t)bwd, (uintptr_t)mode, (uintptr_t)a.round_msgs};
    for (const void *p : {(const void *)a.x1, (const void *)a.x2, (const void *)a.labels, (const void *)a.o[0],
                          (const void *)a.o[1], (const void *)a.xt[0], (const void *)a.xt[1], (const void *)a.d[0],
                          (const void *)a.d[1], (const void *)a.oxt[0], (const void *)a.oxt[1],
                          (const void *)a.od[0], (const void *)a.od[1], (const void *)a.loss,
                          (const void *)a.wait_f[0], (const void *)a.wait_f[1], (const void *)a.wait_b[0],
                          (const void *)a.wait_b[1], (const void *)a.done_f, (const void *)a.done_b})
      key.push_back((uintptr_t)p);
    for (int v : push) key.push_back((uintptr_t)(v + 1));
    if (fwd && !cmp_in_[0].empty()) key.push_back((uintptr_t)(n_fwd_ % (int64_t)cmp_in_[0].size()) + 1);
    if (fwd && !cmp_stash_.empty()) key.push_back((uintptr_t)(n_fwd_ % (int64_t)cmp_stash_.size()) + 1);
    for (int v : pop) key.push_back((uintptr_t)(v + 1));
    auto it = graphs_.find(key);
    if (it == graphs_.end()) {
      const int64_t n0 = Prof::launches.load();
      cudaGraph_t g = nullptr;
      PETRA_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
      capturing = true;
      try {
        enqueue(st);
        capturing = false;
      } catch (...) {
        capturing = false;
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      PETRA_CUDA(cudaStreamEndCapture(st, &g));
      CachedGraph cg;
      cudaError_t e = cudaGraphInstantiate(&cg.exec, g, 0);
      cudaGraphDestroy(g);
      PETRA_CUDA(e);
      cg.kernels = Prof::launches.load() - n0;
      Prof::launches.fetch_sub(cg.kernels);  // counted when the graph is launched
      it = graphs_.emplace(std::move(key), cg).first;
    }
    PETRA_CUDA(cudaGraphLaunch(it->second.exec, st));
    count_launch((int)it->second.kernels);
  }
  if (fwd) {
    have_last_fwd_ = true;
    last_fwd_mb_ = a.fmb;
    ++n_fwd_;
  }
  if (bwd) {
    advance_step(mode);
    ++n_bwd_;
  }
  last_stream_ = st;
}

}  // namespace petra

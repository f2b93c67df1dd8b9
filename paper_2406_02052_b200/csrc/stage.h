// stage.h -- one PETRA stage on one GPU: parameters, FIFOs, workspace and the
// per-tick kernel sequence (Alg. 1).  Internal C++ API.
#pragma once
#include <deque>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/petra.h"
#include "kernels.h"

namespace petra {

// device allocator installed with petra_set_allocator (alloc == null: cudaMalloc)
struct Allocator {
  void *(*alloc)(size_t, int, void *) = nullptr;
  void (*release)(void *, int, void *) = nullptr;
  void *ctx = nullptr;
};
Allocator &allocator();

// device allocation owned by a stage
struct DevBuf {
  void *p = nullptr;
  size_t bytes = 0;
  void (*release)(void *, int, void *) = nullptr;  // the allocator that made it (null: cudaFree)
  void *ctx = nullptr;
  int device = 0;
  DevBuf() = default;
  explicit DevBuf(size_t n);
  ~DevBuf();
  DevBuf(const DevBuf &) = delete;
  DevBuf &operator=(const DevBuf &) = delete;
  template <typename T> T *as() const { return reinterpret_cast<T *>(p); }
};
using DevPtr = std::unique_ptr<DevBuf>;
DevPtr dalloc(size_t bytes);

struct Shape {
  int B = 0, H = 0, W = 0, C = 0;  // per half (or image)
  int64_t numel() const { return (int64_t)B * H * W * C; }
  bool operator==(const Shape &o) const { return B == o.B && H == o.H && W == o.W && C == o.C; }
  bool operator!=(const Shape &o) const { return !(*this == o); }
};

struct Layer {               // conv(no bias) -> BN(train) [-> ReLU]
  ConvGeom g;
  bool relu = true;
  int64_t w_off = 0, g_off = 0, b_off = 0;   // into theta / grad / v
  int64_t rm_off = 0, rv_off = 0;            // into buffers (running stats)
  // Per-context workspace: context 0 = forward, 1 = backward (recompute + VJP).  The
  // forward and the backward of a pipeline tick run concurrently on two streams, so
  // everything either writes has one copy per context; *ctx selects the live one.
  DevPtr z_[2], a_[2], mean_[2], invstd_[2], xb_[2];
  StatsRows stats_rows_[2];                  // rows > 0: BN partials written by the conv epilogue
  const int *ctx = nullptr;
  DevPtr &z() { return z_[*ctx]; }
  DevPtr &a() { return a_[*ctx]; }
  DevPtr &mean() { return mean_[*ctx]; }
  DevPtr &invstd() { return invstd_[*ctx]; }
  Layer *operand_of = nullptr;               // shares that layer's bf16 input operand (same input tensor)
  bool fifo_backed = false;                  // its bf16 operand lives in the unit's FIFO slot (DS / stem)
  __nv_bfloat16 *xb_ext = nullptr;           // ... bound to the slot of the tick being enqueued
  DevPtr &xb() { return operand_of ? operand_of->xb() : xb_[*ctx]; }
  __nv_bfloat16 *xbp() {
    if (operand_of) return operand_of->xbp();
    return fifo_backed ? xb_ext : xb_[*ctx]->as<__nv_bfloat16>();
  }
  StatsRows &stats_rows() { return stats_rows_[*ctx]; }
  StatsFold fold_[2];                        // part != null: statistics left for the consuming BN pass
  StatsFold &fold() { return fold_[*ctx]; }
  DevPtr dz, da, dzb;                        // backward-only workspace
  DevPtr w_bf16, wt_bf16;                    // bf16 shadows of the live weights
  bool z16 = false;                          // z stored in bf16 (tensor-core conv output, reading c24)
  bool is_stem = false;                      // no dgrad: the input is data
  bool xpad = false, dzpad = false;          // xb / dzb zero-bordered [B][H+2][W+2][C] (3x3 stride-1 layers)
  int64_t M() const { return g.M(); }
};

struct Fifo {                // input buffer of a non-reversible unit (reading c5)
  int cap = 0, head = 0, size = 0;
  std::vector<DevPtr> slot0, slot1;   // one tensor (stem) or two halves (DS)
  std::vector<DevPtr> bslot0, bslot1; // their bf16 conv operands (tensor-core path): converted once
                                      // in the forward, read again by the backward's recomputation
  std::deque<uint64_t> ids;
  int peak = 0;
};

struct Unit {
  petra_unit d;
  Shape in, out;                       // per-half shapes (stem: in = image)
  std::vector<Layer> phi;              // REV/DS branch; STEM: phi[0] is the stem conv
  Layer pa, pb;                        // DS projections
  int64_t fc_w = 0, fc_b = 0;          // TAIL offsets
  Fifo fifo;
  DevPtr pool_arg_[2], pool_a_[2];     // STEM max-pool argmax / pre-pool activation (per context)
  const int *ctx = nullptr;
  DevPtr &pool_arg() { return pool_arg_[*ctx]; }
  DevPtr &pool_a() { return pool_a_[*ctx]; }
  // forward / backward output targets (planned at creation): buffer per half
  DevPtr fout[2], bx[2], bd[2];
  int dst() const { return d.dst_half; }
  int src() const { return 1 - d.dst_half; }
};

// bf16 copy of a stream half written by the kernel that produces it: the
// tensor-core operand of the next unit's first convolution (pH > 0: zero-bordered
// H x W layout of the halo kernel)
struct Bf16Out {
  __nv_bfloat16 *p = nullptr;
  int pH = 0, pW = 0;
};

// one tick of a stage for the pipeline: forward (fmb) and/or backward (bmb)
struct TickArgs {
  bool fwd = false, bwd = false;
  uint64_t fmb = 0, bmb = 0;
  const float *x1 = nullptr, *x2 = nullptr;  // forward input (tail: its input)
  const int32_t *labels = nullptr;           // tail only
  float *o[2] = {nullptr, nullptr};          // forward output
  const float *xt[2] = {nullptr, nullptr};   // backward input x~_j
  const float *d[2] = {nullptr, nullptr};    // backward input delta_{j+1}
  float *oxt[2] = {nullptr, nullptr};        // backward output x~_{j-1}
  float *od[2] = {nullptr, nullptr};         // backward output delta_j
  float *loss = nullptr;                     // tail only
  // cross-rank synchronisation set by the pipeline's transport: the forward (backward)
  // part waits on wait_f (wait_b) -- a received message, a send buffer released -- and
  // records done_f (done_b) when its messages are final.  Inside the stage's CUDA graph
  // they are external event nodes (cudaEventWaitExternal / cudaEventRecordExternal).
  cudaEvent_t wait_f[2] = {nullptr, nullptr}, wait_b[2] = {nullptr, nullptr};
  cudaEvent_t done_f = nullptr, done_b = nullptr;
  // bf16 wire format (petra_pipeline_desc.wire): the messages this tick produces (forward
  // outputs, backward x~ and delta) are rounded to bf16 in place before done_f / done_b
  bool round_msgs = false;
};

struct CachedGraph {
  cudaGraphExec_t exec = nullptr;
  int64_t kernels = 0;
};

class Stage {
 public:
  Stage(const petra_stage_desc &desc, uint64_t seed);
  ~Stage();

  const Shape &in_shape() const { return in_; }
  const Shape &out_shape() const { return out_; }
  bool is_last() const { return is_last_; }
  bool stem_first() const { return units_.front().d.kind == PETRA_UNIT_STEM; }
  size_t n_params() const { return (size_t)n_params_; }
  size_t n_buffers() const { return (size_t)n_buffers_; }
  const std::vector<petra_tensor_info> &tensors() const { return tensors_; }
  int64_t version() const { return version_; }
  int fifo_depth() const;
  void memory(petra_memory_report *r) const;
  int classes() const { return units_.back().d.classes; }

  void forward(uint64_t mb, const float *x1, const float *x2, float *o1, float *o2, cudaStream_t st);
  void backward(uint64_t mb, const float *xt1, const float *xt2, const float *d1, const float *d2, float *oxt1,
                float *oxt2, float *od1, float *od2, float lr, cudaStream_t st);
  // evaluation forward (BN on the running statistics, no FIFO push, no state change)
  void eval(const float *x1, const float *x2, float *o1, float *o2, cudaStream_t st);
  void eval_tail(const float *x1, const float *x2, const int32_t *labels, int *correct, float *loss, cudaStream_t st);
  void tail(uint64_t mb, const float *x1, const float *x2, const int32_t *labels, float lr, float *oxt1,
            float *oxt2, float *od1, float *od2, float *loss, cudaStream_t st);
  void tick(const TickArgs &a, float lr, cudaStream_t st, bool use_graph);

  void get_params(float *theta, float *v, float *bufs);
  void set_params(const float *theta, const float *v, const float *bufs);
  void get_grads(float *delta);
  int nonfinite();  // latched device flags: bit 0 loss, bit 1 Delta (NaN / Inf)
  cudaStream_t last_stream() const { return last_stream_; }

 private:
  petra_stage_desc desc_;
  std::vector<Unit> units_;
  Shape in_, out_;
  bool is_last_ = false;
  bool tc_ = false;
  size_t alloc_bytes_ = 0;   // every DevBuf created while this stage was being built
  int64_t n_params_ = 0, n_buffers_ = 0;
  std::vector<petra_tensor_info> tensors_;
  DevPtr theta_, v_, grad_, bufs_, acc_;     // acc_: Delta_j of Alg. 1 (k > 1 only)
  std::vector<SgdSeg> segs_;
  DevPtr segs_dev_;
  int64_t max_seg_ = 0;
  DevPtr chunks_dev_;   // SgdChunk work items of the update (sgd_chunks)
  int n_chunks_ = 0;
  // early per-unit updates (PETRA_EARLY_UPDATE): unit u's work items are chunks
  // [unit_chunk_lo_[u], unit_chunk_hi_[u]); a unit's update runs on the wgrad stream as soon
  // as its backward (dgrad, BN-backward sums) and wgrads are done and this tick's forward has
  // read theta, instead of in the stage's one update launch at the end of the tick
  std::vector<int> unit_chunk_lo_, unit_chunk_hi_;
  bool early_ok_ = false;  // every unit's items contiguous
  struct EarlyUpd {
    bool active = false;
    int mode = 0;
    bool fwd_pending = false;  // the wgrad stream still has to wait for fwd_done_
    std::vector<char> done;    // per unit: updated early this tick
  } eu_;
  cudaEvent_t eu_b_ = nullptr, fwd_done_ = nullptr;
  void early_update(int unit, cudaStream_t st);
  void enqueue_update_rest(int mode, cudaStream_t st);  // the units not updated early
  DevPtr part_[2], spart_[2], wgrad_ws_[2], counters_[2];  // per context (see Layer)
  int ctx_ = 0;                                 // workspace context being enqueued
  DevPtr &part() { return part_[ctx_]; }
  DevPtr &spart() { return spart_[ctx_]; }   // BN partial rows of the conv epilogues
  Layer *pending_[2] = {nullptr, nullptr};    // layer whose statistics fold is not consumed yet
  void flush_fold(cudaStream_t st);           // launch the pending fold as stats_finalize
  const StatsFold *take_fold(Layer &L);       // the fold for L's consuming pass (cleared)
  StatsFold fold_tmp_[2];
  DevPtr &wgrad_ws() { return wgrad_ws_[ctx_]; }
  DevPtr &counters() { return counters_[ctx_]; }
  cudaStream_t side_ = nullptr;                 // the backward's stream (fork / join per tick)
  cudaEvent_t fork_ = nullptr, join_ = nullptr;
  // tensor-core wgrads on their own stream: a layer's dW is needed only by the update, so
  // the wgrad leaves the critical dz -> dgrad -> BN chain of the backward walk (joined
  // before the update); own split-K workspace
  cudaStream_t wg_ = nullptr;
  cudaEvent_t wg_fork_ = nullptr, wg_join_ = nullptr;
  DevPtr wg_ws_;
  bool wg_active_ = false;
  void join_wgrads(cudaStream_t st);
  DevPtr nonfinite_;
  DevPtr evalflag_;
  // tail workspace
  DevPtr feat_, logits_, dlogits_, lossrow_, dfeat_, tail_d_[2], fc_ws_;
  int64_t fc_ws_floats_ = 0;
  // bf16 shadows of stage-level stream halves (TC path)
  int64_t version_ = 0;                          // optimizer updates applied
  int64_t t_ = 1;                                // Alg. 1 step counter t (reading c12: starts at 1)
  int64_t n_fwd_ = 0, n_bwd_ = 0;
  bool eval_ = false;                          // enqueuing an evaluation forward
  std::vector<int> peek_push() const;          // FIFO slots an evaluation forward may use (not reserved)
  // Table 3 comparison buffers (petra_stage_desc.compare_buffers): a ring of stage inputs
  // (delayed-gradient input buffer) and a ring of theta copies (weight stash), one slot
  // written per forward
  std::vector<DevPtr> cmp_in_[2], cmp_stash_;
  void enqueue_compare(const float *x1, const float *x2, cudaStream_t st);
  bool have_last_fwd_ = false;
  uint64_t last_fwd_mb_ = 0;
  cudaStream_t last_stream_ = nullptr;

  void build();
  void alloc_layer(Layer &L, bool inner);
  int64_t add_tensor(int unit, int part, int kind, int decay, std::vector<int> shape, bool buffer);
  void init_params(uint64_t seed);
  static constexpr int kLrRing = 256;
  DevPtr lr_dev_;
  float *lr_host_ = nullptr;
  uint64_t lr_next_ = 0;
  std::map<std::vector<uintptr_t>, CachedGraph> graphs_;
  std::vector<cudaGraphExec_t> prof_execs_;  // one-off graphs of the profiled replay
  void upload_lr(float lr, cudaStream_t st);
  int next_update_mode() const;
  void advance_step(int mode);
  void enqueue_update(int mode, cudaStream_t st);
  std::vector<int> reserve_push(uint64_t mb);
  std::vector<int> take_pop(uint64_t mb);
  void check_fwd(uint64_t mb, const float *x1, const float *x2);
  void enqueue_forward(const float *x1, const float *x2, float *o1, float *o2, const std::vector<int> &push,
                       bool keep, const float **fin, cudaStream_t st);
  void enqueue_backward_walk(int last_unit, bool recompute, const float *cx[2], const float *cd[2], bool rox[2],
                             bool rod[2], float *ox[2], float *od[2], const std::vector<int> &pop, cudaStream_t st);
  void enqueue_backward(const float *xt1, const float *xt2, const float *d1, const float *d2, float *oxt1,
                        float *oxt2, float *od1, float *od2, const std::vector<int> &pop, cudaStream_t st);
  void enqueue_tail(const float *x1, const float *x2, const int32_t *labels, float *oxt1, float *oxt2, float *od1,
                    float *od2, float *loss, const std::vector<int> &push, const std::vector<int> &pop,
                    cudaStream_t st);

  // kernels of one layer / unit
  void conv_fwd(Layer &L, const float *x, cudaStream_t st, bool x_bf16_ready = false, bool running = false);
  void conv_wgrad(Layer &L, const float *x, cudaStream_t st);
  void conv_dgrad(Layer &L, const float *addend, float *out, cudaStream_t st);
  void layer_stats(Layer &L, bool running, cudaStream_t st);
  void branch_forward(std::vector<Layer> &phi, const float *x, bool running, cudaStream_t st, bool ready0 = false);
  void layer_bwd(Layer &L, const float *dy0, const float *dy1, int cs, const float *dst_in, float *dst_out,
                 cudaStream_t st, Bf16Out ob = {});
  void branch_backward(std::vector<Layer> &phi, const float *x, const float *dy, const float *dst_in,
                       float *dst_out, const float *addend, float *dx_out, cudaStream_t st, Bf16Out ob = {});
  Bf16Out src_operand(Unit &next);

  void unit_forward(Unit &u, const float *cur[2], float *out[2], bool keep, cudaStream_t st, Bf16Out ob = {},
                    bool src_ready = false, int ob_half = -1);
  void unit_backward(Unit &u, bool recompute, const float *xin[2], const float *cur_x[2], float *out_x[2],
                     const float *cur_d[2], float *out_d[2], cudaStream_t st, Bf16Out ob = {},
                     bool src_ready = false);
  void bind_fifo_operands(Unit &u, int slot);
};

}  // namespace petra

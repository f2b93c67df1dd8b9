/*
 * petra.h -- C ABI of the B200-native PETRA stage-tick library (libpetra.so).
 *
 * PETRA (arXiv 2406.02052) trains a reversible network split into J stages.
 * At every tick each stage independently (the equation system;
 * Alg. 1):
 *   1. runs its forward  x_j^{t+1} = F_j(x_{j-1}^t, theta_j^t)
 *   2. runs its backward on the message received from stage j+1:
 *        x~_{j-1}^{t+1} = F_j^{-1}(x~_j^t, theta_j^t)   approximate inversion
 *        delta_j^{t+1}  = d_x F_j(x~_{j-1}, theta^t)^T delta_{j+1}
 *        Delta_j^{t+1}  = d_theta F_j(x~_{j-1}, theta^t)^T delta_{j+1}
 *   3. updates theta immediately, no weight stash: theta^{t+1} = Opt(theta^t, Delta)
 *
 * Conventions (all entry points):
 *   - Every function returns petra_status; no C++ exception crosses the ABI.
 *     On error petra_last_error() returns a thread-local detail string.
 *   - Activations are fp32, NHWC, and travel as TWO channel halves {x^1, x^2}
 *     ("split equally into {x_j^1, x_j^2} along the channel
 *     dimension"): each half is a dense [B][H][W][C_half] array.  The input of a
 *     stage whose first unit is the stem is ONE image tensor [B][H][W][3] (x2 = NULL).
 *   - "dev" pointers are CUDA device pointers owned by the caller; "host"
 *     pointers are host memory owned by the caller.  The library owns
 *     everything it allocates (parameters, optimizer slots, FIFOs, workspace)
 *     and frees it in *_destroy.
 *   - Device work is enqueued asynchronously on the caller's stream
 *     (a cudaStream_t passed as void*; NULL = legacy default stream).  Shape and
 *     argument checks are synchronous and host-side.
 *   - A handle is used by one host thread at a time.
 *   - Parameter and gradient arrays are packed fp32 in the order reported by
 *     petra_stage_tensor_info(); conv weights are [C_out][k_h][k_w][C_in].
 *   - There is no CPU fallback: without a CUDA device every compute entry point
 *     returns PETRA_E_CUDA.
 */
#ifndef PETRA_H
#define PETRA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef enum {
  PETRA_OK = 0,
  PETRA_E_ARG = 1,          /* NULL handle/pointer, bad enum, k < 1, lr < 0 or non-finite      */
  PETRA_E_SHAPE = 2,        /* inconsistent shapes between units / stages                       */
  PETRA_E_ODD_CHANNELS = 3, /* a two-stream activation needs an even channel count */
  PETRA_E_EMPTY_BUFFER = 4, /* non-reversible backward with an empty FIFO: schedule bug          */
  PETRA_E_ORDER = 5,        /* backward mb id is not the FIFO head / ids not monotone            */
  PETRA_E_NONFINITE = 6,    /* NaN/Inf loss or Delta (latched device flag, reported by get_params) */
  PETRA_E_CUDA = 7,         /* CUDA runtime error or no device                                   */
  PETRA_E_NCCL = 8,         /* NCCL unavailable (libnccl.so.2 not loadable) or an NCCL call failed */
  PETRA_E_OOM = 9,          /* device allocation failed                                          */
  PETRA_E_UNSUPPORTED = 10  /* configuration not implemented                                     */
} petra_status;

const char *petra_status_str(int status);
const char *petra_last_error(void);
/* Library version string and the compile target ("sm_100a"). */
const char *petra_version(void);

/* Arithmetic of the convolutions.  Streams, BN, coupling add/sub, updates are fp32 in both. */
typedef enum {
  PETRA_FP32 = 0,    /* SIMT fp32 convolutions: parity path (rel 1e-4 vs the fp64 oracle)   */
  PETRA_BF16_TC = 1  /* tcgen05 bf16 x bf16 -> fp32 TMEM implicit GEMM (rel 2e-2 vs oracle) */
} petra_precision;

typedef enum {
  PETRA_UNIT_REV = 0,  /* reversible half-coupling  x[dst] += Phi(x[src])         */
  PETRA_UNIT_DS = 1,   /* downsampling: y[dst] = P_a(x[dst]) + Phi_s(x[src]); y[src] = P_b(x[src])  */
  PETRA_UNIT_STEM = 2, /* conv-BN-ReLU [+ max-pool 3x3/s2] of the image, split into two halves      */
  PETRA_UNIT_TAIL = 3  /* GAP(concat(x1,x2)) -> Linear(+bias) -> softmax cross-entropy (batch mean)  */
} petra_unit_kind;

/* One conv(no bias)-BN[-ReLU] layer; padding is (ksize-1)/2. */
typedef struct {
  int32_t cin, cout, ksize, stride;
} petra_conv;

typedef struct {
  int32_t kind;            /* petra_unit_kind                                                */
  int32_t dst_half;        /* REV/DS: 0 -> x1 is updated ("F"), 1 -> x2 is updated ("G")     */
  int32_t n_layers;        /* REV/DS: layers of Phi (1 basic, 3 bottleneck); STEM: 1         */
  petra_conv layer[3];     /* Phi layers (ReLU after each); STEM: the stem conv              */
  petra_conv proj[2];      /* DS only: P_a (on x[dst]) and P_b (on x[src]), conv1x1/s + BN  */
  int32_t maxpool;         /* STEM only: 1 = max-pool 3x3/s2/p1 after the ReLU               */
  int32_t classes;         /* TAIL only                                                      */
} petra_unit;

typedef struct {
  int32_t n_units;
  const petra_unit *units;
  int32_t batch, in_h, in_w, in_c; /* stage input: in_c = channels per half (or image channels) */
  int32_t precision;               /* petra_precision                                          */
  float momentum;                  /* 0.9                                       */
  float weight_decay;              /* 5e-4 CIFAR / 1e-4 ImageNet                */
  float bn_momentum;               /* 0.1 (reading c9)                                         */
  float bn_eps;                    /* 1e-5 (reading c9)                                        */
  int32_t nesterov;                /* 1                                         */
  int32_t accumulation_k;          /* k >= 1 (Alg. 1 lines 19-23): Delta_j +=
                                      Delta_mb / k every backward; Nesterov update with Delta_j and
                                      reset when t mod k == 0 (t counts backwards from 1)           */
  int32_t fifo_capacity;           /* non-reversible input FIFO depth; >= 2(J-j)+1 (Table 1)   */
  int32_t compare_buffers;         /* 0 for PETRA.  Table 3 comparison modes (PAPER.md:310-330,
                                      memory measurement only; the numerics stay PETRA's):
                                      bit 0 (PETRA_CMP_INPUTS): the stage also buffers the input
                                      of each of its fifo_capacity in-flight micro-batches, as a
                                      delayed-gradient method must (a device copy every forward;
                                      nothing extra when its first unit is non-reversible: its
                                      FIFO holds them already);
                                      bit 1 (PETRA_CMP_STASH): weight stashing -- fifo_capacity-1
                                      = 2(J-j) extra fp32 copies of theta, one written every
                                      forward (PipeDream)                                        */
} petra_stage_desc;
enum { PETRA_CMP_INPUTS = 1, PETRA_CMP_STASH = 2 };

typedef struct petra_stage petra_stage;

/* Device memory the library allocates (parameters, optimizer slots, FIFOs, workspace,
 * mailboxes) comes from cudaMalloc / cudaFree, or, once installed, from the caller's
 * allocator -- e.g. PyTorch's caching allocator, so a training process has one pool.
 * alloc(bytes, device, ctx) returns a device pointer on `device` (the current device
 * when the object is created) or NULL (-> PETRA_E_OOM); release(ptr, device, ctx) frees
 * it.  A buffer is released through the allocator that made it, so installing another
 * one (or NULL, NULL to return to cudaMalloc) affects only objects created afterwards.
 * Process-wide; call it while no other thread creates library objects.
 * Errors: PETRA_E_ARG (exactly one of alloc / release NULL). */
petra_status petra_set_allocator(void *(*alloc)(size_t bytes, int32_t device, void *ctx),
                                 void (*release)(void *ptr, int32_t device, void *ctx), void *ctx);

/* Create a stage on the current CUDA device.  Parameters are initialised from
 * `seed` (Kaiming-uniform conv/linear weights, gamma=1, beta=0, bias=0,
 * running mean 0 / var 1, momentum 0); callers that need identical values on
 * both sides of a parity test overwrite them with petra_stage_set_params().
 * Errors: PETRA_E_ARG, PETRA_E_SHAPE (unit shapes do not chain),
 * PETRA_E_ODD_CHANNELS, PETRA_E_UNSUPPORTED, PETRA_E_OOM, PETRA_E_CUDA. */
petra_status petra_stage_create(const petra_stage_desc *desc, uint64_t seed, petra_stage **out);
petra_status petra_stage_destroy(petra_stage *s);

/* Output activation shape of the stage (per half).  For a tail stage c = classes, h = w = 1. */
petra_status petra_stage_output_shape(const petra_stage *s, int32_t *b, int32_t *h, int32_t *w, int32_t *c);

/* Parameter layout.  n_params: length of theta (== v == Delta); n_buffers:
 * length of the BN running-statistics array. */
petra_status petra_stage_param_count(const petra_stage *s, size_t *n_params, size_t *n_buffers);

/* Device memory of a stage by category (Table 3 accounting, PAPER.md:310-330:
 * PETRA keeps one parameter version and buffers only the inputs of its
 * non-reversible units).  Bytes the library allocated for this stage:
 *   params     theta + BN running statistics (fp32)
 *   optimizer  v, Delta (last backward) and the Delta_j accumulator (k > 1)
 *   shadows    bf16 copies of the live conv weights (tensor-core operands; a copy of
 *              the single live version, rewritten by every update, not a stash)
 *   fifo       input FIFO slots of the non-reversible units (capacity 2(J-j)+1): the fp32
 *              input and, on the tensor-core path, its bf16 conv operands
 *   fifo_live  bytes of those slots holding an input right now
 *   workspace  everything else: per-layer conv outputs / BN statistics / operand
 *              copies of the tick, tail buffers
 *   cmp_inputs, cmp_stash  the comparison buffers of petra_stage_desc.compare_buffers
 *   total      sum of the above categories (fifo_live excluded)
 * Host-only, no synchronisation.  Errors: PETRA_E_ARG (NULL). */
typedef struct {
  uint64_t total, params, optimizer, shadows, fifo, fifo_live, workspace;
  uint64_t cmp_inputs, cmp_stash;  /* compare_buffers modes: the extra input ring / theta stash */
} petra_memory_report;
petra_status petra_stage_memory(const petra_stage *s, petra_memory_report *out);

typedef enum {
  PETRA_T_CONV_W = 0, PETRA_T_BN_GAMMA = 1, PETRA_T_BN_BETA = 2, PETRA_T_FC_W = 3, PETRA_T_FC_B = 4,
  PETRA_T_BN_RMEAN = 5, PETRA_T_BN_RVAR = 6
} petra_tensor_kind;

typedef struct {
  int32_t unit;        /* unit index within the stage                                      */
  int32_t part;        /* 0..2 = Phi layer, 3 = P_a, 4 = P_b, 0 for stem / tail             */
  int32_t kind;        /* petra_tensor_kind                                                */
  int32_t decay;       /* 1 if weight decay applies (not on BN params, biases) */
  int32_t ndim;
  int32_t shape[4];    /* conv: [cout, k, k, cin]; fc: [classes, cin]; vectors: [n]        */
  int64_t offset;      /* element offset into theta (kinds 0-4) or into the buffer array   */
  int64_t count;
} petra_tensor_info;

/* Tensors: all learnable tensors first (theta order), then running stats. */
petra_status petra_stage_num_tensors(const petra_stage *s, int32_t *n);
petra_status petra_stage_tensor_info(const petra_stage *s, int32_t i, petra_tensor_info *info);

/* Copy theta / momentum v / running stats to or from HOST arrays (any pointer
 * may be NULL to skip).  Synchronises the stage's last stream.  get_params
 * also reports a latched PETRA_E_NONFINITE. */
petra_status petra_stage_get_params(petra_stage *s, float *theta, float *v, float *buffers);
petra_status petra_stage_set_params(petra_stage *s, const float *theta, const float *v, const float *buffers);
/* Gradient Delta of the last backward (before the update), host copy. */
petra_status petra_stage_get_grads(petra_stage *s, float *delta);

/* Forward tick (Alg. 1 lines 3-10).  x*_in / x*_out: dev, fp32
 * NHWC halves.  Reversible units retain nothing; non-reversible
 * units push their input onto their device FIFO keyed by mb_id (reading c5).
 * BN uses batch statistics and does NOT update running stats.
 * out must not alias in.  Errors: PETRA_E_ARG, PETRA_E_ORDER (mb_id not
 * increasing), PETRA_E_CUDA. */
petra_status petra_stage_forward(petra_stage *s, uint64_t mb_id,
                                 const float *x1_in, const float *x2_in,
                                 float *x1_out, float *x2_out, void *stream);

/* Backward tick + immediate update with learning rate lr (Alg. 1 lines 11-24;
 * PAPER.md:132-135).  Inputs: the reconstructed output x~_j (xt*_out) and
 * delta_{j+1} (d*_out) received from stage j+1.  Reversible units reconstruct
 * their input with the CURRENT theta (approximate inversion),
 * keep the graph and run the VJP without a second forward;
 * BN running stats are updated in this recomputation.
 * Non-reversible units pop their FIFO (must match mb_id), recompute, VJP, and
 * return the exact buffered input (reading c6).  Outputs: x~_{j-1} (xt*_in)
 * and delta_j (d*_in), dev.  Outputs must not alias inputs.
 * Errors: PETRA_E_ARG, PETRA_E_EMPTY_BUFFER, PETRA_E_ORDER, PETRA_E_CUDA. */
petra_status petra_stage_backward(petra_stage *s, uint64_t mb_id,
                                  const float *xt1_out, const float *xt2_out,
                                  const float *d1_out, const float *d2_out,
                                  float *xt1_in, float *xt2_in, float *d1_in, float *d2_in,
                                  float lr, void *stream);

/* Final stage (Alg. 1 lines 26-35): forward with stored activations (running
 * stats updated here, reading c10), loss, plain backprop, update, all in one
 * call.  Returns the RECEIVED input as x~ (copied to xt*_in, may be NULL) and
 * delta_J w.r.t. that input (reading c7).  labels: dev int32[B].
 * loss_dev: dev float[1] (batch-mean cross-entropy), may be NULL. */
petra_status petra_stage_tail(petra_stage *s, uint64_t mb_id,
                              const float *x1_in, const float *x2_in, const int32_t *labels,
                              float lr, float *xt1_in, float *xt2_in, float *d1_in, float *d2_in,
                              float *loss_dev, void *stream);

/* Evaluation forward (the running statistics of batch normalisation "are
 * then used during model evaluation"): every unit of a NON-final stage
 * with BN normalising by the running mean / variance (invstd = 1/sqrt(var + eps)); nothing
 * is pushed on the FIFOs, no statistics or parameters change.  Layout as
 * petra_stage_forward (x2 NULL for a stem-first stage).  Must not overlap a training
 * forward of the same stage (it uses the forward workspace); non-reversible units need a
 * free FIFO slot (drain the pipeline first).  Enqueued on `stream`.
 * Errors: PETRA_E_ARG, PETRA_E_CUDA. */
petra_status petra_stage_eval(petra_stage *s, const float *x1_in, const float *x2_in, float *x1_out, float *x2_out,
                              void *stream);
/* Final stage: evaluation forward, then the classifier; adds to *correct_dev (device int32)
 * the number of rows whose first-index argmax logit equals the label and writes the
 * batch-mean cross-entropy to *loss_dev (device float).  labels_dev: int32[B].
 * Errors: PETRA_E_ARG, PETRA_E_CUDA. */
petra_status petra_stage_eval_tail(petra_stage *s, const float *x1_in, const float *x2_in, const int32_t *labels_dev,
                                   int32_t *correct_dev, float *loss_dev, void *stream);

/* ------------------------------------------------------------------ pipeline
 * One process (rank) owns a contiguous block of stages.  petra_pipeline_tick
 * runs tick t of every local stage (forward then backward, both at theta^t,
 * then the update; reading c8).  Mailboxes are double-buffered: a message
 * produced at tick t is consumed at t+1 (PAPER.md:131-134 superscripts).
 * Same-rank neighbours hand messages over by pointer.  Cross-rank neighbours
 * exchange only with their neighbours ("each stage ...
 * communicates only with its neighbours"; Alg. 1 Send/Receive):
 * forward messages (x1, x2, labels) to rank+1, backward messages (x~1, x~2, d1,
 * d2; 2x the forward bytes) to rank-1.  The transport moves them:
 *
 *   PETRA_TRANSPORT_NONE   the caller moves the bytes petra_pipeline_comm() lists
 *                          after each tick (world == 1 needs nothing);
 *   PETRA_TRANSPORT_NCCL   the library: ncclSend / ncclRecv on two library-owned
 *                          streams (one per direction), one NCCL group per
 *                          direction and tick.  The forward group of tick t is
 *                          issued when the last local stage's FORWARD of tick t is
 *                          done, so it overlaps that tick's backwards; the
 *                          backward group when the first local stage's backward is
 *                          done.  At tick t+1 only the stage that consumes a
 *                          received message waits for it (external event nodes in
 *                          the stage's CUDA graph); the others start at once.
 *                          nccl_id: 128 bytes from petra_nccl_unique_id() on rank 0,
 *                          given to every rank (e.g. via torch.distributed);
 *   PETRA_TRANSPORT_LOCAL  the same schedule, events and overlap for `world`
 *                          pipelines of ONE process on one device (a test
 *                          transport): ranks find each other by `local_group`
 *                          and the sender copies into the receiver's buffer
 *                          (cudaMemcpyAsync on its comm stream).  The host must
 *                          run tick t of every rank before tick t+1 of any.
 *
 * With a library transport, petra_pipeline_tick joins the caller's stream to the
 * tick's exchange (join_comm != 0, the default: a per-tick device timer then
 * includes the communication) or leaves it running under the next tick
 * (join_comm == 0).
 */
typedef enum { PETRA_TRANSPORT_NONE = 0, PETRA_TRANSPORT_NCCL = 1, PETRA_TRANSPORT_LOCAL = 2 } petra_transport;
/* Message format at stage boundaries ("doubles the cost of
 * backward communications"):
 *   PETRA_WIRE_FP32  messages are the fp32 stream values (default; the inversion
 *                    reconstructs x~ from exactly what the next stage computed);
 *   PETRA_WIRE_BF16  every message a stage sends (x1, x2 forward; x~1, x~2, d1, d2
 *                    backward) is rounded to bf16 (round-to-nearest-even) by the producing
 *                    stage before it is declared final, at EVERY stage boundary whatever the
 *                    rank layout (so the numerics do not depend on it), and cross-rank
 *                    transfers carry 2-byte elements: half the NVLink bytes.  Stage 1's
 *                    injected input is not a message and is not rounded.  The error this
 *                    adds is measured in DESIGN.md (section 9, "bf16 wire"). */
typedef enum { PETRA_WIRE_FP32 = 0, PETRA_WIRE_BF16 = 1 } petra_wire;

typedef struct {
  int32_t n_stages;                /* J                                                */
  const petra_stage_desc *stages;  /* all J stage descriptors (every rank passes all)  */
  const int32_t *stage_rank;       /* rank owning stage j (contiguous, non-decreasing) */
  int32_t rank, world;
  uint64_t seed;                   /* stage j is created with seed + j                 */
  int32_t transport;               /* petra_transport                                  */
  const unsigned char *nccl_id;    /* NCCL: 128 bytes (petra_nccl_unique_id)           */
  int64_t local_group;             /* LOCAL: nonzero key shared by the ranks           */
  int32_t join_comm;               /* library transports: see above (1 = default)      */
  int32_t wire;                    /* petra_wire: message format at stage boundaries   */
} petra_pipeline_desc;

/* NCCL unique id for PETRA_TRANSPORT_NCCL (call on rank 0, share with all ranks).
 * Errors: PETRA_E_NCCL (libnccl.so.2 not loadable), PETRA_E_ARG (NULL). */
petra_status petra_nccl_unique_id(unsigned char out[128]);

typedef struct petra_pipeline petra_pipeline;

#define PETRA_MAX_STAGES 64
typedef struct {              /* integer part is compared bit-exactly with the oracle      */
  int64_t tick;
  int32_t n_stages;           /* J (report covers all stages; non-local entries are replayed) */
  int64_t fwd_mb[PETRA_MAX_STAGES];        /* -1 = idle this tick                        */
  int64_t bwd_mb[PETRA_MAX_STAGES];
  int64_t param_version[PETRA_MAX_STAGES]; /* updates applied before this tick           */
  int64_t fifo_depth[PETRA_MAX_STAGES];    /* summed over the stage's FIFOs, after tick  */
} petra_tick_report;

petra_status petra_pipeline_create(const petra_pipeline_desc *desc, petra_pipeline **out);
petra_status petra_pipeline_destroy(petra_pipeline *p);
/* Borrow the handle of stage j (1-based); NULL if not local. */
petra_status petra_pipeline_stage(petra_pipeline *p, int32_t j, petra_stage **out);

/* Tick t.  inject != 0: stage 1 consumes micro-batch id mb = number of
 * injections so far; x0 (dev, stage-1 input layout) and labels (dev int32[B])
 * are read on the rank owning stage 1 (pass them or NULL elsewhere).  lr: the
 * tick's learning rate.  loss_dev: dev float[1] written by the tail stage
 * (rank owning stage J) when it ran.  report: nullable. */
petra_status petra_pipeline_tick(petra_pipeline *p, int64_t t, int32_t inject,
                                 const float *x0, const int32_t *labels, float lr,
                                 float *loss_dev, void *stream, petra_tick_report *report);

/* Transport plan for the messages this rank must exchange after tick t so
 * that tick t+1 can consume them.  Each entry is one contiguous device buffer. */
typedef struct {
  int32_t peer;      /* rank                                  */
  int32_t send;      /* 1 = send to peer, 0 = receive          */
  void *ptr;         /* dev                                    */
  int64_t bytes;
} petra_comm_entry;
#define PETRA_MAX_COMM 16
typedef struct {
  int32_t n;
  petra_comm_entry e[PETRA_MAX_COMM];
} petra_comm_plan;
petra_status petra_pipeline_comm(petra_pipeline *p, int64_t t, petra_comm_plan *plan);

/* Per-stage device time: enable != 0 starts recording CUDA events around each
 * local stage's work of every tick (on the stage's stream); petra_pipeline_stage_ms
 * synchronises and returns, per stage j = 1..J (0 for non-local stages), the
 * summed milliseconds and the number of ticks recorded since enabling. */
petra_status petra_pipeline_timing(petra_pipeline *p, int32_t enable);
petra_status petra_pipeline_stage_ms(petra_pipeline *p, float *ms, int32_t n, int32_t *ticks);

/* ------------------------------------------------------------------ schedule (host only)
 * The integer bookkeeping petra_pipeline_tick runs, exposed without any device
 * work so the multi-rank routing can be tested on CPU (gloo) and compared
 * bit-exactly with the oracle's tick engine.  stage_rank as in
 * petra_pipeline_desc; nonrev[j-1] = number of non-reversible units of stage j
 * (FIFO accounting); accum_k[j-1] = stage j's accumulation factor k (its
 * param_version advances on every k-th backward, Alg. 1 lines 19-23).  petra_schedule_tick must be called for t = 0, 1, 2, ...;
 * it fills report (all J stages) and the messages THIS rank exchanges after the
 * tick: kind 0 = forward (x1, x2, labels), 1 = backward (x~1, x~2, d1, d2). */
typedef struct petra_schedule petra_schedule;
typedef struct {
  int32_t peer, send, kind, stage; /* stage: 1-based index of the sending stage */
  int64_t mb;
} petra_sched_msg;
typedef struct {
  int32_t n;
  petra_sched_msg m[8];
} petra_sched_msgs;
petra_status petra_schedule_create(int32_t n_stages, const int32_t *stage_rank, const int32_t *nonrev,
                                   const int32_t *accum_k /* nullable: all 1 */, int32_t rank,
                                   petra_schedule **out);
petra_status petra_schedule_tick(petra_schedule *s, int64_t t, int32_t inject, petra_tick_report *report,
                                 petra_sched_msgs *msgs);
petra_status petra_schedule_destroy(petra_schedule *s);

/* ------------------------------------------------------------------ instrumentation
 * petra_launch_count: cumulative number of CUDA kernels the library launched.
 * petra_profile(1) starts recording CUDA events (on the launching stream)
 * around every logical kernel, grouped by category; petra_profile(0) stops.
 * petra_profile_read synchronises the device and returns one entry per
 * category: launches, summed event time, and the ALGORITHMIC flops / bytes of
 * those launches (2*M*N*K per convolution; read+write bytes of the streaming
 * kernels) -- the numerators of the roofline fractions. */
typedef struct {
  char name[32];
  int64_t launches;
  double ms;
  double flops;
  double bytes;
} petra_prof_entry;
/* Kernel-level test hook: run ONE convolution pass on host buffers (device
 * buffers are allocated, used and freed inside; synchronous).
 *   mode 0 forward : out[B*Ho*Wo][Co]  = conv(a = x[B][H][W][Ci], b = w[Co][k][k][Ci])
 *   mode 1 dgrad   : out[B*H*W][Ci]    = addend + conv^T(a = dz[B][Ho][Wo][Co], b = w)
 *   mode 2 wgrad   : out[Co][k][k][Ci] = sum over pixels of dz (a) (x) x (b = x)
 * engine 0 = SIMT fp32 kernels, 1 = tcgen05 bf16 kernels (inputs rounded to bf16;
 * PETRA_E_UNSUPPORTED if the geometry has no tensor-core path), 2 = tcgen05 with the
 * activation operands held zero-bordered ([B][H+2][W+2][C], as the library keeps them
 * for 3x3 stride-1 layers; large grids then run the halo kernel).  addend may be NULL. */
typedef struct {
  int32_t batch, h, w, cin, cout, ksize, stride;
} petra_conv_geom;
petra_status petra_conv_run(int32_t mode, int32_t engine, const petra_conv_geom *g, const float *a,
                            const float *b, const float *addend, float *out);
/* Kernel benchmark: one convolution pass (as petra_conv_run, on seeded random device
 * inputs) repeated `iters` times after one warm-up; *avg_ms = mean device time per pass
 * (CUDA events around one CUDA-graph replay of the `iters` passes, so host-side launch
 * and tensor-map encoding time is excluded).  flags bit 0: forward output z in bf16 (the
 * tensor-core stage layout); bit 1: forward with the BN statistics fused into the
 * epilogue (as a stage runs it); bit 2: time direct launches instead of the graph. */
petra_status petra_conv_bench(int32_t mode, int32_t engine, const petra_conv_geom *g, int32_t flags,
                              int32_t iters, float *avg_ms);
/* Kernel-level test hook of the fused BN statistics: one tensor-core
 * forward convolution with z stored in bf16 and the batch statistics fused into its
 * epilogue, exactly as a stage runs it (engine 1: plain operand, the stem's gathered
 * im2col for Ci <= 4; engine 2: zero-bordered operand, the halo kernel where eligible),
 * then the library's merge.  Each CTA keeps per column the shifted sums of its valid rows
 * (shift = the mean of its first tile) and writes (count, mean, M2); the merge combines
 * them over CTAs with Chan's pairwise update in fp64 in a fixed order.  Outputs (host):
 * z[B*Ho*Wo][Co] (the stored bf16 values as fp32), mean[Co] and the biased variance
 * var[Co] the library normalises with.  Synchronous.  Errors: PETRA_E_ARG,
 * PETRA_E_UNSUPPORTED (no tensor-core path / no fused statistics), PETRA_E_CUDA. */
petra_status petra_conv_bn_stats(const petra_conv_geom *g, int32_t engine, const float *x, const float *w,
                                 float *z, float *mean, float *var);
/* Which engine the library uses for a convolution pass at a given precision:
 * 0 = SIMT fp32, 1 = tcgen05 bf16 (operands rounded to bf16, fp32 accumulation) --
 * the TMA implicit GEMM for Ci, Co multiples of 64, or, for few input channels (the
 * stem: Ci <= 4, k <= 8, Co in {64, 128, 256}; forward and wgrad), the
 * gathered-im2col kernel. */
int32_t petra_conv_engine(const petra_conv_geom *g, int32_t mode, int32_t precision);
/* The tcgen05 im2col kernel's launch plan for a forward (mode 0) or stride-1 dgrad
 * (mode 1) pass of the geometry (host only, no device work): plan[0] = N tile BN,
 * plan[1] = K splits, plan[2] = cluster size (> 1: the splits of a tile are the CTAs
 * of one thread-block cluster reduced through distributed shared memory -- DESIGN.md 7
 * "Cluster split-K"; -2: CTA pairs, M = 256 tiles on cta_group::2 UMMAs -- DESIGN.md 7
 * "CTA pairs").  Errors: PETRA_E_ARG (NULL, bad mode), PETRA_E_UNSUPPORTED (no
 * tensor-core im2col path for the pass). */
petra_status petra_conv_plan(const petra_conv_geom *g, int32_t mode, int32_t *plan);
int64_t petra_launch_count(void);
petra_status petra_profile(int32_t enable);
petra_status petra_profile_read(petra_prof_entry *out, int32_t cap, int32_t *n);
/* The same profile per logical kernel, in enqueue order: category index (the order of
 * petra_profile_read's categories before it drops empty ones is the order of first use;
 * `name` repeats it), event time, algorithmic flops and bytes of that one launch and its
 * largest grid -- for a
 * roofline per launch (each launch's own bound, max(flops / tensor peak, bytes / HBM peak)).
 * Writes min(cap, records) entries, *n = the number of records.  Errors: PETRA_E_ARG (NULL),
 * PETRA_E_CUDA. */
typedef struct {
  char name[32];
  float ms;
  double flops;
  double bytes;
  int32_t ctas;  /* largest grid (CTAs) the logical kernel launched */
} petra_prof_record;
petra_status petra_profile_records(petra_prof_record *out, int32_t cap, int32_t *n);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* PETRA_H */

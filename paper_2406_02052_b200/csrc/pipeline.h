// pipeline.h -- stages of one rank, mailboxes and the neighbour exchange (product code).
#pragma once
#include <array>
#include <memory>
#include <vector>

#include "nccl_dl.h"
#include "schedule.h"
#include "stage.h"

namespace petra {

struct Msg {
  DevPtr x[4];    // forward: x1, x2 ; backward: x~1, x~2, d1, d2
  DevPtr labels;  // forward only
};

class Pipeline {
 public:
  explicit Pipeline(const petra_pipeline_desc &d);
  ~Pipeline();
  Stage *stage(int j) { return (j >= 1 && j <= J_) ? stages_[j].get() : nullptr; }
  void tick(int64_t t, bool inject, const float *x0, const int32_t *labels, float lr, float *loss, cudaStream_t st,
            petra_tick_report *rep);
  void comm(int64_t t, petra_comm_plan *plan);
  void timing(bool on);
  int stage_ms(float *ms, int n);

 private:
  enum { DIR_FWD = 0, DIR_BWD = 1 };
  int J_, rank_, world_;
  int transport_ = PETRA_TRANSPORT_NONE;
  int64_t group_ = 0;
  bool join_comm_ = true;
  int wire_ = PETRA_WIRE_FP32;
  // bf16 wire: 2-byte images of the cross-rank messages ([dir][parity]; send = this rank's
  // outgoing message, recv = the incoming one before it is widened into the ghost buffer)
  Msg wsend_[2][2], wrecv_[2][2];
  Schedule sched_;
  std::vector<petra_stage_desc> descs_;
  std::vector<std::unique_ptr<Stage>> stages_;
  std::vector<std::array<Msg, 2>> fwd_, bwd_;  // [j][parity]: outputs of local stage j
  Msg ghost_fwd_[2], ghost_bwd_[2];            // receive buffers for remote neighbours
  // one stream per local stage: the stages of a tick are independent (they only
  // read mailboxes of the previous tick), so their kernels overlap on the GPU
  std::vector<cudaStream_t> streams_;
  std::vector<cudaEvent_t> done_;
  cudaEvent_t start_ = nullptr;
  DevPtr x0_stage_[2], lab_stage_[2];  // caller inputs copied to fixed buffers (graph keys stay fixed)
  bool graphs_ = true;
  bool timing_ = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tev_[PETRA_MAX_STAGES + 2];
  std::vector<cudaEvent_t> ev_pool_;
  size_t ev_next_ = 0;
  int timed_ticks_ = 0;
  cudaEvent_t ev();

  // ---- library transports (NCCL, LOCAL)
  ncclComm_t nccl_comm_ = nullptr;
  cudaStream_t cs_[2] = {nullptr, nullptr};               // comm stream per direction
  cudaEvent_t cdone_[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [dir][parity]: exchange done
  // per local stage and parity: forward part done, backward part done, whole tick done
  std::vector<std::array<cudaEvent_t, 2>> fdone_, bdone_, tdone_;
  bool lib_transport() const { return transport_ != PETRA_TRANSPORT_NONE; }
  Pipeline *peer(int rank) const;          // LOCAL: the pipeline of another rank
  cudaEvent_t recv_done(int dir, int parity) const;
  void exchange(int64_t t, std::vector<bool> &used);

  Msg &ghost_fwd(int p) { return ghost_fwd_[p]; }
  Msg &ghost_bwd(int p) { return ghost_bwd_[p]; }
};

}  // namespace petra

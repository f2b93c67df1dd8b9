// schedule.h -- host-side PETRA tick bookkeeping (product code, no device work).
//
// Every rank replays the integer schedule of ALL J stages (it is a function of
// the injection history only), so each rank knows which messages exist at each
// tick without extra communication.  Mailboxes are double-buffered: a message
// produced at tick t (parity t&1) is consumed at t+1 (PAPER.md:131-134
// superscripts; reading c8).  Stage j forwards micro-batch m at t = m+j-1 and
// backwards it at t = m+2J-j-1 (delay 2(J-j), Table 1).
#pragma once
#include <array>
#include <cstdint>
#include <vector>

#include "errors.h"

namespace petra {

class Schedule {
 public:
  struct Box {
    bool valid = false;
    int64_t mb = -1;
  };
  struct Step {           // what stage j does at this tick
    int64_t fwd_mb = -1;  // -1: idle
    int64_t bwd_mb = -1;
  };
  enum { MSG_FWD = 0, MSG_BWD = 1 };
  struct Comm {
    int peer, send, kind, stage;  // stage = sender's stage index (1-based)
    int64_t mb;
  };

  // accum_k[j-1] = accumulation factor k of stage j (Alg. 1 lines 19-23): the
  // parameter version advances on every k-th backward (t mod k == 0, t from 1)
  Schedule(int J, std::vector<int> rank_of, std::vector<int> nonrev, int rank, std::vector<int> accum_k = {})
      : J_(J), rank_of_(std::move(rank_of)), nonrev_(std::move(nonrev)), k_(std::move(accum_k)), rank_(rank) {
    if (k_.empty()) k_.assign(J > 0 ? J : 0, 1);
    if (J < 1 || (int)rank_of_.size() != J || (int)nonrev_.size() != J || (int)k_.size() != J)
      throw PetraError(PETRA_E_ARG, "schedule: bad stage count");
    for (int k : k_)
      if (k < 1) throw PetraError(PETRA_E_ARG, "schedule: accumulation k must be >= 1");
    for (int j = 1; j < J; ++j)
      if (rank_of_[j] < rank_of_[j - 1]) throw PetraError(PETRA_E_ARG, "stage_rank must be non-decreasing");
    j0_ = J + 1;
    j1_ = 0;
    for (int j = 1; j <= J; ++j)
      if (rank_of_[j - 1] == rank_) {
        j0_ = std::min(j0_, j);
        j1_ = std::max(j1_, j);
      }
    fwd_.assign(J + 2, {});
    bwd_.assign(J + 2, {});
    version_.assign(J + 2, 0);
    nbwd_.assign(J + 2, 0);
    fifo_.assign(J + 2, 0);
  }

  int J() const { return J_; }
  int first_local() const { return j0_; }
  int last_local() const { return j1_; }
  bool local(int j) const { return j >= 1 && j <= J_ && rank_of_[j - 1] == rank_; }
  int rank_of(int j) const { return rank_of_[j - 1]; }
  int64_t n_injected() const { return n_inject_; }

  // Advance to tick t (must be consecutive).  Fills steps[j] (1-based) and the
  // report arrays (versions used this tick, FIFO depth after it).
  std::vector<Step> tick(int64_t t, bool inject, std::vector<int64_t> *version_used = nullptr,
                         std::vector<int64_t> *fifo_after = nullptr) {
    if (t != last_t_ + 1) throw PetraError(PETRA_E_ORDER, "ticks must be consecutive from 0");
    last_t_ = t;
    const int p = (int)(t & 1), q = p ^ 1;
    std::vector<Step> steps(J_ + 2);
    if (version_used) version_used->assign(J_ + 2, 0);
    for (int j = 1; j <= J_; ++j) {
      int64_t fin = -1, bin = -1;
      if (j == 1) {
        if (inject) fin = n_inject_;
      } else if (fwd_[j - 1][q].valid) {
        fin = fwd_[j - 1][q].mb;
      }
      if (j == J_) bin = fin;
      else if (bwd_[j + 1][q].valid) bin = bwd_[j + 1][q].mb;
      steps[j].fwd_mb = fin;
      steps[j].bwd_mb = bin;
      if (version_used) (*version_used)[j] = version_[j];
      fwd_[j][p] = Box{j < J_ && fin >= 0, fin};
      bwd_[j][p] = Box{j > 1 && bin >= 0, bin};
      if (fin >= 0) fifo_[j] += nonrev_[j - 1];
      if (bin >= 0) {
        fifo_[j] -= nonrev_[j - 1];
        if (++nbwd_[j] % k_[j - 1] == 0) version_[j] += 1;
      }
    }
    if (fifo_after) fifo_after->assign(fifo_.begin(), fifo_.end());
    if (inject) ++n_inject_;
    return steps;
  }

  // Messages this rank exchanges after tick t (to be consumed at t+1).
  std::vector<Comm> comm(int64_t t) const {
    std::vector<Comm> out;
    if (t != last_t_) throw PetraError(PETRA_E_ORDER, "comm plan only for the last tick");
    const int p = (int)(t & 1);
    if (j1_ < 1) return out;
    if (j1_ < J_ && fwd_[j1_][p].valid) out.push_back({rank_of(j1_ + 1), 1, MSG_FWD, j1_, fwd_[j1_][p].mb});
    if (j0_ > 1 && fwd_[j0_ - 1][p].valid)
      out.push_back({rank_of(j0_ - 1), 0, MSG_FWD, j0_ - 1, fwd_[j0_ - 1][p].mb});
    if (j0_ > 1 && bwd_[j0_][p].valid) out.push_back({rank_of(j0_ - 1), 1, MSG_BWD, j0_, bwd_[j0_][p].mb});
    if (j1_ < J_ && bwd_[j1_ + 1][p].valid)
      out.push_back({rank_of(j1_ + 1), 0, MSG_BWD, j1_ + 1, bwd_[j1_ + 1][p].mb});
    return out;
  }

 private:
  int J_;
  std::vector<int> rank_of_, nonrev_, k_;
  int rank_;
  int j0_, j1_;
  std::vector<std::array<Box, 2>> fwd_, bwd_;
  std::vector<int64_t> version_, fifo_, nbwd_;
  int64_t n_inject_ = 0, last_t_ = -1;
};

}  // namespace petra

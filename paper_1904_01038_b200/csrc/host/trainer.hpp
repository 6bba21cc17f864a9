// B200 data-parallel trainer with the reference's Trainer contract
// (include/seqforge/trainer.hpp:80-125, src/trainer.cpp:89-289): W replicas x A
// accumulation, loss-scale seeding of backward, bucketed all-reduce, overflow
// skip + scaler policy, unscale, / global ntokens, optimizer, rebroadcast.
//
// Replica placement: one process per GPU (rank r of `world`), each owning
// workers/world logical replicas. Within a process the replicas run one after
// another on its GPU and fold in index order (trainer.cpp:75-87); across
// processes gradients are summed by bucketed NCCL all-reduce over NVLink.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <functional>
#include <future>
#include <memory>
#include <optional>

#include "collective.hpp"
#include "device_tape.hpp"
#include "plugins.hpp"

namespace sqf {

struct StepStats {
  int64_t step = 0;
  double loss = 0.0, nll = 0.0;
  int64_t ntokens = 0, ncorrect = 0;
  double lr = 0.0;
  bool skipped = false;
  double scale = 0.0;
};

struct EvalStats {
  double loss = 0.0, nll = 0.0;
  int64_t ntokens = 0, ncorrect = 0;
};

class Trainer {
 public:
  // task == nullptr: the task is made through the registry from cfg["task"];
  // world > 1 needs the collective that joins the ranks (NCCL in production)
  Trainer(const Config& cfg, const Registry& reg, std::unique_ptr<TaskBase> task, int rank = 0, int world = 1,
          std::unique_ptr<Collective> coll = nullptr);
  ~Trainer();

  std::optional<StepStats> train_one();
  StepStats train_step(const std::vector<std::vector<MiniBatch>>& sub);
  EvalStats evaluate(const std::vector<SequencePair>& pairs);
  // generation support (generate.cpp): teacher-forced decoder pass of `mb` on
  // the fp32 master; returns the logits of each row's last target position,
  // rows x target_vocab, row-major (reference generate.cpp:86-120)
  std::vector<float> last_position_logits(const MiniBatch& mb);
  // incremental decoding (reference make_incremental_state /
  // forward_decoder_step / reorder_incremental_state, model.cpp:315-557):
  // K/V caches of `rows` hypotheses live on the device; row r decodes
  // sentence row_sentence[r] of `src` (only source fields used); positions
  // up to cap-1. step returns rows x target_vocab logits; reorder gathers
  // cache rows (new row r = old row order[r]).
  void inc_begin(const MiniBatch& src, const std::vector<int>& row_sentence, int cap);
  std::vector<float> inc_step(const std::vector<int>& last_tokens, int pos);
  // the same step with candidate selection on the device (sfk_beam_topk):
  // per row lse, eos log-prob and the kk best (token, log-prob) under
  // key = cum[r] + lp, best first -- rows x kk values come back, not rows x V
  struct BeamCands {
    int kk = 0;
    std::vector<float> lse, eos_lp, lp;
    std::vector<int32_t> tok;
  };
  // empty cum: rank raw logits instead and return them in lp (sampling)
  BeamCands inc_step_topk(const std::vector<int>& last_tokens, int pos, const std::vector<double>& cum, int kk);
  void inc_reorder(const std::vector<int>& order);
  void inc_end();

  int64_t step() const { return step_; }
  int epoch() const { return epoch_; }
  int cursor() const { return pos_; }
  int batches_per_epoch() const { return int(plan_.batches.size()); }
  int workers() const { return workers_; }
  int accum() const { return accum_; }
  bool fp16() const { return fp16_; }
  const Config& config() const { return cfg_; }
  ModelBase& model() { return *model_; }
  OptimizerBase& optimizer() {
    join_optimizer();  // host access to the moments: the update may still run on the side stream
    return *optimizer_;
  }
  // wait (host) for the last optimizer update, which runs on the side stream
  // overlapped with the next step's forward
  void join_optimizer();
  // make the compute stream wait for the last update and return the device
  // time (ms) from the end of the last step's main-stream work to that point
  float flush_ms();
  TaskBase& task() { return *task_; }
  const LossScaler& scaler() const;
  const std::vector<GradientBucket>& buckets() const { return buckets_; }

  // host <-> device parameter sync (canonical order)
  void pull_params();                       // device master -> model().params()
  void push_params();                       // model().params() -> device master, then rebroadcast
  void rebroadcast();
  std::vector<float> reduced_grads();       // last step's reduced gradient, canonical order, as float
  void restore_progress(int64_t step, int epoch, int cursor);
  void restore_scaler(double scale, int64_t successes);
  void set_overflow_injector(std::function<bool(int64_t)> f) { injector_ = std::move(f); }

  int64_t kernel_launches() const { return launches_; }
  int dtype() const { return dtype_; }
  cudaStream_t stream() const { return stream_; }
  int rank() const { return rank_; }
  int world() const { return world_; }
  const char* collective() const { return coll_ ? coll_->name() : "none"; }
  // timing hook: events recorded on the compute stream around the last step
  float last_step_ms() const { return last_ms_; }
  // host<->device bytes of the last step (packed batch ids up; stats + flag down)
  int64_t last_h2d_bytes() const { return h2d_bytes_; }
  int64_t last_d2h_bytes() const { return 36; }
  // per-launch event profiling of subsequent steps (bench roofline evidence)
  // mode 0 off, 1 serialised per-launch timing (every launch alone on the
  // main stream), 2 timeline of the concurrent schedule
  void set_profile(int mode) {
    if (mode && !prof_) prof_ = std::make_unique<Profiler>();
    if (!mode) prof_.reset();
    if (prof_) {
      prof_->concurrent = mode == 2;
      prof_->streams = {stream_, side_, comm_stream_};
    }
  }
  Profiler* profiler() { return prof_.get(); }
  // all-reduce/backward overlap of the last step: bucket indices in issue
  // order, and how many were issued while backward was still running
  const std::vector<int>& overlap_log() const { return overlap_log_; }
  int overlap_early() const { return overlap_early_; }

 private:
  struct IncState {
    int rows = 0, src_width = 0, cap = 0, layers = 0, d = 0;
    int filled = 0;                      // cache positions written so far (reorder copies these)
    size_t es = 4;                       // cache element size (decoding dtype)
    void* self[2] = {nullptr, nullptr};  // double-buffered [layers][rows*cap][2d]
    int cur = 0;
    void* cross = nullptr;               // [rows*src_width][layers*2d]
    int32_t* idx = nullptr;              // device: ids[rows] | self_len[rows] | src_len[rows] | order[rows]
    double* cum = nullptr;               // device [rows]
    void* cands = nullptr;               // device: lse | eos_lp | tok[rows*kk] | lp[rows*kk]
    int cands_kk = 0;
    ~IncState() {
      cudaFree(cum);
      cudaFree(cands);
      cudaFree(self[0]);
      cudaFree(self[1]);
      cudaFree(cross);
      cudaFree(idx);
    }
  };
  std::unique_ptr<IncState> inc_;
  int64_t logits_ld(int V) const;
  const float* logits_as_f32(const void* logits, int64_t n);
  void inc_run(const std::vector<int>& last, int pos, const std::function<void(DeviceTape&, int)>& consume);

  Config cfg_;
  std::unique_ptr<TaskBase> task_;
  std::unique_ptr<ModelBase> model_;
  std::unique_ptr<CriterionBase> criterion_;
  std::unique_ptr<OptimizerBase> optimizer_;
  std::unique_ptr<SchedulerBase> scheduler_;
  std::unique_ptr<LossScaler> scaler_;

  int workers_ = 1, accum_ = 1, max_epochs_ = 1;
  bool fp16_ = false, bf16_ = false, deal_ = false;
  int dtype_ = SFK_F32;
  uint64_t seed_ = 1;
  int rank_ = 0, world_ = 1, local_ = 1;

  // device state (device parameter order)
  int64_t n_ = 0;
  float* master_ = nullptr;
  void* compute_ = nullptr;        // == master_ in fp32 mode
  std::vector<void*> grads_;       // [2 sets][local replicas], compute dtype
  int gset_ = 0, last_gset_ = 0;   // set this step accumulates into / last completed step's set
  void* grad_buf(int lw) const { return grads_[size_t(gset_ * local_ + lw)]; }
  float* pe_ = nullptr;
  double* stats_dev_ = nullptr;    // loss, nll, ntokens, ncorrect
  int32_t* flag_dev_ = nullptr;
  int32_t* counters_ = nullptr;    // zeroed pool for single-launch reductions
  int64_t counter_cursor_ = 0;
  static constexpr int64_t kCounters = 1 << 16;
  int32_t* blob_dev_ = nullptr;
  size_t blob_cap_ = 0;
  int32_t* blob_host_ = nullptr;   // pinned staging
  size_t blob_host_cap_ = 0;
  void* readback_host_ = nullptr;  // pinned: stats + flag
  cudaStream_t stream_ = nullptr;
  cudaStream_t side_ = nullptr;        // parameter-gradient stream (wgrad, bias grad)
  std::vector<cudaEvent_t> evpool_;    // ordering events handed to the tapes
  cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;
  // optimizer update overlapped with the next forward: per-range events the
  // forward waits on (once each), and per grad set the event after which the
  // set may be zeroed again
  std::vector<std::pair<int64_t, int64_t>> adam_ranges_;
  std::vector<cudaEvent_t> adam_range_ev_;
  std::vector<char> adam_range_wait_;
  cudaEvent_t adam_done_[2] = {nullptr, nullptr};
  bool adam_pending_[2] = {false, false};
  cudaEvent_t ev_checked_ = nullptr, ev_flush_ = nullptr;
  bool adam_overlap_ = true;
  void param_wait(int64_t offset, int64_t numel, cudaStream_t s);
  std::unique_ptr<Collective> coll_;
  // Two activation arenas alternate between sub-batches so the side-stream
  // parameter-gradient work of sub-batch i (which reads its activations) can
  // run under the forward of sub-batch i+1; arena k is reused only after the
  // side stream has passed arena_free_[k].
  Arena arena_[2];
  cudaEvent_t arena_free_[2] = {nullptr, nullptr};
  bool arena_busy_[2] = {false, false};

  std::vector<GradientBucket> buckets_;
  EpochPlan plan_;
  int epoch_ = 1, pos_ = 0;
  std::vector<int> order_;
  int64_t step_ = 0;
  std::function<bool(int64_t)> injector_;
  int64_t launches_ = 0;
  float last_ms_ = 0.f;
  int64_t h2d_bytes_ = 0;
  std::unique_ptr<Profiler> prof_;

  // Host-side batch preparation of the next deal-mode step (make_minibatch +
  // packing, trainer.cpp:173-184 / data.cpp:172-219) runs on a worker thread
  // while the GPU executes the current step; it works on a copy of the epoch
  // cursor and is used only if the cursor is still where it started.
  struct Prefetch {
    int epoch0 = 0, pos0 = 0;
    int epoch1 = 0, pos1 = 0;
    std::vector<int> order1;
    bool exhausted = false;
    std::vector<std::vector<MiniBatch>> sub;
    std::vector<PackedBatch> packs;
    std::vector<std::pair<int, int>> which;
  };
  Prefetch plan_deal(int epoch, int pos, std::vector<int> order) const;
  void pack_local(const std::vector<std::vector<MiniBatch>>& sub, std::vector<PackedBatch>& packs,
                  std::vector<std::pair<int, int>>& which) const;
  StepStats run_step(const std::vector<std::vector<MiniBatch>>& sub, std::vector<PackedBatch>& packs,
                     const std::vector<std::pair<int, int>>& which);
  std::future<Prefetch> prefetch_;
  bool prefetch_on_ = true;

  void init(const Registry& reg);
  std::optional<MiniBatch> next_batch();
  size_t esize() const { return dtype_ == SFK_F32 ? 4 : 2; }
  void upload(const std::vector<PackedBatch>& packs, std::vector<DeviceBatch>& out);
  void allreduce_grads();

  // ---- bucketed all-reduce overlapped with the last sub-batch's backward
  bool overlap_ = true, overlap_sim_ = false;
  cudaStream_t comm_stream_ = nullptr;
  // forward-ahead (SQF_FWD_AHEAD, default on): the next sub-batch's forward
  // on its own stream, concurrent with this sub-batch's backward
  cudaStream_t fwd_stream_ = nullptr;
  bool fwd_ahead_ = true;
  int pair_sub_ = 0;    // SQF_PAIR_SUBBATCH: widening (%) allowed when sub-batches share a pass (0 = off)
  int pair_group_ = 6;       // SQF_PAIR_GROUP: at most this many sub-batches per pass
  bool pair_parts_ = true;   // SQF_PAIR_PARTS: passes of unpadded parts (else re-padded merges)
  bool balance_groups_ = true;  // SQF_PAIR_BALANCE: near-equal-sized passes
  cudaEvent_t ev_upload_ = nullptr, fwd_done_[2] = {nullptr, nullptr}, main_done_[2] = {nullptr, nullptr};
  float* gemm_ws_ = nullptr;          // stream-K partial tiles: [main | side]
  int64_t gemm_ws_floats_ = 0;        // per stream
  std::vector<cudaEvent_t> ovl_events_;
  size_t ovl_next_event_ = 0;
  std::vector<int> ovl_remaining_;   // outstanding gradient writes per bucket
  int ovl_next_ = 0;                 // next bucket to issue (issue order = bucket order)
  std::vector<int> overlap_log_;
  int overlap_early_ = 0;
  std::vector<std::pair<int64_t, int>> bucket_index_;  // (start, bucket) sorted by start
  cudaEvent_t ovl_event();
  template <typename F>
  void for_buckets(int64_t offset, int64_t numel, F f) const;
  void ovl_begin(const DeviceTape& tape);
  void ovl_on_write(int64_t offset, int64_t numel);
  void ovl_issue(int b);
  void ovl_finish();
};

}  // namespace sqf

#include "trainer.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <tuple>

namespace sqf {

void set_model_position_table(ModelBase& m, const float* dev);
int ablate_mask();  // device_tape.cpp: SQF_ABLATE measurement knob

Trainer::Trainer(const Config& cfg, const Registry& reg, std::unique_ptr<TaskBase> task, int rank, int world,
                 std::unique_ptr<Collective> coll)
    : cfg_(cfg), task_(std::move(task)), rank_(rank), world_(world), coll_(std::move(coll)) {
  if (world_ < 1 || rank_ < 0 || rank_ >= world_) throw ConfigError("trainer: bad rank/world");
  if (world_ > 1 && !coll_) throw ConfigError("trainer: world > 1 needs a collective (NCCL unique id)");
  if (!task_) task_ = reg.make_task(cfg_.get_str("task"), cfg_);
  init(reg);
}

Trainer::~Trainer() {
  coll_.reset();
  cudaFree(master_);
  if (compute_ != master_) cudaFree(compute_);
  for (void* g : grads_) cudaFree(g);
  cudaFree(pe_);
  cudaFree(gemm_ws_);
  cudaFree(stats_dev_);
  cudaFree(flag_dev_);
  cudaFree(counters_);
  cudaFree(blob_dev_);
  cudaFreeHost(blob_host_);
  cudaFreeHost(readback_host_);
  if (ev0_) cudaEventDestroy(ev0_);
  for (auto e : adam_range_ev_) cudaEventDestroy(e);
  for (auto e : adam_done_)
    if (e) cudaEventDestroy(e);
  if (ev_checked_) cudaEventDestroy(ev_checked_);
  if (ev_flush_) cudaEventDestroy(ev_flush_);
  for (auto e : arena_free_)
    if (e) cudaEventDestroy(e);
  if (ev1_) cudaEventDestroy(ev1_);
  if (stream_) cudaStreamDestroy(stream_);
  if (side_) cudaStreamDestroy(side_);
  if (comm_stream_) cudaStreamDestroy(comm_stream_);
  if (fwd_stream_) cudaStreamDestroy(fwd_stream_);
  if (ev_upload_) cudaEventDestroy(ev_upload_);
  for (auto e : fwd_done_)
    if (e) cudaEventDestroy(e);
  for (auto e : main_done_)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : ovl_events_) cudaEventDestroy(e);
  for (cudaEvent_t e : evpool_) cudaEventDestroy(e);
}

void Trainer::init(const Registry& reg) {
  workers_ = int(cfg_.get_int("workers"));
  accum_ = int(cfg_.get_int("accum"));
  if (workers_ < 1 || accum_ < 1) throw ConfigError("trainer: workers and accum must be at least 1");
  if (workers_ % world_ != 0) throw ConfigError("trainer: workers must be a multiple of the process count");
  local_ = workers_ / world_;
  fp16_ = cfg_.get_bool("fp16");
  bf16_ = cfg_.get_bool("bf16");
  if (fp16_ && bf16_) throw ConfigError("trainer: fp16 and bf16 are exclusive");
  dtype_ = fp16_ ? SFK_F16 : bf16_ ? SFK_BF16 : SFK_F32;
  max_epochs_ = int(cfg_.get_int("max_epochs"));
  if (max_epochs_ < 1) throw ConfigError("trainer: max_epochs must be at least 1");
  seed_ = uint64_t(cfg_.get_int("seed"));
  const std::string dispatch = cfg_.get_str("dispatch");
  if (dispatch != "split" && dispatch != "deal") throw ConfigError("trainer: dispatch must be split or deal");
  deal_ = dispatch == "deal";

  if (cfg_.get_int("src_vocab") == 0) cfg_.set_user("src_vocab", int64_t(task_->source_vocab()));
  if (cfg_.get_int("tgt_vocab") == 0) cfg_.set_user("tgt_vocab", int64_t(task_->target_vocab()));

  model_ = reg.make_model(reg.architecture(cfg_.get_str("arch")).base_model, cfg_, seed_);
  criterion_ = reg.make_criterion(cfg_.get_str("criterion"), cfg_);
  optimizer_ = reg.make_optimizer(cfg_.get_str("optimizer"), cfg_, model_->num_params());
  scheduler_ = reg.make_scheduler(cfg_.get_str("scheduler"), cfg_);
  if (fp16_)
    scaler_ = std::make_unique<LossScaler>(cfg_.get_real("fp16_init_scale"), cfg_.get_int("fp16_scale_window"),
                                           cfg_.get_real("fp16_min_scale"), cfg_.get_real("fp16_max_scale"));

  // buckets over the device order (sizes of manifest entries sorted by device offset)
  std::vector<std::pair<int64_t, int64_t>> dev;
  for (const auto& e : model_->manifest()) dev.emplace_back(e.device_offset, e.numel);
  std::sort(dev.begin(), dev.end());
  std::vector<int64_t> sizes;
  for (auto& p : dev) sizes.push_back(p.second);
  buckets_ = bucket_gradients(sizes, cfg_.get_int("bucket_threshold"));
  for (size_t b = 0; b < buckets_.size(); ++b) bucket_index_.emplace_back(buckets_[b].start, int(b));
  std::sort(bucket_index_.begin(), bucket_index_.end());
  overlap_ = cfg_.get_bool("overlap_allreduce");
  overlap_sim_ = cfg_.get_bool("overlap_simulate");

  const int64_t ms = cfg_.get_int("max_sentences");
  // deal dispatch packs at the per-replica budget; split packs one global batch
  plan_ = make_batches(task_->train_pairs(), cfg_.get_int("max_tokens"),
                       ms > 0 ? std::optional<int>(int(ms)) : std::nullopt, seed_);
  epoch_ = 1;
  pos_ = 0;
  order_ = plan_.batches.empty() ? std::vector<int>{} : shuffle_epoch(plan_, 1);

  // device state
  n_ = model_->num_params();
  // Stream priorities (SQF_STREAM_PRIO): 2 = side stream above main (default),
  // 1 = main above side, 0 = equal. Measured on C4 (ms/step, CTA-pair main
  // GEMMs): 122.4 / 133.7 / 128.1 -- the parameter-gradient side stream is what
  // the end-of-step join waits for, so its blocks go first. The comm stream
  // always gets the top priority.
  int lo = 0, hi = 0;
  cuda_check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "stream priorities");
  const char* prio_env = std::getenv("SQF_STREAM_PRIO");
  const int prio = prio_env ? std::atoi(prio_env) : 2;
  const int mid = std::max(hi, lo - 1);
  int p_main = prio == 1 ? mid : prio == 2 ? lo : lo, p_side = prio == 2 ? mid : lo;
  const int p_comm = hi;
  // SQF_FWD_PRIO: the forward-ahead stream's priority -- 0 (default) lowest,
  // like the main stream; 1 the side stream's; 2 below the main stream, which
  // then sits between it and the side stream
  const char* fp_env = std::getenv("SQF_FWD_PRIO");
  const int fwd_prio = fp_env ? std::atoi(fp_env) : 0;
  int p_fwd = fwd_prio == 1 ? mid : lo;
  if (fwd_prio == 2 && prio == 2) {
    p_main = std::max(hi, lo - 1);
    p_side = std::max(hi, lo - 2);
  }
  cuda_check(cudaStreamCreateWithPriority(&stream_, cudaStreamNonBlocking, p_main), "stream");
  cuda_check(cudaStreamCreateWithPriority(&side_, cudaStreamNonBlocking, p_side), "side stream");
  cuda_check(cudaStreamCreateWithPriority(&comm_stream_, cudaStreamNonBlocking, p_comm), "comm stream");
  cuda_check(cudaStreamCreateWithPriority(&fwd_stream_, cudaStreamNonBlocking, p_fwd), "forward stream");
  {
    const char* e = std::getenv("SQF_FWD_AHEAD");
    fwd_ahead_ = !(e && std::atoi(e) == 0);
  }
  {
    // Sub-batch grouping (16-bit, no dropout): several packed sub-batches of
    // one update run as one pass, so every row-wise launch (GEMM, LayerNorm,
    // xent) covers several times the rows. Same batches, tokens and per-row
    // arithmetic; only the order of the gradient accumulation changes (fewer
    // rounded partial sums). fp32 keeps the reference's sub-batch-by-sub-batch
    // order for its 1e-4 parity, and dropout masks are drawn per sub-batch,
    // so both run one sub-batch per pass. SQF_PAIR_SUBBATCH=0 turns grouping
    // off; with SQF_PAIR_PARTS=0 it is the widening bound P (default 10%) for
    // merging width-sorted neighbours into one re-padded batch.
    const char* e = std::getenv("SQF_PAIR_SUBBATCH");
    pair_sub_ = e ? std::max(0, std::atoi(e)) : 10;
    if (dtype_ == SFK_F32 || cfg_.get_real("dropout") != 0.0) pair_sub_ = 0;
    // SQF_PAIR_PARTS (default 1): the sub-batches of a pass stay unpadded
    // parts (MiniBatch::parts; embedding and attention run per part, every
    // row-wise kernel once over all rows), so any widths can share a pass
    // and the SQF_PAIR_SUBBATCH widening bound does not apply; 0 merges
    // width-sorted neighbours within that bound into one re-padded batch.
    const char* pp = std::getenv("SQF_PAIR_PARTS");
    pair_parts_ = !(pp && std::atoi(pp) == 0);
    // SQF_PAIR_GROUP: sub-batches per pass (default 6 with parts -- an
    // update of 16 runs as 6 + 6 + 4 -- and 2 merged; C4 with the
    // column-fastest GEMM tile order measured 6 >= 8 > 4 > 3 > 16)
    const char* g = std::getenv("SQF_PAIR_GROUP");
    pair_group_ = std::min(g ? std::max(1, std::atoi(g)) : pair_parts_ ? 6 : 2, DeviceBatch::kMaxParts);
    // SQF_PAIR_BALANCE (default 1): passes of near-equal size (16 at 6 ->
    // 6 + 5 + 5 instead of 6 + 6 + 4; measured +0.8%)
    const char* bg = std::getenv("SQF_PAIR_BALANCE");
    balance_groups_ = !(bg && std::atoi(bg) == 0);
  }
  cuda_check(cudaEventCreateWithFlags(&ev_upload_, cudaEventDisableTiming), "event");
  for (auto& e : fwd_done_) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  for (auto& e : main_done_) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  cuda_check(cudaEventCreate(&ev0_), "event");
  for (auto& e : arena_free_) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  cuda_check(cudaEventCreate(&ev1_), "event");
  cuda_check(cudaMalloc(&master_, size_t(n_) * 4), "master");
  if (dtype_ == SFK_F32) {
    compute_ = master_;
  } else {
    cuda_check(cudaMalloc(&compute_, size_t(n_) * 2), "shadow");
  }
  // Every upload/clear below is ordered on stream_ (a non-blocking stream
  // does not order against the legacy stream, and a pageable cudaMemcpy H2D
  // may return before its DMA lands), then joined once at the end of init.
  for (int i = 0; i < 2 * local_; ++i) {
    void* g = nullptr;
    cuda_check(cudaMalloc(&g, size_t(n_) * esize()), "grads");
    cuda_check(cudaMemsetAsync(g, 0, size_t(n_) * esize(), stream_), "grads");
    grads_.push_back(g);
  }
  // optimizer ranges (~8M elements, 256-aligned) and their events
  {
    const char* e = std::getenv("SQF_ADAM_OVERLAP");
    adam_overlap_ = !(e && std::atoi(e) == 0);
    const int64_t chunk = int64_t(8) << 20;
    for (int64_t off = 0; off < n_; off += chunk) adam_ranges_.emplace_back(off, std::min(chunk, n_ - off));
    adam_range_ev_.resize(adam_ranges_.size());
    for (auto& ev : adam_range_ev_) cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
    adam_range_wait_.assign(adam_ranges_.size(), 0);
    for (auto& ev : adam_done_) cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&ev_checked_, cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreate(&ev_flush_), "event");
  }
  const std::vector<float> pe = model_->position_table();
  if (!pe.empty()) {
    cuda_check(cudaMalloc(&pe_, pe.size() * 4), "pe");
    cuda_check(cudaMemcpyAsync(pe_, pe.data(), pe.size() * 4, cudaMemcpyHostToDevice, stream_), "pe upload");
    cuda_check(cudaStreamSynchronize(stream_), "pe upload");
    set_model_position_table(*model_, pe_);
  }
  cuda_check(cudaMalloc(&stats_dev_, 4 * sizeof(double)), "stats");
  cuda_check(cudaMalloc(&flag_dev_, 16), "flag");
  cuda_check(cudaMalloc(&counters_, size_t(kCounters) * 4), "counters");
  {
    int sms = sfk_num_sms();
    if (sms <= 0) sms = 148;
    gemm_ws_floats_ = int64_t(sms) * 2 * 128 * 256;
    // [main | side | forward-ahead] stream-K workspaces
    cuda_check(cudaMalloc(&gemm_ws_, size_t(gemm_ws_floats_) * 3 * 4), "gemm workspace");
  }
  cuda_check(cudaMemsetAsync(counters_, 0, size_t(kCounters) * 4, stream_), "counters");
  cuda_check(cudaMemsetAsync(flag_dev_, 0, 16, stream_), "flag");
  cuda_check(cudaMallocHost(&readback_host_, 64), "readback");
  push_params();
}

const LossScaler& Trainer::scaler() const {
  if (!scaler_) throw ConfigError("trainer: loss scaler exists only in fp16 mode");
  return *scaler_;
}

void Trainer::push_params() {
  join_optimizer();
  std::fill(adam_range_wait_.begin(), adam_range_wait_.end(), 0);
  std::vector<float> dev(static_cast<size_t>(n_));
  model_->to_device_order(model_->params(), dev);
  // on stream_, so the shadow cast in rebroadcast() reads the uploaded master
  cuda_check(cudaMemcpyAsync(master_, dev.data(), size_t(n_) * 4, cudaMemcpyHostToDevice, stream_), "params upload");
  rebroadcast();
}

void Trainer::join_optimizer() {
  if (side_) cuda_check(cudaStreamSynchronize(side_), "optimizer join");
}

float Trainer::flush_ms() {
  for (int k = 0; k < 2; ++k)
    if (adam_pending_[k]) cuda_check(cudaStreamWaitEvent(stream_, adam_done_[k], 0), "stream wait");
  cuda_check(cudaEventRecord(ev_flush_, stream_), "event");
  cuda_check(cudaEventSynchronize(ev_flush_), "flush");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ev1_, ev_flush_);
  return ms;
}

void Trainer::param_wait(int64_t offset, int64_t numel, cudaStream_t s) {
  // a parameter may straddle optimizer ranges (the 32k x 1024 embeddings span
  // four): wait for every range that holds one of its elements
  if (numel <= 0) return;
  const int64_t chunk = int64_t(8) << 20;
  const size_t r0 = size_t(offset / chunk), r1 = size_t((offset + numel - 1) / chunk);
  for (size_t r = r0; r <= r1 && r < adam_range_wait_.size(); ++r)
    if (adam_range_wait_[r]) {
      cuda_check(cudaStreamWaitEvent(s, adam_range_ev_[r], 0), "stream wait");
      adam_range_wait_[r] = 0;
    }
}

void Trainer::rebroadcast() {
  join_optimizer();
  // trainer.cpp:149-156: replicas = quantised master; every rank holds the same
  // master (identical reduced grads -> identical updates), so no traffic
  if (compute_ != master_) sfk_check(sfk_cast(master_, compute_, dtype_, n_, stream_), "rebroadcast");
  cuda_check(cudaStreamSynchronize(stream_), "rebroadcast sync");
}

void Trainer::pull_params() {
  join_optimizer();
  std::vector<float> dev(static_cast<size_t>(n_));
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  cuda_check(cudaMemcpyAsync(dev.data(), master_, size_t(n_) * 4, cudaMemcpyDeviceToHost, stream_), "params download");
  cuda_check(cudaStreamSynchronize(stream_), "params download");
  model_->to_canonical_order(dev, model_->params());
}

std::vector<float> Trainer::reduced_grads() {
  join_optimizer();
  void* g0 = grads_[size_t(last_gset_ * local_)];
  std::vector<float> devf(static_cast<size_t>(n_));
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  if (dtype_ == SFK_F32) {
    cuda_check(cudaMemcpyAsync(devf.data(), g0, size_t(n_) * 4, cudaMemcpyDeviceToHost, stream_), "grads download");
    cuda_check(cudaStreamSynchronize(stream_), "grads download");
  } else {
    float* tmp = nullptr;
    cuda_check(cudaMalloc(&tmp, size_t(n_) * 4), "grads tmp");
    sfk_check(sfk_convert(dtype_, g0, SFK_F32, tmp, n_, stream_), "grads convert");
    cuda_check(cudaStreamSynchronize(stream_), "sync");
    cuda_check(cudaMemcpyAsync(devf.data(), tmp, size_t(n_) * 4, cudaMemcpyDeviceToHost, stream_), "grads download");
    cuda_check(cudaStreamSynchronize(stream_), "grads download");
    cudaFree(tmp);
  }
  std::vector<float> out(static_cast<size_t>(n_));
  model_->to_canonical_order(devf, out);
  return out;
}

void Trainer::restore_progress(int64_t step, int epoch, int cursor) {
  if (step < 0 || epoch < 1 || cursor < 0 || cursor > int(plan_.batches.size()))
    throw IntegrityError("trainer: restored progress out of range");
  step_ = step;
  epoch_ = epoch;
  pos_ = cursor;
  order_ = plan_.batches.empty() ? std::vector<int>{} : shuffle_epoch(plan_, epoch_);
}

void Trainer::restore_scaler(double scale, int64_t successes) {
  if (!scaler_) throw IntegrityError("trainer: scaler state present but fp16 is off");
  scaler_->restore(scale, successes);
}

std::optional<MiniBatch> Trainer::next_batch() {
  // trainer.cpp:173-184
  if (plan_.batches.empty()) return std::nullopt;
  if (pos_ >= int(order_.size())) {
    if (epoch_ >= max_epochs_) return std::nullopt;
    ++epoch_;
    order_ = shuffle_epoch(plan_, epoch_);
    pos_ = 0;
  }
  const std::vector<int>& members = plan_.batches[size_t(order_[size_t(pos_)])];
  ++pos_;
  return make_minibatch(task_->train_pairs(), members);
}

Trainer::Prefetch Trainer::plan_deal(int epoch, int pos, std::vector<int> order) const {
  // next_batch() (trainer.cpp:173-184) on a private copy of the cursor
  Prefetch p;
  p.epoch0 = epoch;
  p.pos0 = pos;
  const auto& pairs = task_->train_pairs();
  auto next = [&]() -> std::optional<MiniBatch> {
    if (plan_.batches.empty()) return std::nullopt;
    if (pos >= int(order.size())) {
      if (epoch >= max_epochs_) return std::nullopt;
      ++epoch;
      order = shuffle_epoch(plan_, epoch);
      pos = 0;
    }
    const std::vector<int>& members = plan_.batches[size_t(order[size_t(pos)])];
    ++pos;
    return make_minibatch(pairs, members);
  };
  p.sub.resize(size_t(workers_));
  for (int w = 0; w < workers_; ++w)
    for (int a = 0; a < accum_; ++a) {
      std::optional<MiniBatch> b = next();
      if (!b) {
        if (w == 0 && a == 0) {
          p.exhausted = true;
          return p;
        }
        p.sub[size_t(w)].push_back(MiniBatch{});
      } else {
        p.sub[size_t(w)].push_back(std::move(*b));
      }
    }
  p.epoch1 = epoch;
  p.pos1 = pos;
  p.order1 = std::move(order);
  pack_local(p.sub, p.packs, p.which);
  return p;
}

namespace {
// Packed batches of one update as one: their rows in order, every row
// right-padded to the widest member (make_minibatch's layout,
// data.cpp:172-219); each row's ids, lengths and corpus index are unchanged.
MiniBatch merge_minibatches(const std::vector<const MiniBatch*>& parts) {
  MiniBatch m;
  for (const MiniBatch* x : parts) {
    m.rows += x->rows;
    m.src_width = std::max(m.src_width, x->src_width);
    m.tgt_width = std::max(m.tgt_width, x->tgt_width);
  }
  const size_t S = size_t(m.src_width), T = size_t(m.tgt_width);
  m.source.assign(size_t(m.rows) * S, kPad);
  m.target_in.assign(size_t(m.rows) * T, kPad);
  m.target_out.assign(size_t(m.rows) * T, kPad);
  size_t r = 0;
  for (const MiniBatch* x : parts) {
    for (int i = 0; i < x->rows; ++i, ++r) {
      const size_t s0 = size_t(i) * size_t(x->src_width), t0 = size_t(i) * size_t(x->tgt_width);
      std::copy_n(x->source.begin() + ptrdiff_t(s0), x->src_width, m.source.begin() + ptrdiff_t(r * S));
      std::copy_n(x->target_in.begin() + ptrdiff_t(t0), x->tgt_width, m.target_in.begin() + ptrdiff_t(r * T));
      std::copy_n(x->target_out.begin() + ptrdiff_t(t0), x->tgt_width, m.target_out.begin() + ptrdiff_t(r * T));
    }
    m.src_lens.insert(m.src_lens.end(), x->src_lens.begin(), x->src_lens.end());
    m.tgt_lens.insert(m.tgt_lens.end(), x->tgt_lens.begin(), x->tgt_lens.end());
    m.members.insert(m.members.end(), x->members.begin(), x->members.end());
    m.ntokens += x->ntokens;
  }
  return m;
}
// The same as parts of one pass without re-padding: id arrays concatenated
// as they are, each part keeping its own widths (MiniBatch::parts); the model
// runs embedding and attention per part, everything row-wise over all rows.
MiniBatch join_minibatches(const std::vector<const MiniBatch*>& parts) {
  MiniBatch m;
  for (const MiniBatch* x : parts) {
    m.rows += x->rows;
    m.src_width = std::max(m.src_width, x->src_width);
    m.tgt_width = std::max(m.tgt_width, x->tgt_width);
    m.source.insert(m.source.end(), x->source.begin(), x->source.end());
    m.target_in.insert(m.target_in.end(), x->target_in.begin(), x->target_in.end());
    m.target_out.insert(m.target_out.end(), x->target_out.begin(), x->target_out.end());
    m.src_lens.insert(m.src_lens.end(), x->src_lens.begin(), x->src_lens.end());
    m.tgt_lens.insert(m.tgt_lens.end(), x->tgt_lens.begin(), x->tgt_lens.end());
    m.members.insert(m.members.end(), x->members.begin(), x->members.end());
    m.ntokens += x->ntokens;
    m.parts.push_back({x->rows, x->src_width, x->tgt_width});
  }
  return m;
}
}  // namespace

void Trainer::pack_local(const std::vector<std::vector<MiniBatch>>& sub, std::vector<PackedBatch>& packs,
                         std::vector<std::pair<int, int>>& which) const {
  packs.clear();
  which.clear();
  for (int lw = 0; lw < local_; ++lw) {
    const int w = rank_ * local_ + lw;
    std::vector<int> idx;
    for (int a = 0; a < accum_; ++a)
      if (sub[size_t(w)][size_t(a)].rows > 0) idx.push_back(a);
    if (pair_sub_ <= 0 || idx.size() < 2) {
      for (int a : idx) {
        packs.push_back(PackedBatch::pack(sub[size_t(w)][size_t(a)]));
        which.emplace_back(lw, a);
      }
      continue;
    }
    // neighbours in width order (least re-padding) pair when the wider one
    // is at most pair_sub_ % wider; the rest run alone
    auto width = [&](int a) {
      const MiniBatch& b = sub[size_t(w)][size_t(a)];
      return std::max(b.src_width, b.tgt_width);
    };
    auto key = [&](int a) {
      const MiniBatch& b = sub[size_t(w)][size_t(a)];
      return std::make_tuple(width(a), b.src_width, b.tgt_width, a);
    };
    std::sort(idx.begin(), idx.end(), [&](int x, int y) { return key(x) < key(y); });
    // parts mode: as many passes as groups of pair_group_ need, sizes
    // balanced (16 at 6 -> 6 + 5 + 5); merged mode: greedy groups
    const int npass = (int(idx.size()) + pair_group_ - 1) / pair_group_;
    int pass = 0;
    for (size_t k = 0; k < idx.size(); ++pass) {
      const int cap = !pair_parts_ || !balance_groups_ ? pair_group_
                      : int(idx.size()) / npass + (pass < int(idx.size()) % npass ? 1 : 0);
      std::vector<const MiniBatch*> group{&sub[size_t(w)][size_t(idx[k])]};
      size_t j = k + 1;
      for (; j < idx.size() && int(group.size()) < cap &&
             (pair_parts_ || int64_t(width(idx[j])) * 100 <= int64_t(width(idx[k])) * (100 + pair_sub_));
           ++j)
        group.push_back(&sub[size_t(w)][size_t(idx[j])]);
      packs.push_back(PackedBatch::pack(group.size() == 1 ? *group[0]
                                        : pair_parts_ ? join_minibatches(group)
                                                      : merge_minibatches(group)));
      which.emplace_back(lw, idx[k]);
      k = j;
    }
  }
}

std::optional<StepStats> Trainer::train_one() {
  if (!deal_) {
    std::optional<MiniBatch> b = next_batch();
    if (!b) return std::nullopt;
    return train_step(split_batch(task_->train_pairs(), *b, workers_, accum_));
  }
  // deal: W*A consecutive per-replica batches of the shuffled plan (fairseq
  // semantics); replayable on the reference through its train_step
  Prefetch p;
  bool have = false;
  if (prefetch_.valid()) {
    p = prefetch_.get();
    have = p.epoch0 == epoch_ && p.pos0 == pos_;
  }
  if (!have) p = plan_deal(epoch_, pos_, order_);
  if (p.exhausted) return std::nullopt;
  epoch_ = p.epoch1;
  pos_ = p.pos1;
  order_ = std::move(p.order1);
  return run_step(p.sub, p.packs, p.which);
}

void Trainer::upload(const std::vector<PackedBatch>& packs, std::vector<DeviceBatch>& out) {
  size_t total = 0;
  for (const auto& p : packs) total += p.blob.size();
  h2d_bytes_ = int64_t(total) * 4;
  if (total == 0) return;
  if (total > blob_host_cap_) {
    cudaFreeHost(blob_host_);
    blob_host_cap_ = total * 2;
    cuda_check(cudaMallocHost(&blob_host_, blob_host_cap_ * 4), "pinned staging");
  }
  if (total > blob_cap_) {
    cuda_check(cudaStreamSynchronize(stream_), "sync");
    cudaFree(blob_dev_);
    blob_cap_ = total * 2;
    cuda_check(cudaMalloc(&blob_dev_, blob_cap_ * 4), "batch blob");
  }
  size_t at = 0;
  out.clear();
  for (const auto& p : packs) {
    std::memcpy(blob_host_ + at, p.blob.data(), p.blob.size() * 4);
    out.push_back(p.bind(blob_dev_ + at));
    at += p.blob.size();
  }
  cuda_check(cudaMemcpyAsync(blob_dev_, blob_host_, total * 4, cudaMemcpyHostToDevice, stream_), "batch H2D");
}

void Trainer::allreduce_grads() {
  if (world_ <= 1) return;
  // bucketed all-reduce over NVLink, buckets in reverse device order (the
  // order backward completes them); same sum on every rank, so every rank
  // then runs the identical update (no rebroadcast traffic)
  coll_->group_start();
  for (const auto& b : buckets_)
    coll_->all_reduce(static_cast<char*>(grad_buf(0)) + b.start * esize(), size_t(b.end - b.start), dtype_, stream_);
  coll_->all_reduce(stats_dev_, 4, SQF_COLL_F64, stream_);
  coll_->group_end();
}

// ---------------------------------------------------------------- overlap
// The reference all-reduces after every replica finished backward
// (trainer.cpp:75-87, 246). Here the buckets (reverse device order, the order
// backward completes them) are all-reduced on a comm stream while the last
// sub-batch's backward is still running: the tape reports every parameter-
// gradient write, a bucket is issued once all of its planned writes are
// enqueued, always in bucket order so every rank issues the identical NCCL
// sequence. The comm stream waits on events of both compute streams taken at
// issue time, which covers every earlier write to that bucket.
cudaEvent_t Trainer::ovl_event() {
  if (ovl_next_event_ == ovl_events_.size()) {
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event create");
    ovl_events_.push_back(e);
  }
  return ovl_events_[ovl_next_event_++];
}


// every bucket a gradient write [offset, offset + numel) touches (a stacked
// parameter group may span several buckets); buckets tile the flat vector
template <typename F>
void Trainer::for_buckets(int64_t offset, int64_t numel, F f) const {
  auto it = std::upper_bound(bucket_index_.begin(), bucket_index_.end(), std::make_pair(offset, INT32_MAX));
  if (it != bucket_index_.begin()) --it;
  for (; it != bucket_index_.end() && it->first < offset + numel; ++it) {
    const GradientBucket& bk = buckets_[size_t(it->second)];
    if (bk.start < offset + numel && offset < bk.end) f(it->second);
  }
}

void Trainer::ovl_begin(const DeviceTape& tape) {
  ovl_remaining_.assign(buckets_.size(), 0);
  for (const auto& w : tape.planned_grad_writes())
    for_buckets(w.first, w.second, [&](int b) { ++ovl_remaining_[size_t(b)]; });
  ovl_next_ = 0;
  ovl_next_event_ = 0;
  overlap_log_.clear();
  overlap_early_ = 0;
  while (ovl_next_ < int(buckets_.size()) && ovl_remaining_[size_t(ovl_next_)] == 0) ovl_issue(ovl_next_++);
}

void Trainer::ovl_on_write(int64_t offset, int64_t numel) {
  for_buckets(offset, numel, [&](int b) {
    if (--ovl_remaining_[size_t(b)] < 0) throw DeviceError("overlap: more gradient writes than planned");
  });
  while (ovl_next_ < int(buckets_.size()) && ovl_remaining_[size_t(ovl_next_)] == 0) {
    ovl_issue(ovl_next_++);
    ++overlap_early_;
  }
}

void Trainer::ovl_issue(int b) {
  cudaEvent_t em = ovl_event(), es = ovl_event();
  cuda_check(cudaEventRecord(em, stream_), "event record");
  cuda_check(cudaEventRecord(es, side_), "event record");
  cuda_check(cudaStreamWaitEvent(comm_stream_, em, 0), "stream wait");
  cuda_check(cudaStreamWaitEvent(comm_stream_, es, 0), "stream wait");
  const GradientBucket& bk = buckets_[size_t(b)];
  if (world_ > 1)
    coll_->all_reduce(static_cast<char*>(grad_buf(0)) + bk.start * esize(), size_t(bk.end - bk.start), dtype_,
                      comm_stream_);
  overlap_log_.push_back(b);
}

void Trainer::ovl_finish() {
  // anything the plan did not see completed (a node without a gradient)
  while (ovl_next_ < int(buckets_.size())) ovl_issue(ovl_next_++);
  cudaEvent_t em = ovl_event();
  cuda_check(cudaEventRecord(em, stream_), "event record");
  cuda_check(cudaStreamWaitEvent(comm_stream_, em, 0), "stream wait");
  if (world_ > 1) coll_->all_reduce(stats_dev_, 4, SQF_COLL_F64, comm_stream_);
  cudaEvent_t done = ovl_event();
  cuda_check(cudaEventRecord(done, comm_stream_), "event record");
  cuda_check(cudaStreamWaitEvent(stream_, done, 0), "stream wait");
}

StepStats Trainer::train_step(const std::vector<std::vector<MiniBatch>>& sub) {
  if (int(sub.size()) != workers_) throw ShapeError("train_step: need one sub-batch list per replica");
  for (const auto& l : sub)
    if (int(l.size()) != accum_) throw ShapeError("train_step: every replica takes exactly accum sub-batches");
  std::vector<PackedBatch> packs;
  std::vector<std::pair<int, int>> which;
  pack_local(sub, packs, which);
  return run_step(sub, packs, which);
}

StepStats Trainer::run_step(const std::vector<std::vector<MiniBatch>>& sub, std::vector<PackedBatch>& packs,
                            const std::vector<std::pair<int, int>>& which) {
  const double scale = fp16_ ? scaler_->scale() : 1.0;
  StepStats stats;
  stats.step = step_ + 1;
  if (fp16_) stats.scale = scale;
  for (const auto& l : sub)
    for (const auto& b : l) stats.ntokens += b.ntokens;  // == sum of active target rows
  if (stats.ntokens == 0) throw ShapeError("train_step: zero target tokens in the minibatch");

  // upload this rank's packed sub-batches in one copy
  std::vector<DeviceBatch> dev;
  cuda_check(cudaEventRecord(ev0_, stream_), "event");
  if (prof_ && prof_->concurrent) {
    prof_->spans.clear();
    prof_->mark_base(stream_);
  }
  upload(packs, dev);
  cuda_check(cudaMemsetAsync(stats_dev_, 0, 4 * sizeof(double), stream_), "stats zero");
  // this step's gradient set (and its overflow flag) was last read by the
  // update two steps ago; the previous step's update may still be running on
  // the side stream and reads the other set's flag, so clearing this one is safe
  if (adam_pending_[gset_]) {
    cuda_check(cudaStreamWaitEvent(stream_, adam_done_[gset_], 0), "stream wait");
    adam_pending_[gset_] = false;
  }
  int32_t* flag_d = flag_dev_ + gset_;
  cuda_check(cudaMemsetAsync(flag_d, 0, 4, stream_), "flag zero");
  for (int lw = 0; lw < local_; ++lw)
    cuda_check(cudaMemsetAsync(grad_buf(lw), 0, size_t(n_) * esize(), stream_), "grad zero");
  launches_ = 0;
  const bool overlap = overlap_ && local_ == 1 && (world_ > 1 || overlap_sim_) && !dev.empty();
  // Forward-ahead: sub-batch i+1's forward is enqueued on fwd_stream_ before
  // sub-batch i's backward, so the two run concurrently (the forward needs
  // only the weights, which do not change inside a step); the backward of
  // i+1 then continues on the main stream. Results are identical either way.
  const bool ahead = fwd_ahead_ && fwd_stream_ && (!prof_ || prof_->concurrent) && dev.size() > 1;
  cudaStream_t fs = ahead ? fwd_stream_ : stream_;
  if (ahead) {
    cuda_check(cudaEventRecord(ev_upload_, stream_), "event record");  // batch upload, zeroed grads
    cuda_check(cudaStreamWaitEvent(fs, ev_upload_, 0), "stream wait");
  }
  std::unique_ptr<DeviceTape> tapes[2];
  CriterionOutput outs[2];
  auto forward = [&](size_t i) {
    const int lw = which[i].first, a = which[i].second;
    const int w = rank_ * local_ + lw;
    model_->set_train_step(step_ * workers_ * accum_ + int64_t(w) * accum_ + a);
    const int k = int(i & 1);
    if (arena_busy_[k]) {
      // the arena's previous sub-batch: its side-stream work and (when the
      // forward runs on its own stream) its main-stream backward
      cuda_check(cudaStreamWaitEvent(fs, arena_free_[k], 0), "arena wait");
      if (ahead) cuda_check(cudaStreamWaitEvent(fs, main_done_[k], 0), "arena wait");
    }
    arena_[k].reset();
    tapes[k] = std::make_unique<DeviceTape>(arena_[k], DeviceParams{master_, compute_, grad_buf(lw), n_}, dtype_, fs);
    DeviceTape& tape = *tapes[k];
    tape.set_use_hook([this](int64_t off, int64_t n, cudaStream_t st) { param_wait(off, n, st); });
    tape.set_profiler(prof_.get());
    tape.set_counters(counters_, kCounters, &counter_cursor_);
    // a profiling pass serialises everything on the main stream so the
    // per-launch event windows measure each kernel alone (no concurrency)
    if (!prof_ || prof_->concurrent) tape.set_side_stream(side_, &evpool_);
    float* ws_fwd = ahead ? gemm_ws_ + 2 * gemm_ws_floats_ : gemm_ws_;
    tape.set_gemm_workspace(ws_fwd, gemm_ws_ + gemm_ws_floats_, gemm_ws_floats_);
    outs[k] = criterion_->compute(*model_, dev[i], tape);
    if (ahead) cuda_check(cudaEventRecord(fwd_done_[k], fs), "event record");
  };
  if (ahead) forward(0);
  for (size_t i = 0; i < dev.size(); ++i) {
    const int k = int(i & 1);
    if (!ahead) forward(i);
    else if (i + 1 < dev.size()) forward(i + 1);
    DeviceTape& tape = *tapes[k];
    if (ahead) {
      cuda_check(cudaStreamWaitEvent(stream_, fwd_done_[k], 0), "stream wait");
      tape.set_main_stream(stream_);
      tape.set_gemm_workspace(gemm_ws_, gemm_ws_ + gemm_ws_floats_, gemm_ws_floats_);
    }
    if (overlap && i + 1 == dev.size()) {
      ovl_begin(tape);
      tape.set_grad_hook([this](int64_t off, int64_t n, cudaStream_t) { ovl_on_write(off, n); });
    }
    // the loss-scale multiply is the backward seed (trainer.cpp:237-239)
    const bool last = i + 1 == dev.size();
    tape.backward(outs[k].loss_node, float(scale), stats_dev_, last);
    if (!last) {
      cuda_check(cudaEventRecord(arena_free_[k], side_), "event record");
      if (ahead) cuda_check(cudaEventRecord(main_done_[k], stream_), "event record");
      arena_busy_[k] = true;
    }
    launches_ += tape.launches();
    tapes[k].reset();
  }
  arena_busy_[0] = arena_busy_[1] = false;  // the last backward joined the side stream
  // in-process replicas fold in index order with re-rounding (trainer.cpp:75-87)
  for (int lw = 1; lw < local_; ++lw) {
    sfk_check(sfk_accumulate(dtype_, grad_buf(0), grad_buf(lw), n_, stream_), "replica fold");
    ++launches_;
  }
  if (overlap)
    ovl_finish();
  else
    allreduce_grads();
  if (prof_) prof_->begin(stream_);
  sfk_check(sfk_nonfinite(dtype_, grad_buf(0), n_, flag_d, stream_), "overflow check");
  ++launches_;

  const bool injected = fp16_ && injector_ && injector_(stats.step);
  const double lr = scheduler_->lr(stats.step);
  const int64_t t_before = optimizer_->step_count();
  // The update runs on the side stream in ~8M-element ranges, overlapped
  // with the next step's forward, which waits per range before it first reads
  // those parameters; the stats read-back below does not wait for it. (Under
  // the profiler, and with SQF_ADAM_OVERLAP=0, it stays on the main stream.)
  const bool adam_side = adam_overlap_ && side_ && (!prof_ || prof_->concurrent);
  if (!injected) {
    GradPrep prep;
    prep.scale = float(scale);
    prep.unscale = fp16_;
    prep.ntokens = float(stats.ntokens);
    // (SQF_ABLATE: results are garbage by design; never skip so the step
    // keeps its full shape)
    prep.skip = ablate_mask() ? nullptr : flag_d;
    cudaStream_t os = stream_;
    if (adam_side) {
      cuda_check(cudaEventRecord(ev_checked_, stream_), "event record");
      cuda_check(cudaStreamWaitEvent(side_, ev_checked_, 0), "stream wait");
      prep.ranges = &adam_ranges_;
      prep.range_done = &adam_range_ev_;
      os = side_;
    }
    optimizer_->apply(master_, compute_ == master_ ? nullptr : compute_, dtype_, grad_buf(0), dtype_, n_, lr, prep,
                      os);
    launches_ += adam_side ? int64_t(adam_ranges_.size()) : 1;
    if (adam_side) {
      std::fill(adam_range_wait_.begin(), adam_range_wait_.end(), 1);
      cuda_check(cudaEventRecord(adam_done_[gset_], side_), "event record");
      adam_pending_[gset_] = true;
    }
  }
  last_gset_ = gset_;
  if (adam_side) gset_ ^= 1;
  // overflow check + update: 2 B grad read (check) + 28 B/param update
  if (prof_) prof_->end(stream_, Profiler::Optim, 0, double(n_) * (esize() + (injected ? 0 : 16 + 2 * esize() + 8)));
  // the next deal-mode step's batches are prepared while this one runs
  if (deal_ && prefetch_on_ && !prefetch_.valid())
    prefetch_ = std::async(std::launch::async, [this, e = epoch_, p = pos_, o = order_] { return plan_deal(e, p, o); });
  char* rb = static_cast<char*>(readback_host_);
  cuda_check(cudaMemcpyAsync(rb, stats_dev_, 4 * sizeof(double), cudaMemcpyDeviceToHost, stream_), "stats D2H");
  cuda_check(cudaMemcpyAsync(rb + 32, flag_d, 4, cudaMemcpyDeviceToHost, stream_), "flag D2H");
  cuda_check(cudaEventRecord(ev1_, stream_), "event");
  cuda_check(cudaStreamSynchronize(stream_), "step sync");
  cudaEventElapsedTime(&last_ms_, ev0_, ev1_);
  if (prof_) prof_->collect();
  const double* st = reinterpret_cast<const double*>(rb);
  const int32_t flag = ablate_mask() ? 0 : *reinterpret_cast<const int32_t*>(rb + 32);
  stats.loss = st[0];
  stats.nll = st[1];
  stats.ncorrect = int64_t(st[3]);

  if (fp16_) {
    if (flag || injected) {
      if (!injected) optimizer_->set_step_count(t_before);  // device update was predicated off
      stats.skipped = true;
      scaler_->update(true);  // may raise DivergenceError at the floor
      return stats;
    }
  } else if (flag) {
    optimizer_->set_step_count(t_before);
    throw DivergenceError("optimizer: non-finite gradient");
  }
  stats.lr = lr;
  step_ = stats.step;
  if (fp16_) scaler_->update(false);
  return stats;
}

EvalStats Trainer::evaluate(const std::vector<SequencePair>& pairs) {
  // trainer.cpp:275-289: teacher-forced scoring on the fp32 master
  join_optimizer();
  EvalStats out;
  if (pairs.empty()) return out;
  EpochPlan plan = make_batches(pairs, cfg_.get_int("max_tokens"), std::nullopt, 0);
  cuda_check(cudaMemsetAsync(stats_dev_, 0, 4 * sizeof(double), stream_), "stats zero");
  for (const auto& members : plan.batches) {
    MiniBatch b = make_minibatch(pairs, members);
    std::vector<PackedBatch> packs{PackedBatch::pack(b)};
    std::vector<DeviceBatch> dev;
    upload(packs, dev);
    arena_[0].reset();
    DeviceTape tape(arena_[0], DeviceParams{master_, master_, nullptr, n_}, SFK_F32, stream_);
    tape.set_counters(counters_, kCounters, &counter_cursor_);
    CriterionOutput c = criterion_->compute(*model_, dev[0], tape);
    tape.finish(c.loss_node, stats_dev_);
    cuda_check(cudaStreamSynchronize(stream_), "eval sync");  // staging buffer reuse
  }
  double st[4];
  cuda_check(cudaMemcpyAsync(st, stats_dev_, sizeof st, cudaMemcpyDeviceToHost, stream_), "eval D2H");
  cuda_check(cudaStreamSynchronize(stream_), "eval D2H");
  out.loss = st[0];
  out.nll = st[1];
  out.ntokens = int64_t(st[2]);
  out.ncorrect = int64_t(st[3]);
  return out;
}

}  // namespace sqf

namespace sqf {

int64_t Trainer::logits_ld(int V) const { return dtype_ == SFK_F32 ? V : (int64_t(V) + 7) / 8 * 8; }

const float* Trainer::logits_as_f32(const void* logits, int64_t n) {
  // 16-bit decoding: widen the logits once on the device (arena scratch)
  if (dtype_ == SFK_F32) return static_cast<const float*>(logits);
  float* f = static_cast<float*>(arena_[0].alloc(size_t(n) * 4));
  sfk_check(sfk_convert(dtype_, logits, SFK_F32, f, n, stream_), "logits widen");
  return f;
}

std::vector<float> Trainer::last_position_logits(const MiniBatch& mb) {
  // reference generate.cpp:86-120 (recompute_logits): decode every row's full
  // prefix and keep the final position's logits; the decoder runs on the
  // device from the fp32 master, only R x V floats come back
  join_optimizer();
  const int V = model_->target_vocab();
  const int R = mb.rows, T = mb.tgt_width;
  std::vector<PackedBatch> packs{PackedBatch::pack(mb)};
  std::vector<DeviceBatch> dev;
  upload(packs, dev);
  arena_[0].reset();
  model_->set_inference(true);
  std::vector<float> out(size_t(R) * V);
  try {
    DeviceTape tape(arena_[0], DeviceParams{master_, compute_, nullptr, n_}, dtype_, stream_);
    tape.set_counters(counters_, kCounters, &counter_cursor_);
    const int lg = model_->forward_to_logits(tape, dev[0]);
    if (tape.rows(lg) != R * T || tape.cols(lg) != V) throw ShapeError("generation: logits shape");
    const int64_t ld = logits_ld(V);
    const float* f = logits_as_f32(tape.out(lg), int64_t(R) * T * ld);
    cuda_check(cudaMemcpy2DAsync(out.data(), size_t(V) * 4, f + size_t(T - 1) * ld, size_t(T) * ld * 4,
                                 size_t(V) * 4, R, cudaMemcpyDeviceToHost, stream_),
               "logits D2H");
    cuda_check(cudaDeviceSynchronize(), "generation sync");
  } catch (...) {
    model_->set_inference(false);
    throw;
  }
  model_->set_inference(false);
  return out;
}

}  // namespace sqf

namespace sqf {

void Trainer::inc_begin(const MiniBatch& src, const std::vector<int>& row_sentence, int cap) {
  // model.cpp:315-465 (forward_encoder + make_incremental_state): the encoder
  // and every layer's cross K/V once per batch, rows replicated per hypothesis
  join_optimizer();
  inc_.reset();
  const int R = int(row_sentence.size()), S = src.src_width;
  if (R < 1 || cap < 1 || S < 1) throw ShapeError("incremental state: empty");
  auto st = std::make_unique<IncState>();
  st->rows = R;
  st->src_width = S;
  st->cap = cap;
  st->layers = model_->decoder_layers();
  st->d = model_->model_dim();
  st->es = dtype_ == SFK_F32 ? 4 : 2;
  const size_t kv_row = size_t(2) * st->d * st->es, layer_bytes = size_t(R) * cap * kv_row;
  const size_t cross_row = size_t(S) * st->layers * kv_row;
  // both halves zeroed: the tensor-core attention loads whole key tiles and
  // masks positions >= k_len in the scores, so unwritten cache rows must
  // hold finite values (0 * NaN would poison P.V)
  for (auto& p : st->self) {
    cuda_check(cudaMalloc(&p, layer_bytes * st->layers), "kv cache");
    cuda_check(cudaMemsetAsync(p, 0, layer_bytes * st->layers, stream_), "kv cache zero");
  }
  cuda_check(cudaMalloc(&st->cross, cross_row * R), "cross cache");
  cuda_check(cudaMalloc(&st->idx, size_t(4) * R * 4), "decoder indices");

  MiniBatch mb;
  mb.rows = src.rows;
  mb.src_width = S;
  mb.tgt_width = 1;
  mb.source = src.source;
  mb.src_lens = src.src_lens;
  mb.target_in.assign(size_t(src.rows), kBos);
  mb.target_out.assign(size_t(src.rows), kPad);
  mb.tgt_lens.assign(size_t(src.rows), 1);
  std::vector<PackedBatch> packs{PackedBatch::pack(mb)};
  std::vector<DeviceBatch> dev;
  upload(packs, dev);
  arena_[0].reset();
  std::vector<int32_t> h(size_t(4) * R, 0);
  for (int r = 0; r < R; ++r) {
    h[size_t(2) * R + r] = std::max(1, src.src_lens.at(size_t(row_sentence[r])));  // empty rows: a pad key
    h[size_t(3) * R + r] = row_sentence[r];
  }
  cuda_check(cudaMemcpyAsync(st->idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice, stream_), "indices H2D");
  model_->set_inference(true);
  try {
    DeviceTape tape(arena_[0], DeviceParams{master_, compute_, nullptr, n_}, dtype_, stream_);
    tape.set_counters(counters_, kCounters, &counter_cursor_);
    const int ckv = model_->encode_cross_kv(tape, dev[0]);
    sfk_check(sfk_gather_rows(tape.out(ckv), st->cross, st->idx + size_t(3) * R, R, int64_t(cross_row),
                              int64_t(cross_row), 1,
                              int64_t(cross_row) * R, stream_),
              "cross cache gather");
    cuda_check(cudaStreamSynchronize(stream_), "incremental state sync");
  } catch (...) {
    model_->set_inference(false);
    throw;
  }
  model_->set_inference(false);
  inc_ = std::move(st);
}

void Trainer::inc_run(const std::vector<int>& last, int pos, const std::function<void(DeviceTape&, int)>& consume) {
  if (!inc_) throw ConfigError("incremental decoding: no state (inc_begin first)");
  IncState& st = *inc_;
  const int R = st.rows;
  if (int(last.size()) != R) throw ShapeError("incremental decoding: one token per row");
  std::vector<int32_t> h(size_t(2) * R);
  for (int r = 0; r < R; ++r) {
    h[size_t(r)] = last[size_t(r)];
    h[size_t(R) + r] = pos + 1;
  }
  cuda_check(cudaMemcpyAsync(st.idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice, stream_), "step H2D");
  arena_[0].reset();
  model_->set_inference(true);
  try {
    DeviceTape tape(arena_[0], DeviceParams{master_, compute_, nullptr, n_}, dtype_, stream_);
    tape.set_counters(counters_, kCounters, &counter_cursor_);
    // forced stream-K on these M = rows GEMMs was measured 6.5x slower
    // end to end (big fp16 beam 4: 27.9 vs 182 sentences/s): plain tiles
    st.filled = std::max(st.filled, pos + 1);
    const int lg = model_->decode_step(tape, st.idx, R, pos, st.self[st.cur], st.cap, st.cross, st.src_width,
                                       st.idx + R, st.idx + size_t(2) * R);
    consume(tape, lg);
    cuda_check(cudaStreamSynchronize(stream_), "step sync");
  } catch (...) {
    model_->set_inference(false);
    throw;
  }
  model_->set_inference(false);
}

std::vector<float> Trainer::inc_step(const std::vector<int>& last, int pos) {
  const int V = model_->target_vocab();
  std::vector<float> out(last.size() * size_t(V));
  inc_run(last, pos, [&](DeviceTape& tape, int lg) {
    const int64_t ld = logits_ld(V), R = int64_t(last.size());
    const float* f = logits_as_f32(tape.out(lg), R * ld);
    cuda_check(cudaMemcpy2DAsync(out.data(), size_t(V) * 4, f, size_t(ld) * 4, size_t(V) * 4, size_t(R),
                                 cudaMemcpyDeviceToHost, stream_),
               "step logits D2H");
  });
  return out;
}

Trainer::BeamCands Trainer::inc_step_topk(const std::vector<int>& last, int pos, const std::vector<double>& cum,
                                          int kk) {
  if (!inc_) throw ConfigError("incremental decoding: no state (inc_begin first)");
  IncState& st = *inc_;
  const int R = st.rows, V = model_->target_vocab();
  kk = std::min(kk, V);
  const bool raw = cum.empty();
  if (!raw && int(cum.size()) != R) throw ShapeError("incremental decoding: one cumulative score per row");
  if (!st.cum) cuda_check(cudaMalloc(&st.cum, size_t(R) * 8), "beam cum");
  if (st.cands_kk < kk) {
    cudaFree(st.cands);
    st.cands = nullptr;
    cuda_check(cudaMalloc(&st.cands, size_t(R) * (2 + 2 * size_t(kk)) * 4), "beam candidates");
    st.cands_kk = kk;
  }
  if (!raw) cuda_check(cudaMemcpyAsync(st.cum, cum.data(), size_t(R) * 8, cudaMemcpyHostToDevice, stream_), "cum H2D");
  BeamCands out;
  out.kk = kk;
  out.lse.resize(size_t(R));
  out.eos_lp.resize(size_t(R));
  out.tok.resize(size_t(R) * kk);
  out.lp.resize(size_t(R) * kk);
  float* lse = static_cast<float*>(st.cands);
  float* eos_lp = lse + R;
  int32_t* tok = reinterpret_cast<int32_t*>(eos_lp + R);
  float* lp = reinterpret_cast<float*>(tok + size_t(R) * kk);
  std::vector<uint32_t> host(size_t(R) * (2 + 2 * size_t(kk)));
  inc_run(last, pos, [&](DeviceTape& tape, int lg) {
    sfk_check(sfk_beam_topk(dtype_, tape.out(lg), logits_ld(V), R, V, raw ? nullptr : st.cum, kk, kEos, lse, eos_lp,
                            tok, lp,
                            stream_),
              "beam_topk");
    // lse | eos_lp | tok | lp are contiguous: one read-back per position
    cuda_check(cudaMemcpyAsync(host.data(), lse, host.size() * 4, cudaMemcpyDeviceToHost, stream_), "candidates D2H");
  });
  std::memcpy(out.lse.data(), host.data(), size_t(R) * 4);
  std::memcpy(out.eos_lp.data(), host.data() + R, size_t(R) * 4);
  std::memcpy(out.tok.data(), host.data() + 2 * size_t(R), size_t(R) * kk * 4);
  std::memcpy(out.lp.data(), host.data() + 2 * size_t(R) + size_t(R) * kk, size_t(R) * kk * 4);
  return out;
}

void Trainer::inc_reorder(const std::vector<int>& order) {
  // model.cpp:540-557: new row r = old row order[r], every layer's K/V
  if (!inc_) throw ConfigError("incremental decoding: no state (inc_begin first)");
  IncState& st = *inc_;
  const int R = st.rows;
  if (int(order.size()) != R) throw ShapeError("reorder: one source row per row");
  std::vector<int32_t> h(order.begin(), order.end());
  for (int v : h)
    if (v < 0 || v >= R) throw BoundsError("reorder: row index out of range");
  cuda_check(cudaMemcpyAsync(st.idx + size_t(3) * R, h.data(), h.size() * 4, cudaMemcpyHostToDevice, stream_),
             "order H2D");
  const int64_t row = int64_t(st.cap) * 2 * st.d * st.es;
  sfk_check(sfk_gather_rows(st.self[st.cur], st.self[st.cur ^ 1], st.idx + size_t(3) * R, R, row,
                            int64_t(st.filled) * 2 * st.d * st.es, st.layers,
                            row * R, stream_),
            "kv cache reorder");
  st.cur ^= 1;
}

void Trainer::inc_end() { inc_.reset(); }

}  // namespace sqf

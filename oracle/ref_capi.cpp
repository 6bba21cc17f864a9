#include <algorithm>
#include <cmath>
// TEST INFRASTRUCTURE ONLY — never linked into, loaded by or called from the
// product path. This file is a thin C-ABI shim over the *unmodified* C++
// reference (seqforge, /root/reference/proj) so Python tests can use the
// reference itself as the parity oracle. It is compiled together with the
// reference's own sources by oracle/Makefile into oracle/_ref/libseqforge_ref.so.
//
// Every entry point forwards to the reference's public API; the only logic
// here is marshalling (flat arrays <-> SequencePair/MiniBatch) and mapping
// the reference's exception taxonomy (common.hpp:11-34) onto status codes.
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "seqforge/checkpoint.hpp"
#include "seqforge/simulator.hpp"
#include "seqforge/common.hpp"
#include "seqforge/criterions.hpp"
#include "seqforge/data.hpp"
#include "seqforge/fp16.hpp"
#include "seqforge/generate.hpp"
#include "seqforge/model.hpp"
#include "seqforge/optim.hpp"
#include "seqforge/registry.hpp"
#include "seqforge/rng.hpp"
#include "seqforge/tape.hpp"
#include "seqforge/tasks.hpp"
#include "seqforge/trainer.hpp"

using namespace seqforge;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const ConfigError*>(&e)) return -1;
  if (dynamic_cast<const ShapeError*>(&e)) return -2;
  if (dynamic_cast<const BoundsError*>(&e)) return -3;
  if (dynamic_cast<const CapacityError*>(&e)) return -4;
  if (dynamic_cast<const IntegrityError*>(&e)) return -5;
  if (dynamic_cast<const DivergenceError*>(&e)) return -6;
  if (dynamic_cast<const RegistryError*>(&e)) return -7;
  if (dynamic_cast<const IoError*>(&e)) return -8;
  return -9;
}

#define GUARD(...)                      \
  try {                                 \
    __VA_ARGS__;                        \
    return 0;                           \
  } catch (const std::exception& e) {   \
    return fail(e);                     \
  }

// Named architectures used by BASELINE.json's configs, registered over the
// reference's pre-norm `transformer` through its public
// Registry::register_architecture (registry.cpp:76-94).
void register_bench_archs(Registry& r) {
  auto add = [&](const char* name, int64_t d, int64_t h, int64_t L, int64_t f) {
    ArchitectureDef a;
    a.name = name;
    a.base_model = "transformer";
    a.overrides = {{"d_model", d},   {"heads", h},          {"enc_layers", L},
                   {"dec_layers", L}, {"d_ffn", f},         {"max_positions", int64_t{256}},
                   {"share_embeddings", false}};
    r.register_architecture(std::move(a), "sqf-oracle");
  };
  add("transformer_base_defaults", 64, 4, 2, 128);
  add("transformer_iwslt_de_en", 512, 4, 6, 1024);
  add("transformer_wmt_en_de", 512, 8, 6, 2048);
  add("transformer_vaswani_wmt_en_de_big", 1024, 16, 6, 4096);
}

Registry& oracle_registry() {
  static Registry reg = [] {
    Registry r;
    register_builtins(r);
    register_bench_archs(r);
    return r;
  }();
  return reg;
}

Dictionary synthetic_dict(int vocab) {
  Dictionary d;
  for (int i = Dictionary::kNumReserved; i < vocab; ++i) d.add_symbol("w" + std::to_string(i), 1);
  return d;
}

struct Corpus {
  std::vector<SequencePair> pairs;
};

class MemTask : public TaskBase {
 public:
  MemTask(const Corpus& c, int sv, int tv)
      : pairs_(c.pairs), src_(synthetic_dict(sv)), tgt_(synthetic_dict(tv)) {}
  const Dictionary& source_dict() const override { return src_; }
  const Dictionary& target_dict() const override { return tgt_; }
  const std::vector<SequencePair>& train_pairs() const override { return pairs_; }

 private:
  std::vector<SequencePair> pairs_;
  Dictionary src_, tgt_;
};

struct TrainerBox {
  Config cfg;
  std::unique_ptr<Trainer> tr;
  std::vector<int64_t> inject;
};

struct StatsC {
  int64_t step;
  double loss;
  double nll;
  int64_t ntokens;
  int64_t ncorrect;
  double lr;
  int32_t skipped;
  int32_t _pad;
  double scale;
};

void fill(StatsC* o, const StepStats& s) {
  o->step = s.step;
  o->loss = s.loss;
  o->nll = s.nll;
  o->ntokens = s.ntokens;
  o->ncorrect = s.ncorrect;
  o->lr = s.lr;
  o->skipped = s.skipped ? 1 : 0;
  o->_pad = 0;
  o->scale = s.scale;
}

void copy_minibatch(const MiniBatch& b, int32_t* dims, int32_t* source, int32_t* target_in,
                    int32_t* target_out, int32_t* src_lens, int32_t* tgt_lens, int64_t* ntokens) {
  dims[0] = b.rows;
  dims[1] = b.src_width;
  dims[2] = b.tgt_width;
  if (source) std::memcpy(source, b.source.data(), b.source.size() * 4);
  if (target_in) std::memcpy(target_in, b.target_in.data(), b.target_in.size() * 4);
  if (target_out) std::memcpy(target_out, b.target_out.data(), b.target_out.size() * 4);
  if (src_lens) std::memcpy(src_lens, b.src_lens.data(), b.src_lens.size() * 4);
  if (tgt_lens) std::memcpy(tgt_lens, b.tgt_lens.data(), b.tgt_lens.size() * 4);
  if (ntokens) *ntokens = b.ntokens;
}

}  // namespace

extern "C" {

const char* sqfref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- numerics
float sqfref_quantize_fp16(float x) { return quantize_fp16(x); }
uint16_t sqfref_f32_to_f16_bits(float x) { return f32_to_f16_bits(x); }
float sqfref_f16_bits_to_f32(uint16_t h) { return f16_bits_to_f32(h); }
void sqfref_quantize_many(float* x, int64_t n) {
  for (int64_t i = 0; i < n; ++i) x[i] = quantize_fp16(x[i]);
}

void sqfref_rng_u64(uint64_t seed, uint64_t stream, uint64_t counter, int n, uint64_t* out) {
  RngStream r(seed, stream, counter);
  for (int i = 0; i < n; ++i) out[i] = r.next_u64();
}
void sqfref_rng_double(uint64_t seed, uint64_t stream, uint64_t counter, int n, double* out) {
  RngStream r(seed, stream, counter);
  for (int i = 0; i < n; ++i) out[i] = r.next_double();
}
void sqfref_rng_normal(uint64_t seed, uint64_t stream, uint64_t counter, int n, double* out) {
  RngStream r(seed, stream, counter);
  for (int i = 0; i < n; ++i) out[i] = r.next_normal();
}
void sqfref_rng_below(uint64_t seed, uint64_t stream, uint64_t counter, uint64_t bound, int n,
                      uint64_t* out) {
  RngStream r(seed, stream, counter);
  for (int i = 0; i < n; ++i) out[i] = r.next_below(bound);
}
void sqfref_positional_row(int pos, int d, float* out) { positional_row(pos, d, out); }

// ---------------------------------------------------------------- corpus / data
void* sqfref_corpus_create(int npairs, const int32_t* src_len, const int32_t* tgt_len,
                           const int32_t* src_ids, const int32_t* tgt_ids) {
  auto* c = new Corpus;
  c->pairs.resize(static_cast<size_t>(npairs));
  int64_t so = 0, to = 0;
  for (int i = 0; i < npairs; ++i) {
    auto& p = c->pairs[static_cast<size_t>(i)];
    p.source.assign(src_ids + so, src_ids + so + src_len[i]);
    p.target.assign(tgt_ids + to, tgt_ids + to + tgt_len[i]);
    p.corpus_index = i;
    so += src_len[i];
    to += tgt_len[i];
  }
  return c;
}
void sqfref_corpus_free(void* c) { delete static_cast<Corpus*>(c); }

// The synthetic WMT-shaped corpus of SURVEY §8(d) (the benchmark's input
// specification, not reference code) drawn from the reference's own RngStream,
// so the CPU reference arm never loads the product library: lengths
// clamp(round(exp(3.1 + 0.6 z)), 1, 200) and clamp(round(ls (1 + 0.1 z')), 1, 200),
// ids by inverse CDF of Zipf(s) over [4, V), eos appended. Two-pass like the
// product call: ids == NULL only reports the lengths and totals.
int sqfref_synthetic_corpus(int npairs, int src_vocab, int tgt_vocab, double zipf_s, uint64_t seed,
                            uint64_t stream, int32_t* src_len, int32_t* tgt_len, int32_t* src_ids, int32_t* tgt_ids,
                            int64_t* src_total, int64_t* tgt_total) {
  if (npairs < 0 || src_vocab <= 4 || tgt_vocab <= 4) return -1;
  auto cdf_of = [&](int vocab) {
    std::vector<double> c(static_cast<size_t>(vocab - 4));
    double run = 0.0;
    for (size_t k = 0; k < c.size(); ++k) c[k] = run += zipf_s > 0 ? std::pow(double(k + 1), -zipf_s) : 1.0;
    for (double& x : c) x /= run;
    return c;
  };
  const std::vector<double> sc = cdf_of(src_vocab), tc = cdf_of(tgt_vocab);
  RngStream rng(seed, stream);
  auto id_of = [&](const std::vector<double>& c) {
    const size_t k = size_t(std::upper_bound(c.begin(), c.end(), rng.next_double()) - c.begin());
    return int32_t(4 + std::min(k, c.size() - 1));
  };
  auto len_of = [](double x) { return int32_t(std::clamp(std::round(x), 1.0, 200.0)); };
  int64_t so = 0, to = 0;
  for (int i = 0; i < npairs; ++i) {
    const int32_t ls = len_of(std::exp(3.1 + 0.6 * rng.next_normal()));
    const int32_t lt = len_of(double(ls) * (1.0 + 0.1 * rng.next_normal()));
    src_len[i] = ls + 1;
    tgt_len[i] = lt + 1;
    for (int32_t j = 0; j < ls; ++j) {
      const int32_t t = id_of(sc);
      if (src_ids) src_ids[so + j] = t;
    }
    for (int32_t j = 0; j < lt; ++j) {
      const int32_t t = id_of(tc);
      if (tgt_ids) tgt_ids[to + j] = t;
    }
    if (src_ids) src_ids[so + ls] = 2;  // eos
    if (tgt_ids) tgt_ids[to + lt] = 2;
    so += ls + 1;
    to += lt + 1;
  }
  *src_total = so;
  *tgt_total = to;
  return 0;
}

// make_batches (data.cpp:115-161): returns batch count; sizes/members are
// written into caller buffers of capacity npairs.
int sqfref_make_batches(void* corpus, int64_t max_tokens, int max_sentences, uint64_t seed,
                        int32_t* nbatches, int32_t* sizes, int32_t* members) {
  GUARD({
    auto* c = static_cast<Corpus*>(corpus);
    EpochPlan p = make_batches(c->pairs, max_tokens,
                               max_sentences > 0 ? std::optional<int>(max_sentences) : std::nullopt,
                               seed);
    *nbatches = static_cast<int32_t>(p.batches.size());
    int64_t k = 0;
    for (size_t b = 0; b < p.batches.size(); ++b) {
      sizes[b] = static_cast<int32_t>(p.batches[b].size());
      for (int m : p.batches[b]) members[k++] = m;
    }
  })
}

// shuffle_epoch (data.cpp:163-170) for a plan with `nbatches` batches
int sqfref_shuffle_epoch(int nbatches, uint64_t seed, int epoch, int32_t* order) {
  GUARD({
    EpochPlan p;
    p.batches.resize(static_cast<size_t>(nbatches));
    p.shuffle_seed = seed;
    std::vector<int> o = shuffle_epoch(p, epoch);
    for (size_t i = 0; i < o.size(); ++i) order[i] = o[i];
  })
}

// make_minibatch (data.cpp:172-219); dims = {rows, src_width, tgt_width}
int sqfref_make_minibatch(void* corpus, const int32_t* members, int n, int32_t* dims,
                          int32_t* source, int32_t* target_in, int32_t* target_out,
                          int32_t* src_lens, int32_t* tgt_lens, int64_t* ntokens) {
  GUARD({
    auto* c = static_cast<Corpus*>(corpus);
    std::vector<int> m(members, members + n);
    MiniBatch b = make_minibatch(c->pairs, m);
    copy_minibatch(b, dims, source, target_in, target_out, src_lens, tgt_lens, ntokens);
  })
}

int sqfref_bucket_gradients(const int64_t* sizes, int n, int64_t threshold, int32_t* nbuckets,
                            int64_t* starts, int64_t* ends) {
  GUARD({
    std::vector<int64_t> s(sizes, sizes + n);
    auto b = bucket_gradients(s, threshold);
    *nbuckets = static_cast<int32_t>(b.size());
    for (size_t i = 0; i < b.size(); ++i) {
      starts[i] = b[i].start;
      ends[i] = b[i].end;
    }
  })
}

// ---------------------------------------------------------------- schedules / optimizer / scaler
int sqfref_inverse_sqrt(double base, int64_t warmup, double init, int64_t step, double* out) {
  GUARD({ *out = InverseSqrtSchedule(base, warmup, init).lr(step); })
}
int sqfref_cosine_restart(double base, double eta_min, int64_t period, double t_mult, int64_t step,
                          double* out) {
  GUARD({ *out = CosineRestartSchedule(base, eta_min, period, t_mult).lr(step); })
}

// Adam (optim.cpp:48-66): one apply with moments/step restored from the caller
int sqfref_adam(float* params, const float* grads, int64_t n, float* m, float* v, int64_t t,
                double lr, double b1, double b2, double eps) {
  GUARD({
    AdamOptimizer opt(n, b1, b2, eps);
    opt.load_state_blobs({{"adam.m", std::vector<float>(m, m + n)},
                          {"adam.v", std::vector<float>(v, v + n)}});
    opt.set_step_count(t);
    opt.apply(std::span<float>(params, static_cast<size_t>(n)),
              std::span<const float>(grads, static_cast<size_t>(n)), lr);
    auto blobs = opt.state_blobs();
    std::memcpy(m, blobs[0].second.data(), static_cast<size_t>(n) * 4);
    std::memcpy(v, blobs[1].second.data(), static_cast<size_t>(n) * 4);
  })
}

// LossScaler (trainer.cpp:21-48) driven by an overflow sequence; returns the
// index of the update that diverged in *diverged_at (-1 if none)
int sqfref_scaler_run(double init, int64_t window, double mn, double mx, const uint8_t* overflow,
                      int n, double* scales, int32_t* diverged_at) {
  GUARD({
    LossScaler s(init, window, mn, mx);
    *diverged_at = -1;
    for (int i = 0; i < n; ++i) {
      try {
        s.update(overflow[i] != 0);
      } catch (const DivergenceError&) {
        *diverged_at = i;
        return 0;
      }
      scales[i] = s.scale();
    }
  })
}

// ---------------------------------------------------------------- single tape ops
// softmax_xent (tape.cpp:151-168, 259-290, 481-502) with backward seeded by
// `seed` on active rows (tape.cpp:506-516).
int sqfref_xent(const float* logits, int rows, int vocab, const int32_t* gold,
                const uint8_t* active, float eps, int fp16, float seed, float* loss_rows,
                float* nll_rows, uint8_t* correct, float* dlogits) {
  GUARD({
    std::vector<float> none;
    Tape tape{std::span<const float>(none.data(), 0), fp16 ? DType::F16E : DType::F32};
    int l = tape.leaf(Tensor({rows, vocab}, std::vector<float>(logits, logits + int64_t(rows) * vocab)));
    int x = tape.softmax_xent(l, std::vector<int>(gold, gold + rows),
                              std::vector<uint8_t>(active, active + rows), eps);
    const TapeNode& n = tape.node(x);
    for (int r = 0; r < rows; ++r) {
      loss_rows[r] = n.out.data()[r];
      nll_rows[r] = n.nll[static_cast<size_t>(r)];
      correct[r] = n.correct[static_cast<size_t>(r)];
    }
    if (dlogits) {
      std::vector<float> pg;
      tape.backward(x, seed, pg);
      std::memcpy(dlogits, tape.node(l).grad.data(), sizeof(float) * size_t(rows) * vocab);
    }
  })
}

// layer_norm (tape.cpp:96-107, 211-222, 383-418): forward + backward_from(dy)
int sqfref_layer_norm(const float* x, int rows, int d, const float* gamma, const float* beta,
                      int fp16, const float* dy, float* y, float* dx, float* dgamma,
                      float* dbeta) {
  GUARD({
    std::vector<float> p(gamma, gamma + d);
    p.insert(p.end(), beta, beta + d);
    Tape tape{p, fp16 ? DType::F16E : DType::F32};
    int in = tape.leaf(Tensor({rows, d}, std::vector<float>(x, x + int64_t(rows) * d)));
    int o = tape.layer_norm(in, ParamRef{0, 1, d}, ParamRef{d, 1, d});
    std::memcpy(y, tape.out(o).data(), sizeof(float) * size_t(rows) * d);
    if (dy) {
      std::vector<float> pg(static_cast<size_t>(2 * d), 0.0f);
      Tensor g({rows, d}, std::vector<float>(dy, dy + int64_t(rows) * d));
      tape.backward_from(o, g, pg);
      std::memcpy(dx, tape.node(in).grad.data(), sizeof(float) * size_t(rows) * d);
      std::memcpy(dgamma, pg.data(), sizeof(float) * d);
      std::memcpy(dbeta, pg.data() + d, sizeof(float) * d);
    }
  })
}

// attention (tape.cpp:123-149, 229-258, 426-480)
int sqfref_attention(const float* q, int rq, const float* k, const float* v, int rk, int d,
                     int heads, const int32_t* key_base, const int32_t* key_len, int fp16,
                     const float* dout, float* out, float* dq, float* dk, float* dv) {
  GUARD({
    std::vector<float> none;
    Tape tape{std::span<const float>(none.data(), 0), fp16 ? DType::F16E : DType::F32};
    int iq = tape.leaf(Tensor({rq, d}, std::vector<float>(q, q + int64_t(rq) * d)));
    int ik = tape.leaf(Tensor({rk, d}, std::vector<float>(k, k + int64_t(rk) * d)));
    int iv = tape.leaf(Tensor({rk, d}, std::vector<float>(v, v + int64_t(rk) * d)));
    int o = tape.attention(iq, ik, iv, heads, std::vector<int>(key_base, key_base + rq),
                           std::vector<int>(key_len, key_len + rq));
    std::memcpy(out, tape.out(o).data(), sizeof(float) * size_t(rq) * d);
    if (dout) {
      std::vector<float> pg;
      Tensor g({rq, d}, std::vector<float>(dout, dout + int64_t(rq) * d));
      tape.backward_from(o, g, pg);
      std::memcpy(dq, tape.node(iq).grad.data(), sizeof(float) * size_t(rq) * d);
      std::memcpy(dk, tape.node(ik).grad.data(), sizeof(float) * size_t(rk) * d);
      std::memcpy(dv, tape.node(iv).grad.data(), sizeof(float) * size_t(rk) * d);
    }
  })
}

// matmul_nt (+ add_bias when bias != null), tape.cpp:46-67, 182-197, 324-358
int sqfref_linear(const float* x, int rows, int in_dim, const float* w, const float* bias,
                  int out_dim, int fp16, const float* dy, float* y, float* dx, float* dw,
                  float* db) {
  GUARD({
    std::vector<float> p(w, w + int64_t(out_dim) * in_dim);
    if (bias) p.insert(p.end(), bias, bias + out_dim);
    Tape tape{p, fp16 ? DType::F16E : DType::F32};
    int in = tape.leaf(Tensor({rows, in_dim}, std::vector<float>(x, x + int64_t(rows) * in_dim)));
    int o = tape.matmul_nt(in, ParamRef{0, out_dim, in_dim});
    if (bias) o = tape.add_bias(o, ParamRef{int64_t(out_dim) * in_dim, 1, out_dim});
    std::memcpy(y, tape.out(o).data(), sizeof(float) * size_t(rows) * out_dim);
    if (dy) {
      std::vector<float> pg(p.size(), 0.0f);
      Tensor g({rows, out_dim}, std::vector<float>(dy, dy + int64_t(rows) * out_dim));
      tape.backward_from(o, g, pg);
      std::memcpy(dx, tape.node(in).grad.data(), sizeof(float) * size_t(rows) * in_dim);
      std::memcpy(dw, pg.data(), sizeof(float) * size_t(out_dim) * in_dim);
      if (bias) std::memcpy(db, pg.data() + int64_t(out_dim) * in_dim, sizeof(float) * out_dim);
    }
  })
}

// ---------------------------------------------------------------- trainer
// arch + raw user overrides resolved exactly as Registry::resolve_architecture
// (registry.cpp:96-110); the task is the in-memory corpus (trainer.hpp:84-85).
void* sqfref_trainer_create(const char* arch, const char** keys, const char** vals, int n,
                            void* corpus, int src_vocab, int tgt_vocab) {
  try {
    std::vector<std::pair<std::string, std::string>> user;
    for (int i = 0; i < n; ++i) user.emplace_back(keys[i], vals[i]);
    auto box = std::make_unique<TrainerBox>();
    box->cfg = oracle_registry().resolve_architecture(arch, user);
    auto task = std::make_unique<MemTask>(*static_cast<Corpus*>(corpus), src_vocab, tgt_vocab);
    box->tr = std::make_unique<Trainer>(box->cfg, std::move(task), oracle_registry());
    return box.release();
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
void sqfref_trainer_free(void* h) { delete static_cast<TrainerBox*>(h); }

int sqfref_trainer_set_injector(void* h, const int64_t* steps, int n) {
  GUARD({
    auto* b = static_cast<TrainerBox*>(h);
    b->inject.assign(steps, steps + n);
    std::vector<int64_t> s = b->inject;
    b->tr->set_overflow_injector([s](int64_t step) {
      for (int64_t x : s)
        if (x == step) return true;
      return false;
    });
  })
}

// returns 1 when the data stream is exhausted (trainer.cpp:204-208)
int sqfref_trainer_train_one(void* h, StatsC* out) {
  try {
    auto st = static_cast<TrainerBox*>(h)->tr->train_one();
    if (!st) return 1;
    fill(out, *st);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// explicit dispatch (trainer.cpp:210-273): counts[w*A+a] members each
int sqfref_trainer_train_step(void* h, void* corpus, const int32_t* members, const int32_t* counts,
                              int workers, int accum, StatsC* out) {
  GUARD({
    auto* c = static_cast<Corpus*>(corpus);
    std::vector<std::vector<MiniBatch>> sub(static_cast<size_t>(workers));
    int64_t k = 0;
    for (int w = 0; w < workers; ++w)
      for (int a = 0; a < accum; ++a) {
        int cnt = counts[w * accum + a];
        std::vector<int> m(members + k, members + k + cnt);
        k += cnt;
        if (cnt == 0) {
          sub[static_cast<size_t>(w)].push_back(MiniBatch{});
        } else {
          sub[static_cast<size_t>(w)].push_back(make_minibatch(c->pairs, m));
        }
      }
    fill(out, static_cast<TrainerBox*>(h)->tr->train_step(sub));
  })
}

int64_t sqfref_trainer_num_params(void* h) { return static_cast<TrainerBox*>(h)->tr->model().num_params(); }
int sqfref_trainer_params(void* h, float* out) {
  GUARD({
    auto p = static_cast<TrainerBox*>(h)->tr->model().params();
    std::memcpy(out, p.data(), p.size() * 4);
  })
}
int sqfref_trainer_set_params(void* h, const float* in) {
  GUARD({
    auto* b = static_cast<TrainerBox*>(h);
    auto p = b->tr->model().params();
    std::memcpy(p.data(), in, p.size() * 4);
    b->tr->rebroadcast();
  })
}
int sqfref_trainer_replica_params(void* h, int w, float* out) {
  GUARD({
    auto p = static_cast<TrainerBox*>(h)->tr->replica(w).params();
    std::memcpy(out, p.data(), p.size() * 4);
  })
}
int sqfref_trainer_manifest_size(void* h) {
  return static_cast<int>(static_cast<TrainerBox*>(h)->tr->model().manifest().size());
}
int sqfref_trainer_manifest_entry(void* h, int i, char* name, int cap, int64_t* offset,
                                  int64_t* numel) {
  GUARD({
    const auto& e = static_cast<TrainerBox*>(h)->tr->model().manifest().at(static_cast<size_t>(i));
    std::snprintf(name, static_cast<size_t>(cap), "%s", e.name.c_str());
    *offset = e.offset;
    *numel = e.numel;
  })
}
int sqfref_trainer_adam_state(void* h, float* m, float* v, int64_t* t) {
  GUARD({
    auto& opt = static_cast<TrainerBox*>(h)->tr->optimizer();
    for (auto& [name, data] : opt.state_blobs()) {
      if (name == "adam.m") std::memcpy(m, data.data(), data.size() * 4);
      if (name == "adam.v") std::memcpy(v, data.data(), data.size() * 4);
    }
    *t = opt.step_count();
  })
}
int sqfref_trainer_scaler(void* h, double* scale, int64_t* good) {
  GUARD({
    const auto& s = static_cast<TrainerBox*>(h)->tr->scaler();
    *scale = s.scale();
    *good = s.successes();
  })
}
int sqfref_trainer_progress(void* h, int64_t* step, int32_t* epoch, int32_t* cursor,
                            int32_t* nbatches) {
  GUARD({
    auto* t = static_cast<TrainerBox*>(h)->tr.get();
    *step = t->step();
    *epoch = t->epoch();
    *cursor = t->cursor();
    *nbatches = t->batches_per_epoch();
  })
}
int sqfref_trainer_buckets(void* h, int32_t* n, int64_t* starts, int64_t* ends) {
  GUARD({
    const auto& b = static_cast<TrainerBox*>(h)->tr->buckets();
    *n = static_cast<int32_t>(b.size());
    if (starts)
      for (size_t i = 0; i < b.size(); ++i) {
        starts[i] = b[i].start;
        ends[i] = b[i].end;
      }
  })
}

// One sub-batch forward+backward on the (shadow of the) master parameters,
// restated from train_step's inner body (trainer.cpp:223-240) with the
// reference's own Tape/criterion: fills grad (caller-zeroed or accumulated).
int sqfref_trainer_subbatch_grad(void* h, void* corpus, const int32_t* members, int n, float seed,
                                 float* grad, StatsC* out) {
  GUARD({
    auto* b = static_cast<TrainerBox*>(h);
    auto* c = static_cast<Corpus*>(corpus);
    Trainer& t = *b->tr;
    std::unique_ptr<ModelBase> rep = t.model().clone();
    if (t.fp16()) {
      auto p = rep->params();
      for (float& x : p) x = quantize_fp16(x);
    }
    auto crit = oracle_registry().make_criterion(b->cfg.get_str("criterion"), b->cfg);
    MiniBatch mb = make_minibatch(c->pairs, std::vector<int>(members, members + n));
    Tape tape{rep->params(), t.fp16() ? DType::F16E : DType::F32};
    CriterionOutput co = crit->compute(*rep, mb, tape);
    tape.backward(co.loss_node, seed,
                  std::span<float>(grad, static_cast<size_t>(rep->num_params())));
    StepStats s;
    s.loss = co.loss;
    s.nll = co.nll;
    s.ntokens = co.ntokens;
    s.ncorrect = co.ncorrect;
    fill(out, s);
  })
}

// Trainer::evaluate (trainer.cpp:275-289) over a corpus
int sqfref_trainer_evaluate(void* h, void* corpus, double* loss, double* nll, int64_t* ntokens,
                            int64_t* ncorrect) {
  GUARD({
    EvalStats e = static_cast<TrainerBox*>(h)->tr->evaluate(static_cast<Corpus*>(corpus)->pairs);
    *loss = e.loss;
    *nll = e.nll;
    *ntokens = e.ntokens;
    *ncorrect = e.ncorrect;
  })
}

// ---------------------------------------------------------------- translation task
// the reference's TranslationTask (tasks.cpp:7-33) built from a resolved config;
// dumps "<src_vocab> <tgt_vocab> <npairs>\n" then one "src ids | tgt ids" line per pair
int sqfref_task_dump(const char* arch, const char** keys, const char** vals, int n, char* out, int64_t cap) {
  GUARD({
    std::vector<std::pair<std::string, std::string>> user;
    for (int i = 0; i < n; ++i) user.emplace_back(keys[i], vals[i]);
    Config cfg = oracle_registry().resolve_architecture(arch, user);
    TranslationTask task(cfg);
    std::string text = std::to_string(task.source_dict().size()) + " " + std::to_string(task.target_dict().size()) +
                       " " + std::to_string(task.train_pairs().size()) + "\n";
    for (const auto& p : task.train_pairs()) {
      for (int x : p.source) text += std::to_string(x) + " ";
      text += "|";
      for (int x : p.target) text += " " + std::to_string(x);
      text += "\n";
    }
    if (int64_t(text.size()) + 1 > cap) throw BoundsError("buffer");
    std::memcpy(out, text.c_str(), text.size() + 1);
  })
}

// ---------------------------------------------------------------- timeline model
// the reference's simulate_timeline + format_report on a scenario given as
// arrays (its text parser takes a std::istream, which must not be used here:
// under a Python process with numpy loaded first the iostream facets of the
// host libstdc++ differ from this library's)
int sqfref_simulate_timeline(int workers, int accum, int mode, const double* compute, const double* comm, int nb,
                             char* report, int cap) {
  GUARD({
    SimScenario sc;
    sc.workers = workers;
    sc.accum = accum;
    sc.mode = mode == 0 ? SyncMode::SerialSync : mode == 1 ? SyncMode::Overlap : SyncMode::OverlapAccum;
    for (int w = 0; w < workers; ++w) sc.compute.emplace_back(compute + int64_t(w) * accum, compute + int64_t(w + 1) * accum);
    sc.comm.assign(comm, comm + nb);
    const std::string text = format_report(simulate_timeline(sc));
    if (int(text.size()) + 1 > cap) throw BoundsError("buffer");
    std::memcpy(report, text.c_str(), text.size() + 1);
  })
}

// ---------------------------------------------------------------- checkpoints
// the reference's own writer (checkpoint.cpp:187-224) and raw reader (226-320)
int sqfref_trainer_save(void* h, const char* path) {
  GUARD(save_checkpoint(*static_cast<TrainerBox*>(h)->tr, path))
}
int sqfref_checkpoint_read(const char* path, int32_t* version, int64_t* nparams, float* params, int64_t* nopt,
                           float* opt) {
  GUARD({
    RawCheckpoint raw = read_checkpoint(path);
    *version = raw.version;
    *nparams = int64_t(raw.params.size());
    *nopt = int64_t(raw.opt.size());
    if (params) std::memcpy(params, raw.params.data(), raw.params.size() * 4);
    if (opt) std::memcpy(opt, raw.opt.data(), raw.opt.size() * 4);
  })
}
int sqfref_checkpoint_meta(const char* path, const char* key, char* out, int cap) {
  GUARD({
    RawCheckpoint raw = read_checkpoint(path);
    auto it = raw.meta.find(key);
    if (it == raw.meta.end()) throw IntegrityError(std::string("no key ") + key);
    if (int(it->second.size()) + 1 > cap) throw BoundsError("buffer");
    std::memcpy(out, it->second.c_str(), it->second.size() + 1);
  })
}

// ---------------------------------------------------------------- generation
// generate.hpp:46-90 on the trainer's model; mode 0 beam, 1 diverse, 2 sample
int sqfref_generate(void* h, int mode, const int32_t* source, const int32_t* src_lens, int rows, int src_width,
                    int beam, int max_len, int groups, int topk, double lenpen, double strength,
                    double temperature, uint64_t seed, const uint64_t* stream_ids, int no_cache, void** out) {
  GUARD({
    const auto& model = dynamic_cast<const TransformerModel&>(static_cast<TrainerBox*>(h)->tr->model());
    MiniBatch b;
    b.rows = rows;
    b.src_width = src_width;
    b.source.assign(source, source + static_cast<size_t>(rows) * src_width);
    b.src_lens.assign(src_lens, src_lens + rows);
    GenConfig g;
    g.beam = beam;
    g.max_len = max_len;
    g.diverse_groups = groups;
    g.topk = topk;
    g.lenpen = lenpen;
    g.diverse_strength = strength;
    g.temperature = temperature;
    g.seed = seed;
    g.no_cache = no_cache != 0;
    auto res = std::make_unique<std::vector<std::vector<Hypothesis>>>();
    if (mode == 0) {
      *res = beam_search(model, b, g);
    } else if (mode == 1) {
      *res = diverse_beam_search(model, b, g);
    } else {
      std::vector<uint64_t> ids;
      if (stream_ids) ids.assign(stream_ids, stream_ids + rows);
      for (Hypothesis& x : top_k_sample(model, b, g, ids)) res->push_back({std::move(x)});
    }
    *out = res.release();
  })
}
int sqfref_gen_count(void* g, int s) {
  return static_cast<int>((*static_cast<std::vector<std::vector<Hypothesis>>*>(g))[static_cast<size_t>(s)].size());
}
int sqfref_gen_hyp(void* g, int s, int k, int32_t* tokens, float* steps, int cap, int32_t* len, double* cum,
                   double* score, int32_t* finish_step, int32_t* finished) {
  const Hypothesis& x = (*static_cast<std::vector<std::vector<Hypothesis>>*>(g))[static_cast<size_t>(s)]
                                                                                [static_cast<size_t>(k)];
  *len = static_cast<int32_t>(x.tokens.size());
  if (*len > cap) return -3;
  for (int i = 0; i < *len; ++i) {
    tokens[i] = x.tokens[static_cast<size_t>(i)];
    steps[i] = x.step_scores[static_cast<size_t>(i)];
  }
  *cum = x.cum_logprob;
  *score = x.score;
  *finish_step = x.finish_step;
  *finished = x.finished ? 1 : 0;
  return 0;
}
void sqfref_gen_free(void* g) { delete static_cast<std::vector<std::vector<Hypothesis>>*>(g); }
int sqfref_sample_from_topk(const float* logits, int vocab, int k, double temperature, double u, int32_t* out) {
  GUARD({ *out = sample_from_topk(logits, vocab, k, temperature, u); })
}
int sqfref_batch_for_inference(const int32_t* lens, int n, int64_t max_tokens, int32_t* ngroups, int32_t* sizes,
                               int32_t* members) {
  GUARD({
    std::vector<std::vector<int>> src(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) src[static_cast<size_t>(i)].assign(static_cast<size_t>(lens[i]), 4);
    auto groups = batch_for_inference(src, max_tokens);
    *ngroups = static_cast<int32_t>(groups.size());
    int64_t at = 0;
    for (size_t i = 0; i < groups.size(); ++i) {
      sizes[i] = static_cast<int32_t>(groups[i].size());
      for (int m : groups[i]) members[at++] = m;
    }
  })
}

}  // extern "C"

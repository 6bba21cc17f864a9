// C ABI (include/sqf_trainer.h) over the host trainer. Exceptions never cross
// the boundary: they become the reference's error classes as status codes.
#include <cstring>
#include <functional>
#include <memory>
#include <string>

#include "../../../include/sqf_trainer.h"
#include "nccl_dyn.hpp"
#include "checkpoint.hpp"
#include "generate.hpp"
#include "simulator.hpp"
#include "trainer.hpp"

namespace sqf {
namespace {

thread_local std::string g_err;
thread_local int g_code = 0;

int code_of(const std::exception& e);
int fail(const std::exception& e) {
  g_err = e.what();
  return g_code = code_of(e);
}
int code_of(const std::exception& e) {
  if (dynamic_cast<const ConfigError*>(&e)) return -1;
  if (dynamic_cast<const ShapeError*>(&e)) return -2;
  if (dynamic_cast<const BoundsError*>(&e)) return -3;
  if (dynamic_cast<const CapacityError*>(&e)) return -4;
  if (dynamic_cast<const IntegrityError*>(&e)) return -5;
  if (dynamic_cast<const DivergenceError*>(&e)) return -6;
  if (dynamic_cast<const RegistryError*>(&e)) return -7;
  if (dynamic_cast<const IoError*>(&e)) return -8;
  if (dynamic_cast<const DeviceError*>(&e)) return -10;
  return -9;
}

#define SQF_GUARD(...)                \
  try {                               \
    __VA_ARGS__;                      \
    return 0;                         \
  } catch (const std::exception& e) { \
    return fail(e);                   \
  }

struct Corpus {
  std::vector<SequencePair> pairs;
};

std::vector<SequencePair> unpack_pairs(int npairs, const int32_t* sl, const int32_t* tl, const int32_t* si,
                                       const int32_t* ti) {
  std::vector<SequencePair> out(static_cast<size_t>(npairs));
  int64_t so = 0, to = 0;
  for (int i = 0; i < npairs; ++i) {
    out[size_t(i)].source.assign(si + so, si + so + sl[i]);
    out[size_t(i)].target.assign(ti + to, ti + to + tl[i]);
    out[size_t(i)].corpus_index = i;
    so += sl[i];
    to += tl[i];
  }
  return out;
}

class MemoryTask : public TaskBase {
 public:
  MemoryTask(std::vector<SequencePair> p, int sv, int tv) : pairs_(std::move(p)), sv_(sv), tv_(tv) {}
  int source_vocab() const override { return sv_; }
  int target_vocab() const override { return tv_; }
  const std::vector<SequencePair>& train_pairs() const override { return pairs_; }

 private:
  std::vector<SequencePair> pairs_;
  int sv_, tv_;
};

std::vector<std::pair<std::string, std::string>> user_kv(const char* const* k, const char* const* v, int n) {
  std::vector<std::pair<std::string, std::string>> out;
  for (int i = 0; i < n; ++i) out.emplace_back(k[i], v[i]);
  return out;
}

void fill(sqf_step_stats* o, const StepStats& s) {
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

Trainer* T(void* t) { return static_cast<Trainer*>(t); }

}  // namespace
}  // namespace sqf

using namespace sqf;

extern "C" {

const char* sqf_last_error(void) { return g_err.c_str(); }
int sqf_last_status(void) { return g_code; }

int sqf_nccl_unique_id(void* out128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  if (NcclApi::get().GetUniqueId(&id) != ncclSuccess) {
    g_err = "ncclGetUniqueId failed";
    return -10;
  }
  std::memcpy(out128, &id, 128);
  return 0;
}

static void* create_trainer(const char* arch, const char* const* keys, const char* const* vals, int n,
                            const int32_t* src_len, const int32_t* tgt_len, const int32_t* src_ids,
                            const int32_t* tgt_ids, int npairs, int src_vocab, int tgt_vocab, int rank, int world,
                            const std::function<std::unique_ptr<Collective>()>& coll) {
  try {
    const Registry& reg = global_registry();
    Config cfg = reg.resolve_architecture(arch, user_kv(keys, vals, n));
    std::unique_ptr<TaskBase> task;
    if (npairs > 0)
      task = std::make_unique<MemoryTask>(unpack_pairs(npairs, src_len, tgt_len, src_ids, tgt_ids), src_vocab,
                                          tgt_vocab);
    return new Trainer(cfg, reg, std::move(task), rank, world, world > 1 ? coll() : nullptr);
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void* sqf_trainer_create(const char* arch, const char* const* keys, const char* const* vals, int n,
                         const int32_t* src_len, const int32_t* tgt_len, const int32_t* src_ids,
                         const int32_t* tgt_ids, int npairs, int src_vocab, int tgt_vocab, int rank, int world,
                         const void* nccl_id) {
  return create_trainer(arch, keys, vals, n, src_len, tgt_len, src_ids, tgt_ids, npairs, src_vocab, tgt_vocab, rank,
                        world, [&]() -> std::unique_ptr<Collective> {
                          if (!nccl_id) throw ConfigError("trainer: world > 1 needs an NCCL unique id");
                          ncclUniqueId id;
                          std::memcpy(&id, nccl_id, sizeof id);
                          return make_nccl_collective(rank, world, id);
                        });
}

void* sqf_trainer_create_host_collective(const char* arch, const char* const* keys, const char* const* vals, int n,
                                         const int32_t* src_len, const int32_t* tgt_len, const int32_t* src_ids,
                                         const int32_t* tgt_ids, int npairs, int src_vocab, int tgt_vocab, int rank,
                                         int world, sqf_host_allreduce_fn fn, void* user) {
  return create_trainer(arch, keys, vals, n, src_len, tgt_len, src_ids, tgt_ids, npairs, src_vocab, tgt_vocab, rank,
                        world, [&] { return make_host_collective(fn, user); });
}

const char* sqf_trainer_collective(void* t) { return t ? T(t)->collective() : "none"; }

void sqf_trainer_free(void* t) { delete T(t); }

void* sqf_task_create(const char* arch, const char* const* keys, const char* const* vals, int n) {
  try {
    const Registry& reg = global_registry();
    Config cfg = reg.resolve_architecture(arch, user_kv(keys, vals, n));
    return reg.make_task(cfg.get_str("task"), cfg).release();
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void sqf_task_free(void* t) { delete static_cast<TaskBase*>(t); }

int sqf_task_info(void* t, int32_t* src_vocab, int32_t* tgt_vocab, int32_t* npairs, int64_t* src_tokens,
                  int64_t* tgt_tokens) {
  SQF_GUARD({
    const TaskBase& task = *static_cast<TaskBase*>(t);
    *src_vocab = task.source_vocab();
    *tgt_vocab = task.target_vocab();
    *npairs = int32_t(task.train_pairs().size());
    int64_t a = 0, b = 0;
    for (const auto& p : task.train_pairs()) a += int64_t(p.source.size()), b += int64_t(p.target.size());
    *src_tokens = a;
    *tgt_tokens = b;
  })
}

int sqf_task_pairs(void* t, int32_t* src_len, int32_t* tgt_len, int32_t* src_ids, int32_t* tgt_ids) {
  SQF_GUARD({
    const auto& pairs = static_cast<TaskBase*>(t)->train_pairs();
    int64_t a = 0, b = 0;
    for (size_t i = 0; i < pairs.size(); ++i) {
      src_len[i] = int32_t(pairs[i].source.size());
      tgt_len[i] = int32_t(pairs[i].target.size());
      for (int x : pairs[i].source) src_ids[a++] = x;
      for (int x : pairs[i].target) tgt_ids[b++] = x;
    }
  })
}

int sqf_trainer_train_one(void* t, sqf_step_stats* out) {
  try {
    auto st = T(t)->train_one();
    if (!st) return 1;
    fill(out, *st);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int sqf_trainer_train_step(void* t, const int32_t* members, const int32_t* counts, sqf_step_stats* out) {
  SQF_GUARD({
    Trainer& tr = *T(t);
    const auto& pairs = tr.task().train_pairs();
    std::vector<std::vector<MiniBatch>> sub(size_t(tr.workers()));
    int64_t k = 0;
    for (int w = 0; w < tr.workers(); ++w)
      for (int a = 0; a < tr.accum(); ++a) {
        const int c = counts[w * tr.accum() + a];
        std::vector<int> m(members + k, members + k + c);
        k += c;
        sub[size_t(w)].push_back(c == 0 ? MiniBatch{} : make_minibatch(pairs, m));
      }
    fill(out, tr.train_step(sub));
  })
}

int sqf_trainer_evaluate(void* t, const int32_t* idx, int n, double* loss, double* nll, int64_t* ntokens,
                         int64_t* ncorrect) {
  SQF_GUARD({
    Trainer& tr = *T(t);
    const auto& pairs = tr.task().train_pairs();
    std::vector<SequencePair> sel;
    for (int i = 0; i < n; ++i) {
      SequencePair p = pairs.at(size_t(idx[i]));
      p.corpus_index = i;
      sel.push_back(std::move(p));
    }
    EvalStats e = tr.evaluate(sel);
    *loss = e.loss;
    *nll = e.nll;
    *ntokens = e.ntokens;
    *ncorrect = e.ncorrect;
  })
}

int64_t sqf_trainer_num_params(void* t) { return T(t)->model().num_params(); }

int sqf_trainer_params(void* t, float* out) {
  SQF_GUARD({
    T(t)->pull_params();
    auto p = T(t)->model().params();
    std::memcpy(out, p.data(), p.size() * 4);
  })
}

int sqf_trainer_set_params(void* t, const float* in) {
  SQF_GUARD({
    auto p = T(t)->model().params();
    std::memcpy(p.data(), in, p.size() * 4);
    T(t)->push_params();
  })
}

int sqf_trainer_last_grads(void* t, float* out) {
  SQF_GUARD({
    auto g = T(t)->reduced_grads();
    std::memcpy(out, g.data(), g.size() * 4);
  })
}

int sqf_trainer_manifest_size(void* t) { return int(T(t)->model().manifest().size()); }

int sqf_trainer_manifest_entry(void* t, int i, char* name, int cap, int64_t* offset, int64_t* numel,
                               int64_t* device_offset) {
  SQF_GUARD({
    const auto& e = T(t)->model().manifest().at(size_t(i));
    std::snprintf(name, size_t(cap), "%s", e.name.c_str());
    *offset = e.offset;
    *numel = e.numel;
    *device_offset = e.device_offset;
  })
}

int sqf_trainer_adam_state(void* t, float* m, float* v, int64_t* step_count) {
  SQF_GUARD({
    Trainer& tr = *T(t);
    for (auto& [name, data] : tr.optimizer().state_blobs()) {
      std::vector<float> canon(data.size());
      tr.model().to_canonical_order(data, canon);
      if (name == "adam.m") std::memcpy(m, canon.data(), canon.size() * 4);
      if (name == "adam.v") std::memcpy(v, canon.data(), canon.size() * 4);
    }
    *step_count = tr.optimizer().step_count();
  })
}

int sqf_trainer_scaler(void* t, double* scale, int64_t* successes) {
  SQF_GUARD({
    const LossScaler& s = T(t)->scaler();
    *scale = s.scale();
    *successes = s.successes();
  })
}

int sqf_trainer_progress(void* t, int64_t* step, int32_t* epoch, int32_t* cursor, int32_t* nbatches) {
  SQF_GUARD({
    *step = T(t)->step();
    *epoch = T(t)->epoch();
    *cursor = T(t)->cursor();
    *nbatches = T(t)->batches_per_epoch();
  })
}

int sqf_trainer_set_injector(void* t, const int64_t* steps, int n) {
  SQF_GUARD({
    std::vector<int64_t> s(steps, steps + n);
    T(t)->set_overflow_injector([s](int64_t step) { return std::find(s.begin(), s.end(), step) != s.end(); });
  })
}

int sqf_trainer_restore(void* t, int64_t step, int32_t epoch, int32_t cursor, double scale, int64_t successes) {
  SQF_GUARD({
    T(t)->restore_progress(step, epoch, cursor);
    if (T(t)->fp16()) T(t)->restore_scaler(scale, successes);
  })
}

int64_t sqf_trainer_kernel_launches(void* t) { return T(t)->kernel_launches(); }
float sqf_trainer_last_step_ms(void* t) { return T(t)->last_step_ms(); }
float sqf_trainer_flush_ms(void* t) {
  try {
    return T(t)->flush_ms();
  } catch (const std::exception& e) {
    fail(e);
    return -1.f;
  }
}
int64_t sqf_trainer_last_io_bytes(void* t, int64_t* d2h) {
  *d2h = T(t)->last_d2h_bytes();
  return T(t)->last_h2d_bytes();
}
void* sqf_trainer_stream(void* t) { return static_cast<void*>(T(t)->stream()); }

int sqf_simulate_timeline(const char* scenario, char* report, int cap) {
  SQF_GUARD({
    const std::string text = format_report(simulate_timeline(parse_scenario(scenario)));
    if (int(text.size()) + 1 > cap) throw BoundsError("sqf_simulate_timeline: report buffer too small");
    std::memcpy(report, text.c_str(), text.size() + 1);
  })
}

int sqf_trainer_save(void* t, const char* path) { SQF_GUARD(save_checkpoint(*T(t), path)) }

int sqf_trainer_load(void* t, const char* path, int32_t* version) {
  SQF_GUARD({
    const int v = load_checkpoint_into(*T(t), path);
    if (version) *version = v;
  })
}

int sqf_checkpoint_info(const char* path, int32_t* version, int64_t* nparams, int64_t* nopt, int64_t* meta_bytes) {
  SQF_GUARD({
    const RawCheckpoint raw = read_checkpoint(path);
    int64_t mb = 0;
    for (const auto& [k, v] : raw.meta) mb += int64_t(k.size() + v.size() + 4);
    *version = raw.version;
    *nparams = int64_t(raw.params.size());
    *nopt = int64_t(raw.opt.size());
    *meta_bytes = mb + 1;
  })
}

int sqf_checkpoint_read(const char* path, float* params, float* opt, char* meta, int64_t meta_cap) {
  SQF_GUARD({
    const RawCheckpoint raw = read_checkpoint(path);
    if (params) std::memcpy(params, raw.params.data(), raw.params.size() * 4);
    if (opt) std::memcpy(opt, raw.opt.data(), raw.opt.size() * 4);
    if (meta) {
      std::string text;
      for (const auto& [k, v] : raw.meta) text += k + " = " + v + "\n";
      if (int64_t(text.size()) + 1 > meta_cap) throw BoundsError("sqf_checkpoint_read: meta buffer too small");
      std::memcpy(meta, text.c_str(), text.size() + 1);
    }
  })
}

int sqf_trainer_overlap_log(void* t, int32_t* order, int cap, int32_t* early) {
  const std::vector<int>& log = T(t)->overlap_log();
  const int n = int(log.size());
  for (int i = 0; i < n && i < cap; ++i) order[i] = log[size_t(i)];
  *early = T(t)->overlap_early();
  return n;
}

int sqf_trainer_set_profile(void* t, int on) { SQF_GUARD(T(t)->set_profile(on)) }

int sqf_trainer_timeline(void* t, float* out, int cap) {
  Profiler* p = T(t)->profiler();
  if (!p) return 0;
  const int n = int(p->spans.size());
  for (int i = 0; i < n && i < cap; ++i) {
    const auto& s = p->spans[size_t(i)];
    out[4 * i] = float(s.stream);
    out[4 * i + 1] = float(s.cat);
    out[4 * i + 2] = s.t0;
    out[4 * i + 3] = s.t1;
  }
  return n;
}

const char* sqf_trainer_profile(void* t, int cls, double* ms, double* flops, double* bytes, int64_t* launches) {
  Profiler* p = T(t)->profiler();
  if (cls < 0 || cls >= Profiler::kCats) return nullptr;
  *ms = p ? p->ms[cls] : 0.0;
  *flops = p ? p->flops[cls] : 0.0;
  *bytes = p ? p->bytes[cls] : 0.0;
  *launches = p ? p->count[cls] : 0;
  return Profiler::name(cls);
}

// ---------------------------------------------------------------- host-only
int sqf_synthetic_corpus(int npairs, int src_vocab, int tgt_vocab, double zipf_s, uint64_t seed, int32_t* src_len,
                         int32_t* tgt_len, int32_t* src_ids, int32_t* tgt_ids, int64_t* src_total,
                         int64_t* tgt_total) {
  SQF_GUARD({
    auto pairs = synthetic_corpus(npairs, src_vocab, tgt_vocab, zipf_s, seed);
    int64_t so = 0, to = 0;
    for (int i = 0; i < npairs; ++i) {
      const auto& p = pairs[size_t(i)];
      if (src_len) src_len[i] = int32_t(p.source.size());
      if (tgt_len) tgt_len[i] = int32_t(p.target.size());
      if (src_ids) std::copy(p.source.begin(), p.source.end(), src_ids + so);
      if (tgt_ids) std::copy(p.target.begin(), p.target.end(), tgt_ids + to);
      so += int64_t(p.source.size());
      to += int64_t(p.target.size());
    }
    *src_total = so;
    *tgt_total = to;
  })
}

void* sqf_corpus_create(int npairs, const int32_t* sl, const int32_t* tl, const int32_t* si, const int32_t* ti) {
  auto* c = new Corpus;
  c->pairs = unpack_pairs(npairs, sl, tl, si, ti);
  return c;
}
void sqf_corpus_free(void* c) { delete static_cast<Corpus*>(c); }

int sqf_make_batches(void* corpus, int64_t max_tokens, int max_sentences, uint64_t seed, int32_t* nbatches,
                     int32_t* sizes, int32_t* members) {
  SQF_GUARD({
    const auto& pairs = static_cast<Corpus*>(corpus)->pairs;
    EpochPlan p = make_batches(pairs, max_tokens, max_sentences > 0 ? std::optional<int>(max_sentences) : std::nullopt,
                               seed);
    *nbatches = int32_t(p.batches.size());
    int64_t k = 0;
    for (size_t b = 0; b < p.batches.size(); ++b) {
      sizes[b] = int32_t(p.batches[b].size());
      for (int m : p.batches[b]) members[k++] = m;
    }
  })
}

int sqf_shuffle_epoch(int nbatches, uint64_t seed, int epoch, int32_t* order) {
  SQF_GUARD({
    EpochPlan p;
    p.batches.resize(size_t(nbatches));
    p.shuffle_seed = seed;
    auto o = shuffle_epoch(p, epoch);
    std::copy(o.begin(), o.end(), order);
  })
}

int sqf_make_minibatch(void* corpus, const int32_t* members, int n, int32_t* dims, int32_t* source,
                       int32_t* target_in, int32_t* target_out, int32_t* src_lens, int32_t* tgt_lens,
                       int64_t* ntokens) {
  SQF_GUARD({
    MiniBatch b = make_minibatch(static_cast<Corpus*>(corpus)->pairs, std::vector<int>(members, members + n));
    dims[0] = b.rows;
    dims[1] = b.src_width;
    dims[2] = b.tgt_width;
    if (source) std::copy(b.source.begin(), b.source.end(), source);
    if (target_in) std::copy(b.target_in.begin(), b.target_in.end(), target_in);
    if (target_out) std::copy(b.target_out.begin(), b.target_out.end(), target_out);
    if (src_lens) std::copy(b.src_lens.begin(), b.src_lens.end(), src_lens);
    if (tgt_lens) std::copy(b.tgt_lens.begin(), b.tgt_lens.end(), tgt_lens);
    if (ntokens) *ntokens = b.ntokens;
  })
}

int sqf_split_counts(int rows, int workers, int accum, int32_t* counts) {
  SQF_GUARD({
    const int groups = workers * accum;
    if (groups < 1) throw ConfigError("split: workers and accum must be at least 1");
    for (int g = 0; g < groups; ++g) counts[g] = rows / groups + (g < rows % groups ? 1 : 0);
  })
}

int sqf_bucket_gradients(const int64_t* sizes, int n, int64_t threshold, int32_t* nbuckets, int64_t* starts,
                         int64_t* ends) {
  SQF_GUARD({
    auto b = bucket_gradients(std::vector<int64_t>(sizes, sizes + n), threshold);
    *nbuckets = int32_t(b.size());
    for (size_t i = 0; i < b.size(); ++i) {
      starts[i] = b[i].start;
      ends[i] = b[i].end;
    }
  })
}

int sqf_model_init(const char* arch, const char* const* keys, const char* const* vals, int n, float* params,
                   int64_t cap, int64_t* num_params, int* manifest_size) {
  SQF_GUARD({
    const Registry& reg = global_registry();
    Config cfg = reg.resolve_architecture(arch, user_kv(keys, vals, n));
    auto m = reg.make_model(reg.architecture(cfg.get_str("arch")).base_model, cfg,
                            uint64_t(cfg.get_int("seed")));
    *num_params = m->num_params();
    *manifest_size = int(m->manifest().size());
    if (params && cap >= m->num_params()) std::memcpy(params, m->params().data(), size_t(m->num_params()) * 4);
  })
}

int sqf_scaler_run(double init, int64_t window, double mn, double mx, const uint8_t* overflow, int n,
                   double* scales, int32_t* diverged_at) {
  SQF_GUARD({
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

int sqf_schedule_lr(const char* name, double base, int64_t warmup, double init, double eta_min, int64_t period,
                    double t_mult, int64_t step, double* out) {
  SQF_GUARD({
    Config c = engine_default_config();
    c.set_user("lr", base);
    c.set_user("warmup", warmup);
    c.set_user("warmup_init_lr", init);
    c.set_user("eta_min", eta_min);
    c.set_user("cosine_period", period);
    c.set_user("cosine_t_mult", t_mult);
    *out = global_registry().make_scheduler(name, c)->lr(step);
  })
}

float sqf_quantize_fp16(float x) { return quantize_fp16(x); }

int sqf_gen_config_default(void* t, sqf_gen_config* out) {
  SQF_GUARD({
    GenConfig g = gen_config_from(T(t)->config());
    *out = sqf_gen_config{g.beam, g.max_len, g.diverse_groups, g.topk, g.lenpen, g.diverse_strength,
                          g.temperature, g.seed, g.no_cache ? 1 : 0, g.host_select ? 1 : 0};
  })
}

int sqf_generate(void* t, int mode, const int32_t* source, const int32_t* src_lens, int rows, int src_width,
                 const sqf_gen_config* c, const uint64_t* stream_ids, void** out) {
  SQF_GUARD({
    if (mode < 0 || mode > 2) throw ConfigError("generation: mode must be 0 (beam), 1 (diverse) or 2 (sample)");
    if (rows < 1 || src_width < 0) throw ShapeError("generation: batch has no rows");
    MiniBatch b;
    b.rows = rows;
    b.src_width = src_width;
    b.source.assign(source, source + size_t(rows) * src_width);
    b.src_lens.assign(src_lens, src_lens + rows);
    for (int s = 0; s < rows; ++s)
      if (src_lens[s] < 0 || src_lens[s] > src_width) throw ShapeError("generation: source length out of range");
    GenConfig g;
    g.beam = c->beam;
    g.max_len = c->max_len;
    g.diverse_groups = c->diverse_groups;
    g.topk = c->topk;
    g.lenpen = c->lenpen;
    g.diverse_strength = c->diverse_strength;
    g.temperature = c->temperature;
    g.seed = c->seed;
    g.no_cache = c->no_cache != 0;
    g.host_select = c->host_select != 0;
    auto res = std::make_unique<std::vector<std::vector<Hypothesis>>>();
    if (mode == 0) {
      *res = beam_search(*T(t), b, g);
    } else if (mode == 1) {
      *res = diverse_beam_search(*T(t), b, g);
    } else {
      std::vector<uint64_t> ids;
      if (stream_ids) ids.assign(stream_ids, stream_ids + rows);
      for (Hypothesis& h : top_k_sample(*T(t), b, g, ids)) res->push_back({std::move(h)});
    }
    *out = res.release();
  })
}

int sqf_gen_count(void* g, int s) {
  auto& r = *static_cast<std::vector<std::vector<Hypothesis>>*>(g);
  if (s < 0 || size_t(s) >= r.size()) return -3;
  return int(r[size_t(s)].size());
}

int sqf_gen_hyp(void* g, int s, int k, int32_t* tokens, float* step_scores, int cap, int32_t* len,
                double* cum_logprob, double* score, int32_t* finish_step, int32_t* finished) {
  SQF_GUARD({
    auto& r = *static_cast<std::vector<std::vector<Hypothesis>>*>(g);
    const Hypothesis& h = r.at(size_t(s)).at(size_t(k));
    *len = int32_t(h.tokens.size());
    if (int(h.tokens.size()) > cap) throw BoundsError("generation: token buffer too small");
    std::copy(h.tokens.begin(), h.tokens.end(), tokens);
    std::copy(h.step_scores.begin(), h.step_scores.end(), step_scores);
    *cum_logprob = h.cum_logprob;
    *score = h.score;
    *finish_step = h.finish_step;
    *finished = h.finished ? 1 : 0;
  })
}

void sqf_gen_free(void* g) { delete static_cast<std::vector<std::vector<Hypothesis>>*>(g); }

int sqf_score_hypothesis(double cum_logprob, int64_t length, double alpha, double* out) {
  SQF_GUARD({ *out = score_hypothesis(cum_logprob, length, alpha); })
}

int sqf_sample_from_topk(const float* logits, int vocab, int k, double temperature, double u, int32_t* out) {
  SQF_GUARD({ *out = sample_from_topk(logits, vocab, k, temperature, u); })
}

int sqf_batch_for_inference(const int32_t* lens, int n, int64_t max_tokens, int32_t* ngroups, int32_t* sizes,
                            int32_t* members) {
  SQF_GUARD({
    std::vector<std::vector<int>> src(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) src[size_t(i)].assign(size_t(lens[i]), 0);
    auto groups = batch_for_inference(src, max_tokens);
    *ngroups = int32_t(groups.size());
    int64_t at = 0;
    for (size_t i = 0; i < groups.size(); ++i) {
      sizes[i] = int32_t(groups[i].size());
      for (int m : groups[i]) members[at++] = m;
    }
  })
}

}  // extern "C"

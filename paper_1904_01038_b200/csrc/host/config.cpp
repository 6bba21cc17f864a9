#include "config.hpp"

#include <cstdio>

#include "plugins.hpp"
#include <sstream>

namespace sqf {

namespace {
const char* kind(size_t i) {
  static const char* names[] = {"bool", "int", "real", "string"};
  return names[i < 4 ? i : 3];
}
}  // namespace

void Config::declare(const std::string& key, ConfigValue def) {
  if (!values_.try_emplace(key, Entry{std::move(def), Provenance::Default}).second)
    throw ConfigError("config: key '" + key + "' declared twice");
}

const Config::Entry& Config::entry(const std::string& key) const {
  auto it = values_.find(key);
  if (it == values_.end()) throw ConfigError("config: unknown key '" + key + "'");
  return it->second;
}

Config::Entry& Config::entry_mut(const std::string& key) {
  auto it = values_.find(key);
  if (it == values_.end()) throw ConfigError("config: unknown key '" + key + "'");
  return it->second;
}

void Config::set_typed(const std::string& key, ConfigValue v, Provenance p) {
  Entry& e = entry_mut(key);
  if (e.v.index() != v.index())
    throw ConfigError("config: key '" + key + "' expects " + kind(e.v.index()) + ", got " +
                      kind(v.index()));
  e.v = std::move(v);
  e.prov = p;
}

void Config::set_arch(const std::string& key, ConfigValue v) { set_typed(key, std::move(v), Provenance::Architecture); }
void Config::set_user(const std::string& key, ConfigValue v) { set_typed(key, std::move(v), Provenance::User); }

void Config::set_user_raw(const std::string& key, const std::string& raw) {
  Entry& e = entry_mut(key);
  auto bad = [&]() { return ConfigError("config: key '" + key + "' expects " + kind(e.v.index()) + ", got '" + raw + "'"); };
  switch (e.v.index()) {
    case 0:
      if (raw == "true" || raw == "1") e.v = true;
      else if (raw == "false" || raw == "0") e.v = false;
      else throw bad();
      break;
    case 1: {
      size_t used = 0;
      int64_t x = 0;
      try { x = std::stoll(raw, &used); } catch (const std::exception&) { throw bad(); }
      if (used != raw.size()) throw bad();
      e.v = x;
      break;
    }
    case 2: {
      size_t used = 0;
      double x = 0;
      try { x = std::stod(raw, &used); } catch (const std::exception&) { throw bad(); }
      if (used != raw.size()) throw bad();
      e.v = x;
      break;
    }
    default:
      e.v = raw;
  }
  e.prov = Provenance::User;
}

bool Config::get_bool(const std::string& key) const {
  if (auto* p = std::get_if<bool>(&entry(key).v)) return *p;
  throw ConfigError("config: key '" + key + "' is not bool");
}
int64_t Config::get_int(const std::string& key) const {
  if (auto* p = std::get_if<int64_t>(&entry(key).v)) return *p;
  throw ConfigError("config: key '" + key + "' is not int");
}
double Config::get_real(const std::string& key) const {
  const Entry& e = entry(key);
  if (auto* p = std::get_if<double>(&e.v)) return *p;
  if (auto* p = std::get_if<int64_t>(&e.v)) return static_cast<double>(*p);
  throw ConfigError("config: key '" + key + "' is not real");
}
const std::string& Config::get_str(const std::string& key) const {
  if (auto* p = std::get_if<std::string>(&entry(key).v)) return *p;
  throw ConfigError("config: key '" + key + "' is not string");
}
Config::Provenance Config::provenance(const std::string& key) const { return entry(key).prov; }

std::vector<std::string> Config::keys() const {
  std::vector<std::string> out;
  for (const auto& kv : values_) out.push_back(kv.first);
  return out;
}

std::string Config::value_string(const std::string& key) const {
  const Entry& e = entry(key);
  switch (e.v.index()) {
    case 0: return std::get<bool>(e.v) ? "true" : "false";
    case 1: return std::to_string(std::get<int64_t>(e.v));
    case 2: {
      char buf[64];
      std::snprintf(buf, sizeof buf, "%a", std::get<double>(e.v));
      return buf;
    }
    default: return std::get<std::string>(e.v);
  }
}

void Config::merge_from(const Config& other) {
  for (const auto& kv : other.values_) values_[kv.first] = kv.second;
}

// ---------------------------------------------------------------- registry
namespace {
template <typename M>
std::string names_of(const M& m) {
  std::ostringstream ss;
  bool first = true;
  for (const auto& kv : m) {
    ss << (first ? "" : ", ") << kv.first;
    first = false;
  }
  return first ? "(none)" : ss.str();
}
template <typename M>
std::vector<std::string> keys_of(const M& m) {
  std::vector<std::string> out;
  for (const auto& kv : m) out.push_back(kv.first);
  return out;
}
template <typename M, typename C>
void insert(M& m, const char* ns, const std::string& name, C ctor, const std::string& origin) {
  if (name.empty()) throw RegistryError(std::string(ns) + ": plugin name must be non-empty");
  auto it = m.find(name);
  if (it != m.end())
    throw RegistryError(std::string(ns) + " '" + name + "': already registered by '" + it->second.origin +
                        "', duplicate registration from '" + origin + "'");
  m.emplace(name, typename M::mapped_type{std::move(ctor), origin});
}
template <typename M>
const auto& lookup(const M& m, const char* ns, const std::string& name) {
  auto it = m.find(name);
  if (it == m.end())
    throw RegistryError(std::string("unknown ") + ns + " '" + name + "'; registered: " + names_of(m));
  return it->second;
}
// ctor failures are re-raised as RegistryError("<ns> '<name>': <what>") (registry.cpp:112-161)
template <typename F>
auto wrap(const char* ns, const std::string& name, F&& f) -> decltype(f()) {
  try {
    return f();
  } catch (const std::exception& e) {
    throw RegistryError(std::string(ns) + " '" + name + "': " + e.what());
  }
}
}  // namespace

void Registry::register_model(const std::string& name, ModelCtor ctor, Config defaults, const std::string& origin) {
  insert(models_, "model", name, std::move(ctor), origin);
  model_defaults_.emplace(name, std::move(defaults));
}
void Registry::register_criterion(const std::string& n, CriterionCtor c, const std::string& o) { insert(criterions_, "criterion", n, std::move(c), o); }
void Registry::register_task(const std::string& n, TaskCtor c, const std::string& o) { insert(tasks_, "task", n, std::move(c), o); }
void Registry::register_optimizer(const std::string& n, OptimizerCtor c, const std::string& o) { insert(optimizers_, "optimizer", n, std::move(c), o); }
void Registry::register_scheduler(const std::string& n, SchedulerCtor c, const std::string& o) { insert(schedulers_, "scheduler", n, std::move(c), o); }

void Registry::register_architecture(ArchitectureDef def, const std::string& origin) {
  if (def.name.empty()) throw RegistryError("architecture: name must be non-empty");
  if (!models_.count(def.base_model))
    throw RegistryError("architecture '" + def.name + "': unknown base model '" + def.base_model + "'");
  const Config& defaults = model_defaults_.at(def.base_model);
  const Config engine = engine_default_config();
  for (const auto& kv : def.overrides)
    if (!defaults.has(kv.first) && !engine.has(kv.first))
      throw RegistryError("architecture '" + def.name + "': overrides undeclared key '" + kv.first + "'");
  auto it = architectures_.find(def.name);
  if (it != architectures_.end())
    throw RegistryError("architecture '" + def.name + "': already registered by '" + it->second.second +
                        "', duplicate registration from '" + origin + "'");
  const std::string name = def.name;
  architectures_.emplace(name, std::make_pair(std::move(def), origin));
}

Config Registry::resolve_architecture(const std::string& arch,
                                      const std::vector<std::pair<std::string, std::string>>& user) const {
  const ArchitectureDef& def = architecture(arch);
  Config c = engine_default_config();
  c.merge_from(model_defaults_.at(def.base_model));
  c.set_arch("arch", arch);
  for (const auto& kv : def.overrides) c.set_arch(kv.first, kv.second);
  for (const auto& kv : user) c.set_user_raw(kv.first, kv.second);
  return c;
}

std::unique_ptr<ModelBase> Registry::make_model(const std::string& n, const Config& cfg, uint64_t seed) const {
  const auto& s = lookup(models_, "model", n);
  return wrap("model", n, [&] { return s.ctor(cfg, seed); });
}
std::unique_ptr<CriterionBase> Registry::make_criterion(const std::string& n, const Config& cfg) const {
  const auto& s = lookup(criterions_, "criterion", n);
  return wrap("criterion", n, [&] { return s.ctor(cfg); });
}
std::unique_ptr<TaskBase> Registry::make_task(const std::string& n, const Config& cfg) const {
  const auto& s = lookup(tasks_, "task", n);
  return wrap("task", n, [&] { return s.ctor(cfg); });
}
std::unique_ptr<OptimizerBase> Registry::make_optimizer(const std::string& n, const Config& cfg, int64_t np) const {
  const auto& s = lookup(optimizers_, "optimizer", n);
  return wrap("optimizer", n, [&] { return s.ctor(cfg, np); });
}
std::unique_ptr<SchedulerBase> Registry::make_scheduler(const std::string& n, const Config& cfg) const {
  const auto& s = lookup(schedulers_, "scheduler", n);
  return wrap("scheduler", n, [&] { return s.ctor(cfg); });
}

const ArchitectureDef& Registry::architecture(const std::string& name) const {
  auto it = architectures_.find(name);
  if (it == architectures_.end())
    throw RegistryError("unknown architecture '" + name + "'; registered: " + names_of(architectures_));
  return it->second.first;
}
std::vector<std::string> Registry::model_names() const { return keys_of(models_); }
std::vector<std::string> Registry::criterion_names() const { return keys_of(criterions_); }
std::vector<std::string> Registry::task_names() const { return keys_of(tasks_); }
std::vector<std::string> Registry::optimizer_names() const { return keys_of(optimizers_); }
std::vector<std::string> Registry::scheduler_names() const { return keys_of(schedulers_); }
std::vector<std::string> Registry::architecture_names() const { return keys_of(architectures_); }
const Config& Registry::model_defaults(const std::string& name) const {
  auto it = model_defaults_.find(name);
  if (it == model_defaults_.end())
    throw RegistryError("unknown model '" + name + "'; registered: " + names_of(models_));
  return it->second;
}

Config engine_default_config() {
  Config c;
  const std::vector<std::pair<const char*, ConfigValue>> keys = {
      {"seed", int64_t{1}}, {"arch", std::string{"tiny_transformer"}}, {"task", std::string{"translation"}},
      {"train_src", std::string{}}, {"train_tgt", std::string{}}, {"valid_src", std::string{}},
      {"valid_tgt", std::string{}}, {"dict_src", std::string{}}, {"dict_tgt", std::string{}},
      {"min_count", int64_t{1}}, {"max_tokens", int64_t{1024}}, {"max_sentences", int64_t{0}},
      {"workers", int64_t{1}}, {"accum", int64_t{1}}, {"fp16", false}, {"fp16_init_scale", 128.0},
      {"fp16_scale_window", int64_t{256}}, {"fp16_min_scale", 0.03125}, {"fp16_max_scale", 32768.0},
      {"bucket_threshold", int64_t{16384}}, {"max_steps", int64_t{-1}}, {"max_epochs", int64_t{1}},
      {"save_interval", int64_t{100}}, {"save_dir", std::string{"checkpoints"}},
      {"criterion", std::string{"label_smoothed_cross_entropy"}}, {"label_smoothing", 0.1},
      {"optimizer", std::string{"adam"}}, {"lr", 5e-4}, {"adam_beta1", 0.9}, {"adam_beta2", 0.98},
      {"adam_eps", 1e-8}, {"scheduler", std::string{"inverse_sqrt"}}, {"warmup", int64_t{400}},
      {"warmup_init_lr", 0.0}, {"cosine_period", int64_t{1000}}, {"cosine_t_mult", 1.0}, {"eta_min", 0.0},
      {"beam", int64_t{4}}, {"lenpen", 0.6}, {"max_len", int64_t{0}}, {"diverse_groups", int64_t{1}},
      {"diverse_strength", 0.5}, {"sampling", false}, {"topk", int64_t{1}}, {"temperature", 1.0},
      {"nbest", int64_t{1}},
      // ---- B200 additions (declared keys, same override rules)
      {"dispatch", std::string{"split"}},      // split: trainer.cpp:186-202; deal: per-GPU packed batches
      {"bf16", false},                         // bf16 compute, fp32 grads, scale fixed at 1
      {"synthetic_pairs", int64_t{0}},         // task "synthetic": corpus size
      {"zipf_s", 1.1},                         // task "synthetic": token-id skew
      {"rank", int64_t{0}},                    // data-parallel rank of this process
      {"overlap_allreduce", true},             // start bucket all-reduces during the last backward
      {"overlap_simulate", false},             // testing: run the overlap schedule without NCCL (world 1)
  };
  for (const auto& kv : keys) c.declare(kv.first, kv.second);
  return c;
}

Config transformer_default_config() {
  Config c;
  c.declare("src_vocab", int64_t{0});
  c.declare("tgt_vocab", int64_t{0});
  c.declare("d_model", int64_t{64});
  c.declare("heads", int64_t{4});
  c.declare("enc_layers", int64_t{2});
  c.declare("dec_layers", int64_t{2});
  c.declare("d_ffn", int64_t{128});
  c.declare("max_positions", int64_t{256});
  c.declare("dropout", 0.0);
  c.declare("share_embeddings", false);
  return c;
}

}  // namespace sqf

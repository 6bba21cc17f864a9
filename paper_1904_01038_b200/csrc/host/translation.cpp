#include "translation.hpp"

#include <algorithm>
#include <fstream>
#include <map>
#include <sstream>

namespace sqf {

Dictionary::Dictionary() {
  for (const char* s : {"<s>", "<pad>", "</s>", "<unk>"}) add(s, 0);
}

int Dictionary::add(const std::string& sym, int64_t count) {
  auto it = std::lower_bound(sorted_.begin(), sorted_.end(), sym,
                             [](const std::pair<std::string, int>& e, const std::string& s) { return e.first < s; });
  if (it != sorted_.end() && it->first == sym) throw ConfigError("dictionary: duplicate symbol '" + sym + "'");
  const int id = size();
  syms_.push_back(sym);
  counts_.push_back(count);
  sorted_.insert(it, {sym, id});
  return id;
}

int Dictionary::index(const std::string& sym) const {
  auto it = std::lower_bound(sorted_.begin(), sorted_.end(), sym,
                             [](const std::pair<std::string, int>& e, const std::string& s) { return e.first < s; });
  return it != sorted_.end() && it->first == sym ? it->second : kUnk;
}

const std::string& Dictionary::symbol(int id) const {
  if (id < 0 || id >= size()) throw BoundsError("dictionary: id out of range");
  return syms_[size_t(id)];
}

int64_t Dictionary::count(int id) const {
  if (id < 0 || id >= size()) throw BoundsError("dictionary: id out of range");
  return counts_[size_t(id)];
}

std::vector<int> Dictionary::encode(const std::vector<std::string>& tokens) const {
  std::vector<int> ids;
  ids.reserve(tokens.size() + 1);
  for (const auto& t : tokens) ids.push_back(index(t));
  ids.push_back(kEos);
  return ids;
}

Dictionary Dictionary::load(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw IoError("dictionary: cannot read " + path);
  Dictionary d;
  for (std::string line; std::getline(f, line);) {
    if (line.empty()) continue;
    std::istringstream ls(line);
    std::string sym;
    int64_t n = 0;
    if (!(ls >> sym >> n)) throw IoError("dictionary: malformed line '" + line + "'");
    d.add(sym, n);
  }
  return d;
}

Dictionary Dictionary::build(const std::vector<std::vector<std::string>>& corpus, int64_t min_count) {
  if (min_count < 1) throw ConfigError("build_dictionary: min_count must be >= 1");
  std::map<std::string, int64_t> freq;
  for (const auto& sent : corpus)
    for (const auto& t : sent) ++freq[t];
  std::vector<std::pair<std::string, int64_t>> keep;
  std::copy_if(freq.begin(), freq.end(), std::back_inserter(keep), [&](const auto& e) { return e.second >= min_count; });
  std::stable_sort(keep.begin(), keep.end(), [](const auto& a, const auto& b) {
    return a.second != b.second ? a.second > b.second : a.first < b.first;
  });
  Dictionary d;
  for (const auto& [sym, n] : keep) d.add(sym, n);
  return d;
}

std::vector<std::vector<std::string>> read_tokenized_lines(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw IoError("corpus: cannot read " + path);
  std::vector<std::vector<std::string>> lines;
  for (std::string line; std::getline(f, line);) {
    std::istringstream ls(line);
    std::vector<std::string> toks;
    for (std::string t; ls >> t;) toks.push_back(t);
    lines.push_back(std::move(toks));
  }
  return lines;
}

std::vector<SequencePair> load_parallel_corpus(const std::string& src_path, const std::string& tgt_path,
                                               const Dictionary& src, const Dictionary& tgt) {
  const auto s = read_tokenized_lines(src_path), t = read_tokenized_lines(tgt_path);
  if (s.size() != t.size()) throw IoError("corpus: line count mismatch between " + src_path + " and " + tgt_path);
  std::vector<SequencePair> pairs(s.size());
  for (size_t i = 0; i < s.size(); ++i) pairs[i] = {src.encode(s[i]), tgt.encode(t[i]), int(i)};
  return pairs;
}

TranslationTask::TranslationTask(const Config& cfg) {
  const std::string ts = cfg.get_str("train_src"), tt = cfg.get_str("train_tgt");
  const std::string vs = cfg.get_str("valid_src"), vt = cfg.get_str("valid_tgt");
  if (ts.empty() != tt.empty()) throw ConfigError("translation: train_src and train_tgt must be given together");
  if (vs.empty() != vt.empty()) throw ConfigError("translation: valid_src and valid_tgt must be given together");
  const int64_t min_count = cfg.get_int("min_count");
  auto dict = [&](const std::string& file, const std::string& train) {
    if (!file.empty()) return Dictionary::load(file);
    if (!train.empty()) return Dictionary::build(read_tokenized_lines(train), min_count);
    return Dictionary();
  };
  src_ = dict(cfg.get_str("dict_src"), ts);
  tgt_ = dict(cfg.get_str("dict_tgt"), tt);
  if (!ts.empty()) train_ = load_parallel_corpus(ts, tt, src_, tgt_);
  if (!vs.empty()) valid_ = load_parallel_corpus(vs, vt, src_, tgt_);
}

}  // namespace sqf

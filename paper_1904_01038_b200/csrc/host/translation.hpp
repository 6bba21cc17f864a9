// The file-based `translation` task (reference tasks.cpp:7-33, Dictionary and
// corpus loading data.cpp:13-120, 225-271): whitespace-tokenised parallel
// text, dictionaries either loaded ("sym count" lines) or built from the
// training side (count >= min_count, most frequent first, ties by symbol),
// the four reserved symbols <s> <pad> </s> <unk> at ids 0..3, unknown words
// -> <unk>, every sentence eos-terminated, corpus_index = line number.
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "plugins.hpp"

namespace sqf {

class Dictionary {
 public:
  Dictionary();
  int size() const { return int(syms_.size()); }
  int add(const std::string& sym, int64_t count);  // ConfigError on duplicates
  int index(const std::string& sym) const;         // kUnk when absent
  const std::string& symbol(int id) const;
  int64_t count(int id) const;
  std::vector<int> encode(const std::vector<std::string>& tokens) const;  // + eos
  static Dictionary load(const std::string& path);
  static Dictionary build(const std::vector<std::vector<std::string>>& corpus, int64_t min_count);

 private:
  std::vector<std::string> syms_;
  std::vector<int64_t> counts_;
  std::vector<std::pair<std::string, int>> sorted_;  // symbol -> id, by symbol
};

std::vector<std::vector<std::string>> read_tokenized_lines(const std::string& path);
std::vector<SequencePair> load_parallel_corpus(const std::string& src_path, const std::string& tgt_path,
                                               const Dictionary& src, const Dictionary& tgt);

class TranslationTask : public TaskBase {
 public:
  explicit TranslationTask(const Config& cfg);
  int source_vocab() const override { return src_.size(); }
  int target_vocab() const override { return tgt_.size(); }
  const std::vector<SequencePair>& train_pairs() const override { return train_; }
  const std::vector<SequencePair>& valid_pairs() const { return valid_; }

 private:
  Dictionary src_, tgt_;
  std::vector<SequencePair> train_, valid_;
};

}  // namespace sqf

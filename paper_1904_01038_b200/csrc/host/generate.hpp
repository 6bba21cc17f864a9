// Sequence generation over the B200 trainer's model (reference
// include/seqforge/generate.hpp, src/generate.cpp): beam search, diverse beam
// search, top-k sampling, inference batching. The decoder runs on the device
// (Trainer::inc_* / last_position_logits, the trainer's compute weights:
// fp32 master, or the fp16/bf16 shadow on the tensor-core kernels); the host keeps
// the reference's selection rules (candidate order, stable ties, eos banking,
// admissible early stop, final n-best order) so hypotheses match it.
//
// Decoding: by default incremental, with per-layer K/V caches on the device
// (reorder = a row gather kernel); no_cache selects the reference's cache-free
// mode (generate.cpp:86-120), which re-decodes every live prefix per step.
#pragma once

#include <cstdint>
#include <vector>

#include "common.hpp"
#include "config.hpp"

namespace sqf {

class Trainer;

struct GenConfig {
  int beam = 4;
  double lenpen = 0.6;
  int max_len = 0;  // 0 = 2 * source_len + 8
  int diverse_groups = 1;
  double diverse_strength = 0.5;
  int topk = 1;
  double temperature = 1.0;
  uint64_t seed = 1;
  bool no_cache = false;  // re-decode the full prefix each step (generate.hpp:21)
  bool host_select = false;  // B200: rank all rows x V candidates on the host (testing)
};

// generate.cpp:15-26
GenConfig gen_config_from(const Config& cfg);

struct Hypothesis {
  std::vector<int> tokens;
  std::vector<float> step_scores;
  double cum_logprob = 0.0;
  bool finished = false;
  int finish_step = 0;
  double score = 0.0;
};

// generate.cpp:28-32
double score_hypothesis(double cum_logprob, int64_t length, double alpha);

// generate.cpp:123-345 (groups = 1)
std::vector<std::vector<Hypothesis>> beam_search(Trainer& tr, const MiniBatch& batch, const GenConfig& cfg);
// generate.cpp:347-351 (groups = cfg.diverse_groups, lambda = cfg.diverse_strength)
std::vector<std::vector<Hypothesis>> diverse_beam_search(Trainer& tr, const MiniBatch& batch,
                                                         const GenConfig& cfg);
// generate.cpp:385-457
std::vector<Hypothesis> top_k_sample(Trainer& tr, const MiniBatch& batch, const GenConfig& cfg,
                                     const std::vector<uint64_t>& stream_ids = {});
// generate.cpp:353-383
int sample_from_topk(const float* logits, int vocab, int k, double temperature, double u);
// generate.cpp:459-480
std::vector<std::vector<int>> batch_for_inference(const std::vector<std::vector<int>>& sources,
                                                  int64_t max_tokens);

}  // namespace sqf

// Host-side vocabulary shared by the B200 trainer: error taxonomy, RNG, data
// pipeline types. Mirrors the reference's public names (seqforge/common.hpp,
// rng.hpp, data.hpp) so code written against the reference reads the same.
#pragma once

#include <array>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace sqf {

// Error taxonomy (reference: include/seqforge/common.hpp:11-34) plus
// DeviceError for CUDA/NCCL failures, which the reference cannot raise.
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ShapeError : std::runtime_error { using std::runtime_error::runtime_error; };
struct BoundsError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CapacityError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IntegrityError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DivergenceError : std::runtime_error { using std::runtime_error::runtime_error; };
struct RegistryError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IoError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };

// Counter-based generator: (seed, stream, counter) -> u64 through three
// MurmurHash3 fmix64 rounds (reference rng.cpp:10-27). Bit-exact by design:
// parameter init, epoch shuffles and dropout masks must replay the
// reference's streams.
class RngStream {
 public:
  RngStream(uint64_t seed, uint64_t stream_id, uint64_t counter = 0)
      : seed_(seed), stream_(stream_id), counter_(counter) {}

  static constexpr uint64_t fmix64(uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k;
  }
  static constexpr uint64_t hash(uint64_t seed, uint64_t stream, uint64_t counter) {
    return fmix64(fmix64(fmix64(seed + 0x9e3779b97f4a7c15ull) ^ stream) ^ counter);
  }

  uint64_t next_u64() { return hash(seed_, stream_, counter_++); }
  // uniform [0,1) from the top 53 bits (rng.cpp:29-31)
  double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double next_normal();              // Box-Muller, two ticks (rng.cpp:33-41)
  uint64_t next_below(uint64_t n);   // 128-bit multiply-shift (rng.cpp:43-51)

  template <typename T>
  void shuffle(std::vector<T>& v) {  // Fisher-Yates (rng.hpp:22-28)
    for (size_t i = v.size(); i > 1; --i) {
      size_t j = static_cast<size_t>(next_below(i));
      std::swap(v[i - 1], v[j]);
    }
  }
  uint64_t counter() const { return counter_; }

 private:
  uint64_t seed_, stream_, counter_;
};

inline constexpr uint64_t kStreamInit = 0;
inline constexpr uint64_t kStreamDropoutBase = 1ull << 32;  // | (step << 8) | site
inline constexpr uint64_t kStreamCorpus = 4242;             // synthetic corpus

inline constexpr int kBos = 0, kPad = 1, kEos = 2, kUnk = 3, kNumReserved = 4;

struct SequencePair {
  std::vector<int> source;  // eos-terminated
  std::vector<int> target;  // eos-terminated
  int corpus_index = 0;
};

struct MiniBatch {
  int rows = 0, src_width = 0, tgt_width = 0;
  std::vector<int> source, target_in, target_out, src_lens, tgt_lens, members;
  int64_t ntokens = 0;
  // several packed batches in one pass (trainer.cpp pack_local): (rows,
  // src_width, tgt_width) of each, their id arrays concatenated unpadded;
  // empty: one batch of rows x src_width / tgt_width
  std::vector<std::array<int, 3>> parts;
};

struct EpochPlan {
  std::vector<std::vector<int>> batches;
  uint64_t shuffle_seed = 0;
};

// data.cpp:115-161 — sort by (tgt len, src len, corpus idx); greedy pack under
// rows * max(S_max, T_max) <= max_tokens (and rows <= max_sentences).
EpochPlan make_batches(const std::vector<SequencePair>& pairs, int64_t max_tokens,
                       std::optional<int> max_sentences, uint64_t shuffle_seed);
// data.cpp:163-170
std::vector<int> shuffle_epoch(const EpochPlan& plan, int epoch);
// data.cpp:172-219
MiniBatch make_minibatch(const std::vector<SequencePair>& pairs, const std::vector<int>& members);
// trainer.cpp:186-202 ("split" dispatch): rows -> W*A contiguous groups
std::vector<std::vector<MiniBatch>> split_batch(const std::vector<SequencePair>& pairs,
                                                const MiniBatch& batch, int workers, int accum);

// Synthetic WMT-shaped corpus: lengths clamp(round(exp(3.1+0.6z)),1,200),
// target ~ source*(1+0.1z'), ids Zipf(zipf_s) over [4, vocab) (uniform if zipf_s <= 0).
std::vector<SequencePair> synthetic_corpus(int npairs, int src_vocab, int tgt_vocab, double zipf_s,
                                           uint64_t seed, uint64_t stream = kStreamCorpus);

struct GradientBucket {
  int64_t start = 0, end = 0;
};
// trainer.cpp:50-73 — cut in reverse order at `threshold` elements
std::vector<GradientBucket> bucket_gradients(const std::vector<int64_t>& sizes, int64_t threshold);

// LossScaler (trainer.cpp:21-48)
class LossScaler {
 public:
  LossScaler(double init, int64_t window, double min_scale, double max_scale);
  double scale() const { return scale_; }
  int64_t successes() const { return good_; }
  int64_t window() const { return window_; }
  void update(bool overflowed);
  void restore(double scale, int64_t successes);

 private:
  double scale_;
  int64_t window_;
  double min_, max_;
  int64_t good_ = 0;
};

// binary16 round-to-nearest-even round trip (fp16.cpp:22-76), host side
uint16_t f32_to_f16_bits(float x);
float f16_bits_to_f32(uint16_t h);
inline float quantize_fp16(float x) { return f16_bits_to_f32(f32_to_f16_bits(x)); }

// model.cpp:12-19
void positional_row(int pos, int d, float* out);

}  // namespace sqf

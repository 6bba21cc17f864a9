// Host data pipeline: batch packing, epoch shuffles, padded id matrices,
// synthetic corpus. Everything here is integer work that must agree
// bit-for-bit with the reference (batch composition and padding masks are a
// parity gate), so it runs on the host exactly once per batch and is then
// uploaded; see DESIGN.md "Data layout".
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>

#include "common.hpp"

namespace sqf {

double RngStream::next_normal() {
  // two ticks per draw, no cached spare (reference rng.cpp:33-41)
  double u1 = next_double();
  const double u2 = next_double();
  if (u1 <= 0.0) u1 = 0x1.0p-53;
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

uint64_t RngStream::next_below(uint64_t n) {
  if (n <= 1) return 0;
  const unsigned __int128 wide = static_cast<unsigned __int128>(next_u64()) * n;
  return static_cast<uint64_t>(wide >> 64);
}

EpochPlan make_batches(const std::vector<SequencePair>& pairs, int64_t max_tokens,
                       std::optional<int> max_sentences, uint64_t shuffle_seed) {
  if (max_tokens < 1) throw ConfigError("make_batches: max_tokens must be >= 1");
  if (max_sentences && *max_sentences < 1)
    throw ConfigError("make_batches: max_sentences must be >= 1");
  std::vector<int> idx(pairs.size());
  std::iota(idx.begin(), idx.end(), 0);
  auto key = [&](int i) {
    const SequencePair& p = pairs[static_cast<size_t>(i)];
    return std::make_tuple(p.target.size(), p.source.size(), p.corpus_index);
  };
  std::sort(idx.begin(), idx.end(), [&](int a, int b) { return key(a) < key(b); });

  EpochPlan plan;
  plan.shuffle_seed = shuffle_seed;
  std::vector<int> open;
  int64_t width = 0;  // max(S_max, T_max) of the open batch
  for (int i : idx) {
    const SequencePair& p = pairs[static_cast<size_t>(i)];
    const int64_t w = static_cast<int64_t>(std::max(p.source.size(), p.target.size()));
    const int64_t n = static_cast<int64_t>(open.size()) + 1;
    const bool fits = n * std::max(width, w) <= max_tokens && (!max_sentences || n <= *max_sentences);
    if (!open.empty() && !fits) {
      plan.batches.push_back(std::move(open));
      open.clear();
      width = 0;
    }
    open.push_back(p.corpus_index);
    width = std::max(width, w);
  }
  if (!open.empty()) plan.batches.push_back(std::move(open));
  return plan;
}

std::vector<int> shuffle_epoch(const EpochPlan& plan, int epoch) {
  if (epoch < 1) throw ConfigError("shuffle_epoch: epoch must be >= 1");
  std::vector<int> order(plan.batches.size());
  std::iota(order.begin(), order.end(), 0);
  RngStream(plan.shuffle_seed, static_cast<uint64_t>(epoch)).shuffle(order);
  return order;
}

MiniBatch make_minibatch(const std::vector<SequencePair>& pairs, const std::vector<int>& members) {
  std::vector<const SequencePair*> rows;
  rows.reserve(members.size());
  for (int ci : members) {
    const SequencePair* hit = nullptr;
    if (ci >= 0 && ci < static_cast<int>(pairs.size()) && pairs[static_cast<size_t>(ci)].corpus_index == ci)
      hit = &pairs[static_cast<size_t>(ci)];
    else
      for (const auto& p : pairs)
        if (p.corpus_index == ci) { hit = &p; break; }
    if (!hit) throw BoundsError("make_minibatch: corpus index not present");
    rows.push_back(hit);
  }
  MiniBatch b;
  b.rows = static_cast<int>(rows.size());
  for (const auto* p : rows) {
    b.src_width = std::max(b.src_width, static_cast<int>(p->source.size()));
    b.tgt_width = std::max(b.tgt_width, static_cast<int>(p->target.size()));
  }
  const size_t S = static_cast<size_t>(b.src_width), T = static_cast<size_t>(b.tgt_width);
  b.source.assign(b.rows * S, kPad);
  b.target_in.assign(b.rows * T, kPad);
  b.target_out.assign(b.rows * T, kPad);
  for (size_t r = 0; r < rows.size(); ++r) {
    const auto& src = rows[r]->source;
    const auto& tgt = rows[r]->target;
    std::copy(src.begin(), src.end(), b.source.begin() + static_cast<ptrdiff_t>(r * S));
    // teacher forcing: bos then target[:-1]; output side is the target itself
    b.target_in[r * T] = kBos;
    if (!tgt.empty()) std::copy(tgt.begin(), tgt.end() - 1, b.target_in.begin() + static_cast<ptrdiff_t>(r * T + 1));
    std::copy(tgt.begin(), tgt.end(), b.target_out.begin() + static_cast<ptrdiff_t>(r * T));
    b.src_lens.push_back(static_cast<int>(src.size()));
    b.tgt_lens.push_back(static_cast<int>(tgt.size()));
    b.ntokens += static_cast<int64_t>(tgt.size());
    b.members.push_back(rows[r]->corpus_index);
  }
  return b;
}

std::vector<std::vector<MiniBatch>> split_batch(const std::vector<SequencePair>& pairs,
                                                const MiniBatch& batch, int workers, int accum) {
  const int groups = workers * accum;
  const int base = batch.rows / groups, extra = batch.rows % groups;
  std::vector<std::vector<MiniBatch>> out(static_cast<size_t>(workers));
  int row = 0;
  for (int g = 0; g < groups; ++g) {
    const int take = base + (g < extra ? 1 : 0);
    std::vector<int> m(batch.members.begin() + row, batch.members.begin() + row + take);
    row += take;
    out[static_cast<size_t>(g / accum)].push_back(make_minibatch(pairs, m));
  }
  return out;
}

std::vector<SequencePair> synthetic_corpus(int npairs, int src_vocab, int tgt_vocab, double zipf_s,
                                           uint64_t seed, uint64_t stream) {
  if (npairs < 0 || src_vocab <= kNumReserved || tgt_vocab <= kNumReserved)
    throw ConfigError("synthetic_corpus: need npairs >= 0 and vocab > 4");
  // inverse-CDF tables for Zipf(s) over ranks 1..V-4 -> ids 4..V-1
  auto make_cdf = [&](int vocab) {
    std::vector<double> cdf(static_cast<size_t>(vocab - kNumReserved));
    double acc = 0.0;
    for (size_t k = 0; k < cdf.size(); ++k) {
      acc += zipf_s > 0 ? std::pow(static_cast<double>(k + 1), -zipf_s) : 1.0;
      cdf[k] = acc;
    }
    for (double& c : cdf) c /= acc;
    return cdf;
  };
  const std::vector<double> src_cdf = make_cdf(src_vocab), tgt_cdf = make_cdf(tgt_vocab);
  RngStream rng(seed, stream);
  auto draw = [&](const std::vector<double>& cdf) {
    const double u = rng.next_double();
    const size_t k = static_cast<size_t>(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
    return kNumReserved + static_cast<int>(std::min(k, cdf.size() - 1));
  };
  auto clamp_len = [](double x) { return static_cast<int>(std::clamp(std::round(x), 1.0, 200.0)); };
  std::vector<SequencePair> out(static_cast<size_t>(npairs));
  for (int i = 0; i < npairs; ++i) {
    SequencePair& p = out[static_cast<size_t>(i)];
    const int ls = clamp_len(std::exp(3.1 + 0.6 * rng.next_normal()));
    const int lt = clamp_len(static_cast<double>(ls) * (1.0 + 0.1 * rng.next_normal()));
    for (int j = 0; j < ls; ++j) p.source.push_back(draw(src_cdf));
    for (int j = 0; j < lt; ++j) p.target.push_back(draw(tgt_cdf));
    p.source.push_back(kEos);
    p.target.push_back(kEos);
    p.corpus_index = i;
  }
  return out;
}

std::vector<GradientBucket> bucket_gradients(const std::vector<int64_t>& sizes, int64_t threshold) {
  if (threshold < 1) throw ConfigError("bucket_gradients: threshold must be at least 1");
  std::vector<int64_t> start(sizes.size() + 1, 0);
  for (size_t i = 0; i < sizes.size(); ++i) {
    if (sizes[i] < 1) throw ConfigError("bucket_gradients: parameter sizes must be positive");
    start[i + 1] = start[i] + sizes[i];
  }
  std::vector<GradientBucket> out;
  size_t hi = sizes.size();
  int64_t acc = 0;
  for (size_t i = sizes.size(); i-- > 0;) {
    acc += sizes[i];
    if (acc >= threshold) {
      out.push_back({start[i], start[hi]});
      hi = i;
      acc = 0;
    }
  }
  if (hi > 0) out.push_back({0, start[hi]});
  return out;
}

namespace {
bool is_pow2(double x) {
  int e = 0;
  return x > 0.0 && std::frexp(x, &e) == 0.5;
}
}  // namespace

LossScaler::LossScaler(double init, int64_t window, double min_scale, double max_scale)
    : scale_(init), window_(window), min_(min_scale), max_(max_scale) {
  if (window_ < 1) throw ConfigError("loss scaler: window must be at least 1");
  if (!is_pow2(scale_) || !is_pow2(min_) || !is_pow2(max_))
    throw ConfigError("loss scaler: scales must be powers of two");
  if (min_ > scale_ || scale_ > max_) throw ConfigError("loss scaler: initial scale outside [min, max]");
}

void LossScaler::update(bool overflowed) {
  if (overflowed) {
    good_ = 0;
    scale_ *= 0.5;
    if (scale_ < min_) throw DivergenceError("loss scale fell below its floor; training diverged");
    return;
  }
  if (++good_ >= window_) {
    good_ = 0;
    scale_ = std::min(2.0 * scale_, max_);
  }
}

void LossScaler::restore(double scale, int64_t successes) {
  if (!is_pow2(scale) || scale < min_ || scale > max_ || successes < 0 || successes >= window_)
    throw IntegrityError("loss scaler: restored state out of range");
  scale_ = scale;
  good_ = successes;
}

uint16_t f32_to_f16_bits(float x) {
  uint32_t f;
  std::memcpy(&f, &x, 4);
  const uint32_t sign = (f >> 16) & 0x8000u;
  const int be = static_cast<int>((f >> 23) & 0xFF);
  const uint32_t man = f & 0x7FFFFFu;
  if (be == 0xFF) return static_cast<uint16_t>(sign | (man ? 0x7E00u : 0x7C00u));
  const int e = be - 127;
  if (e >= 16) return static_cast<uint16_t>(sign | 0x7C00u);
  // significand with implicit bit; value = sig * 2^(e-23)
  const uint32_t sig = be ? (man | 0x800000u) : man;
  // target exponent: normal half keeps 10 fraction bits; below 2^-14 the
  // ulp is fixed at 2^-24
  const int shift = e >= -14 ? 13 : 13 + (-14 - e);
  if (shift > 25) return static_cast<uint16_t>(sign);
  uint32_t q = sig >> shift;
  const uint32_t rem = sig & ((1u << shift) - 1u), half = 1u << (shift - 1);
  if (rem > half || (rem == half && (q & 1u))) ++q;
  // for normals q includes the implicit bit at 2^10; adding the biased
  // exponent minus one lets a mantissa carry roll into the exponent (and
  // onto the infinity pattern) for free
  const uint32_t h = e >= -14 ? (static_cast<uint32_t>(e + 14) << 10) + q : q;
  return static_cast<uint16_t>(sign | h);
}

float f16_bits_to_f32(uint16_t h) {
  const uint32_t sign = static_cast<uint32_t>(h & 0x8000u) << 16;
  const int e = (h >> 10) & 0x1F;
  const uint32_t man = h & 0x3FFu;
  float mag;
  if (e == 0) mag = std::ldexp(static_cast<float>(man), -24);
  else if (e == 31) mag = man ? std::numeric_limits<float>::quiet_NaN() : std::numeric_limits<float>::infinity();
  else mag = std::ldexp(static_cast<float>(man | 0x400u), e - 25);
  uint32_t bits;
  std::memcpy(&bits, &mag, 4);
  bits |= sign;
  float out;
  std::memcpy(&out, &bits, 4);
  return out;
}

void positional_row(int pos, int d, float* out) {
  // float pow/sin/cos exactly as model.cpp:12-19 evaluates them
  for (int i = 0; 2 * i < d; ++i) {
    const float angle = static_cast<float>(pos) *
                        std::pow(10000.0f, -2.0f * static_cast<float>(i) / static_cast<float>(d));
    out[2 * i] = std::sin(angle);
    if (2 * i + 1 < d) out[2 * i + 1] = std::cos(angle);
  }
}

}  // namespace sqf

// Built-in plug-ins, registered through the same public Registry calls a user
// plug-in would use (reference builtins.cpp:13-65): the pre-norm transformer
// (model.cpp), cross_entropy / label_smoothed_cross_entropy (criterions.cpp),
// adam / sgd (optim.cpp), fixed / inverse_sqrt / cosine_restart schedules,
// and the tasks. Named architectures add the BASELINE.json configs.
#include <cmath>

#include "translation.hpp"
#include "device_tape.hpp"
#include "plugins.hpp"

namespace sqf {

// ------------------------------------------------------------------ model
void ModelBase::to_device_order(std::span<const float> canonical, std::span<float> device) const {
  for (const auto& e : manifest())
    std::copy(canonical.begin() + e.offset, canonical.begin() + e.offset + e.numel, device.begin() + e.device_offset);
}
void ModelBase::to_canonical_order(std::span<const float> device, std::span<float> canonical) const {
  for (const auto& e : manifest())
    std::copy(device.begin() + e.device_offset, device.begin() + e.device_offset + e.numel,
              canonical.begin() + e.offset);
}

// Pre-norm encoder-decoder transformer (model.cpp:36-281). Canonical
// parameter order and init are the reference's exactly (bit-identical
// initial parameters); the device order groups wq|wk|wv and bq|bk|bv of each
// attention block so Q/K/V (self) and K/V (cross) run as one GEMM each.
class TransformerModel : public ModelBase {
 public:
  TransformerModel(const Config& cfg, uint64_t seed)
      : src_vocab_(int(cfg.get_int("src_vocab"))),
        tgt_vocab_(int(cfg.get_int("tgt_vocab"))),
        d_(int(cfg.get_int("d_model"))),
        heads_(int(cfg.get_int("heads"))),
        ffn_(int(cfg.get_int("d_ffn"))),
        max_pos_(int(cfg.get_int("max_positions"))),
        enc_n_(int(cfg.get_int("enc_layers"))),
        dec_n_(int(cfg.get_int("dec_layers"))),
        dropout_(float(cfg.get_real("dropout"))),
        share_(cfg.get_bool("share_embeddings")),
        seed_(seed) {
    if (src_vocab_ < kNumReserved || tgt_vocab_ < kNumReserved)
      throw ConfigError("transformer: vocab sizes must cover the reserved symbols");
    if (d_ <= 0 || heads_ <= 0 || d_ % heads_ != 0)
      throw ConfigError("transformer: d_model must be a positive multiple of heads");
    if (enc_n_ < 1 || dec_n_ < 1) throw ConfigError("transformer: need at least one encoder and one decoder layer");
    if (ffn_ <= 0) throw ConfigError("transformer: d_ffn must be positive");
    if (dropout_ < 0.0f || dropout_ >= 1.0f) throw ConfigError("transformer: dropout must be in [0, 1)");
    if (max_pos_ < 2) throw ConfigError("transformer: max_positions must be at least 2");
    build_layout();
    init_params();
  }

  std::span<float> params() override { return params_; }
  std::span<const float> params() const override { return {params_.data(), params_.size()}; }
  const std::vector<ParamManifestEntry>& manifest() const override { return manifest_; }
  int64_t num_params() const override { return int64_t(params_.size()); }
  int target_vocab() const override { return tgt_vocab_; }
  int max_positions() const override { return max_pos_; }
  std::unique_ptr<ModelBase> clone() const override { return std::make_unique<TransformerModel>(*this); }
  void set_train_step(int64_t s) override { train_step_ = s; }
  void set_inference(bool on) override { inference_ = on; }

  std::vector<float> position_table() const override {
    std::vector<float> pe(size_t(max_pos_) * d_);
    for (int p = 0; p < max_pos_; ++p) positional_row(p, d_, pe.data() + size_t(p) * d_);
    return pe;
  }
  void set_position_table(const float* dev) { pe_dev_ = dev; }

  int forward_to_logits(DeviceTape& tape, const DeviceBatch& b) const override {
    if (b.src_width > max_pos_)
      throw CapacityError("transformer: source length " + std::to_string(b.src_width) + " exceeds max_positions " +
                          std::to_string(max_pos_));
    if (b.tgt_width > max_pos_)
      throw CapacityError("transformer: target length " + std::to_string(b.tgt_width) + " exceeds max_positions " +
                          std::to_string(max_pos_));
    if (!pe_dev_) throw ConfigError("transformer: position table not uploaded");
    int site = 0;  // model.cpp:277-281: one site counter across encoder and decoder
    const int enc = encode(tape, b, site);
    return decode(tape, b, enc, site);
  }

  int decoder_layers() const override { return dec_n_; }
  int model_dim() const override { return d_; }

  int encode_cross_kv(DeviceTape& t, const DeviceBatch& b) const override {
    if (b.src_width > max_pos_)
      throw CapacityError("transformer: source length " + std::to_string(b.src_width) + " exceeds max_positions " +
                          std::to_string(max_pos_));
    if (!pe_dev_) throw ConfigError("transformer: position table not uploaded");
    if (dec_.empty()) throw ConfigError("transformer: no decoder layers");
    int site = 0;
    return t.linear(encode(t, b, site), cross_kv_w_, &cross_kv_b_, false);
  }

  // model.cpp:466-538 (forward_decoder_step): the decoder of decode() for one
  // position, self-attention over the cached keys/values of positions 0..pos
  int decode_step(DeviceTape& t, const int32_t* ids, int rows, int pos, void* self_cache, int cap,
                  const void* cross, int src_width, const int32_t* self_len,
                  const int32_t* src_len) const override {
    if (pos >= max_pos_ || pos >= cap)
      throw CapacityError("transformer: decoding position " + std::to_string(pos) + " exceeds max_positions " +
                          std::to_string(max_pos_));
    if (!pe_dev_) throw ConfigError("transformer: position table not uploaded");
    const size_t es = t.dtype() == SFK_F32 ? 4 : 2;
    const size_t kv_row = size_t(2) * d_ * es, layer_bytes = size_t(rows) * cap * kv_row;
    // width 1: the row's position is the table row the pointer starts at
    int x = t.embedding(tgt_embed_, ids, rows, 1, std::sqrt(float(d_)), pe_dev_ + size_t(pos) * d_,
                        DeviceBatch::Segs{});
    const int ckv = t.external(cross, rows * src_width, 2 * d_ * dec_n_);
    int li = 0;
    for (const Layer& l : dec_) {
      const int z = t.layer_norm(x, l.ln1g, l.ln1b);
      const ParamRef bqkv = l.self.bqkv();
      const int qkv = t.linear(z, l.self.wqkv(), &bqkv, false);
      char* cache = static_cast<char*>(self_cache) + size_t(li) * layer_bytes;
      cuda_check(cudaMemcpy2DAsync(cache + size_t(pos) * kv_row, size_t(cap) * kv_row,
                                   static_cast<const char*>(t.out(qkv)) + size_t(d_) * es, size_t(3) * d_ * es,
                                   kv_row, size_t(rows), cudaMemcpyDeviceToDevice, t.stream()),
                 "kv cache append");
      const int kv = t.external(cache, rows * cap, 2 * d_);
      const int a = t.attention(qkv, 0, kv, 0, d_, d_, heads_, rows, 1, cap, false, self_len);
      x = t.linear(a, l.self.wo, &l.self.bo, false, x);
      const int z2 = t.layer_norm(x, l.ln2g, l.ln2b);
      const int cq = t.linear(z2, l.cross.wq, &l.cross.bq, false);
      const int kc = 2 * d_ * li++;
      const int ca = t.attention(cq, 0, ckv, kc, kc + d_, d_, heads_, rows, 1, src_width, false, src_len);
      x = t.linear(ca, l.cross.wo, &l.cross.bo, false, x);
      const int z3 = t.layer_norm(x, l.ln3g, l.ln3b);
      const int h = t.linear(z3, l.w1, &l.b1, true);
      x = t.linear(h, l.w2, &l.b2, false, x);
    }
    x = t.layer_norm(x, dec_lng_, dec_lnb_);
    return t.logits(x, out_proj_);
  }

 private:
  struct Attn {
    ParamRef wq, wk, wv, wo, bq, bk, bv, bo;
    ParamRef wqkv() const { return {wq.offset, 3 * wq.rows, wq.cols}; }  // device-contiguous
    ParamRef bqkv() const { return {bq.offset, 1, 3 * bq.cols}; }
    ParamRef wkv() const { return {wk.offset, 2 * wk.rows, wk.cols}; }
    ParamRef bkv() const { return {bk.offset, 1, 2 * bk.cols}; }
  };
  struct Layer {
    ParamRef ln1g, ln1b, ln2g, ln2b, ln3g, ln3b, w1, b1, w2, b2;
    Attn self, cross;
  };

  int src_vocab_, tgt_vocab_, d_, heads_, ffn_, max_pos_, enc_n_, dec_n_;
  float dropout_;
  bool inference_ = false;  // generation: no dropout sites
  bool share_;
  uint64_t seed_;
  int64_t train_step_ = 0;
  std::vector<float> params_;
  std::vector<ParamManifestEntry> manifest_;
  ParamRef src_embed_, tgt_embed_, out_proj_, enc_lng_, enc_lnb_, dec_lng_, dec_lnb_;
  ParamRef cross_kv_w_{}, cross_kv_b_{};  // all decoder layers' cross K/V projections, stacked
  std::vector<Layer> enc_, dec_;
  const float* pe_dev_ = nullptr;

  // canonical reservation (model.cpp:62-133); device offsets assigned after
  void build_layout() {
    int64_t off = 0;
    auto res = [&](const std::string& name, int rows, int cols) {
      ParamManifestEntry e;
      e.name = name;
      e.shape = rows == 1 ? std::vector<int>{cols} : std::vector<int>{rows, cols};
      e.offset = off;
      e.numel = int64_t(rows) * cols;
      manifest_.push_back(e);
      off += e.numel;
    };
    auto attn = [&](const std::string& p) {
      for (const char* s : {".wq", ".bq", ".wk", ".bk", ".wv", ".bv", ".wo", ".bo"})
        res(p + s, s[1] == 'w' ? d_ : 1, d_);
    };
    const int d = d_;
    res("src_embed", src_vocab_, d);
    res("tgt_embed", tgt_vocab_, d);
    for (int i = 0; i < enc_n_; ++i) {
      const std::string p = "enc." + std::to_string(i);
      res(p + ".ln1.g", 1, d);
      res(p + ".ln1.b", 1, d);
      attn(p + ".self");
      res(p + ".ln2.g", 1, d);
      res(p + ".ln2.b", 1, d);
      res(p + ".ffn.w1", ffn_, d);
      res(p + ".ffn.b1", 1, ffn_);
      res(p + ".ffn.w2", d, ffn_);
      res(p + ".ffn.b2", 1, d);
    }
    res("enc.ln.g", 1, d);
    res("enc.ln.b", 1, d);
    for (int i = 0; i < dec_n_; ++i) {
      const std::string p = "dec." + std::to_string(i);
      res(p + ".ln1.g", 1, d);
      res(p + ".ln1.b", 1, d);
      attn(p + ".self");
      res(p + ".ln2.g", 1, d);
      res(p + ".ln2.b", 1, d);
      attn(p + ".cross");
      res(p + ".ln3.g", 1, d);
      res(p + ".ln3.b", 1, d);
      res(p + ".ffn.w1", ffn_, d);
      res(p + ".ffn.b1", 1, ffn_);
      res(p + ".ffn.w2", d, ffn_);
      res(p + ".ffn.b2", 1, d);
    }
    res("dec.ln.g", 1, d);
    res("dec.ln.b", 1, d);
    if (!share_) res("out_proj", tgt_vocab_, d);
    params_.assign(size_t(off), 0.0f);

    // device order: canonical, except (1) each attention block is laid out
    // wq wk wv wo bq bk bv bo (weights contiguous, biases contiguous) and (2)
    // the cross-attention K/V projections of all decoder layers form one
    // region right after the encoder -- [wk wv] of layer 0..L-1, then [bk bv]
    // of layer 0..L-1 -- so they are one GEMM over the encoder output in each
    // direction (their gradients complete after the decoder's, before the
    // encoder's, which is where the region sits in reverse device order)
    auto rank = [](const std::string& name) {
      static const char* order[] = {".wq", ".wk", ".wv", ".wo", ".bq", ".bk", ".bv", ".bo"};
      for (int i = 0; i < 8; ++i) {
        const std::string s = order[i];
        if (name.size() > s.size() && name.compare(name.size() - s.size(), s.size(), s) == 0) return i;
      }
      return -1;
    };
    auto is_cross_kv = [&](const std::string& name) {
      const int r = rank(name);
      return name.rfind("dec.", 0) == 0 && name.find(".cross.") != std::string::npos && (r == 1 || r == 2 || r == 5 || r == 6);
    };
    std::vector<size_t> kv_w, kv_b;  // manifest indices of the stacked region, in region order
    for (int l = 0; l < dec_n_; ++l)
      for (const char* s : {".wk", ".wv"}) kv_w.push_back(0), kv_w.back() = [&] {
          const std::string nm = "dec." + std::to_string(l) + ".cross" + s;
          for (size_t j = 0; j < manifest_.size(); ++j)
            if (manifest_[j].name == nm) return j;
          throw ConfigError("transformer: missing parameter " + nm);
        }();
    for (int l = 0; l < dec_n_; ++l)
      for (const char* s : {".bk", ".bv"}) kv_b.push_back(0), kv_b.back() = [&] {
          const std::string nm = "dec." + std::to_string(l) + ".cross" + s;
          for (size_t j = 0; j < manifest_.size(); ++j)
            if (manifest_[j].name == nm) return j;
          throw ConfigError("transformer: missing parameter " + nm);
        }();
    int64_t doff = 0;
    auto place = [&](size_t j) {
      manifest_[j].device_offset = doff;
      doff += manifest_[j].numel;
    };
    for (size_t i = 0; i < manifest_.size();) {
      if (rank(manifest_[i].name) < 0) {
        place(i);
        if (manifest_[i].name == "enc.ln.b") {
          for (size_t j : kv_w) place(j);
          for (size_t j : kv_b) place(j);
        }
        ++i;
        continue;
      }
      for (int r = 0; r < 8; ++r)
        for (size_t j = i; j < i + 8; ++j)
          if (rank(manifest_[j].name) == r && !is_cross_kv(manifest_[j].name)) place(j);
      i += 8;
    }
    auto ref = [&](const std::string& name) {
      for (const auto& e : manifest_)
        if (e.name == name)
          return ParamRef{e.device_offset, e.shape.size() == 1 ? 1 : e.shape[0], e.shape.back()};
      throw ConfigError("transformer: missing parameter " + name);
    };
    auto attn_ref = [&](const std::string& p) {
      return Attn{ref(p + ".wq"), ref(p + ".wk"), ref(p + ".wv"), ref(p + ".wo"),
                  ref(p + ".bq"), ref(p + ".bk"), ref(p + ".bv"), ref(p + ".bo")};
    };
    src_embed_ = ref("src_embed");
    tgt_embed_ = ref("tgt_embed");
    out_proj_ = share_ ? tgt_embed_ : ref("out_proj");
    enc_lng_ = ref("enc.ln.g");
    enc_lnb_ = ref("enc.ln.b");
    dec_lng_ = ref("dec.ln.g");
    dec_lnb_ = ref("dec.ln.b");
    if (dec_n_ > 0) {
      cross_kv_w_ = ParamRef{ref("dec.0.cross.wk").offset, dec_n_ * 2 * d, d};
      cross_kv_b_ = ParamRef{ref("dec.0.cross.bk").offset, 1, dec_n_ * 2 * d};
    }
    for (int i = 0; i < enc_n_; ++i) {
      const std::string p = "enc." + std::to_string(i);
      Layer l;
      l.ln1g = ref(p + ".ln1.g");
      l.ln1b = ref(p + ".ln1.b");
      l.self = attn_ref(p + ".self");
      l.ln2g = ref(p + ".ln2.g");
      l.ln2b = ref(p + ".ln2.b");
      l.w1 = ref(p + ".ffn.w1");
      l.b1 = ref(p + ".ffn.b1");
      l.w2 = ref(p + ".ffn.w2");
      l.b2 = ref(p + ".ffn.b2");
      enc_.push_back(l);
    }
    for (int i = 0; i < dec_n_; ++i) {
      const std::string p = "dec." + std::to_string(i);
      Layer l;
      l.ln1g = ref(p + ".ln1.g");
      l.ln1b = ref(p + ".ln1.b");
      l.self = attn_ref(p + ".self");
      l.ln2g = ref(p + ".ln2.g");
      l.ln2b = ref(p + ".ln2.b");
      l.cross = attn_ref(p + ".cross");
      l.ln3g = ref(p + ".ln3.g");
      l.ln3b = ref(p + ".ln3.b");
      l.w1 = ref(p + ".ffn.w1");
      l.b1 = ref(p + ".ffn.b1");
      l.w2 = ref(p + ".ffn.w2");
      l.b2 = ref(p + ".ffn.b2");
      dec_.push_back(l);
    }
  }

  // model.cpp:135-150: gains 1, biases 0, weights float(0.02 * N(0,1)) in
  // canonical manifest order from RngStream(seed, 0)
  void init_params() {
    RngStream rng(seed_, kStreamInit);
    for (const auto& e : manifest_) {
      const size_t dot = e.name.rfind('.');
      const std::string last = dot == std::string::npos ? e.name : e.name.substr(dot + 1);
      float* p = params_.data() + e.offset;
      if (last == "g") {
        std::fill(p, p + e.numel, 1.0f);
      } else if (last[0] != 'b') {
        for (int64_t i = 0; i < e.numel; ++i) p[i] = static_cast<float>(0.02 * rng.next_normal());
      }
    }
  }

  // model.cpp:199-227
  // model.cpp:156-163: dropout site n of the step draws from stream
  // kStreamDropoutBase | (train_step << 8) | n; sites count in recording order
  int maybe_dropout(DeviceTape& t, int x, int& site, int residual = -1) const {
    if (dropout_ <= 0.0f || inference_) return x;
    const uint64_t stream = (uint64_t(1) << 32) | (uint64_t(train_step_) << 8) | uint64_t(site++);
    return t.dropout(x, dropout_, seed_, stream, residual);
  }
  // x + dropout(linear(in)): the residual add rides in the GEMM epilogue when
  // there is no dropout, else in the dropout kernel (model.cpp:218-224)
  int residual(DeviceTape& t, int in, const ParamRef& w, const ParamRef* b, bool relu, int x, int& site) const {
    if (dropout_ <= 0.0f || inference_) return t.linear(in, w, b, relu, x);
    return maybe_dropout(t, t.linear(in, w, b, relu), site, x);
  }

  // a pass over several packed batches (DeviceBatch parts): the embedding
  // and attention run per part, every row-wise op over all rows at once
  static std::vector<DeviceTape::EmbSpan> emb_spans(const DeviceBatch& b, bool src) {
    std::vector<DeviceTape::EmbSpan> v;
    for (int k = 0; k < b.parts(); ++k) {
      const DeviceBatch::Part pt = b.get_part(k);
      const int w = src ? pt.src_width : pt.tgt_width;
      v.push_back({src ? pt.src_pos0 : pt.tgt_pos0, pt.rows * w, w});
    }
    return v;
  }
  enum class Span { Source, Target, Cross };
  static std::vector<DeviceTape::AttnPart> attn_parts(const DeviceBatch& b, Span sp) {
    std::vector<DeviceTape::AttnPart> v;
    for (int k = 0; k < b.parts(); ++k) {
      const DeviceBatch::Part pt = b.get_part(k);
      if (sp == Span::Source)
        v.push_back({pt.rows, pt.src_width, pt.src_width, pt.src_pos0, pt.src_pos0, pt.src_lens});
      else if (sp == Span::Target)
        v.push_back({pt.rows, pt.tgt_width, pt.tgt_width, pt.tgt_pos0, pt.tgt_pos0, nullptr});
      else
        v.push_back({pt.rows, pt.tgt_width, pt.src_width, pt.tgt_pos0, pt.src_pos0, pt.src_lens});
    }
    return v;
  }

  int encode(DeviceTape& t, const DeviceBatch& b, int& site) const {
    const auto spans = emb_spans(b, true);
    const auto parts = attn_parts(b, Span::Source);
    int x = t.embedding(src_embed_, b.source, int(b.src_positions()), spans, std::sqrt(float(d_)), pe_dev_,
                        b.src_segs);
    x = maybe_dropout(t, x, site);
    for (const Layer& l : enc_) {
      const int z = t.layer_norm(x, l.ln1g, l.ln1b);
      const ParamRef bqkv = l.self.bqkv();
      const int qkv = t.linear(z, l.self.wqkv(), &bqkv, false);
      const int a = t.attention(qkv, 0, qkv, d_, 2 * d_, d_, heads_, parts, false);
      x = residual(t, a, l.self.wo, &l.self.bo, false, x, site);
      const int z2 = t.layer_norm(x, l.ln2g, l.ln2b);
      const int h = t.linear(z2, l.w1, &l.b1, true);
      x = residual(t, h, l.w2, &l.b2, false, x, site);
    }
    return t.layer_norm(x, enc_lng_, enc_lnb_);
  }

  // model.cpp:229-275
  int decode(DeviceTape& t, const DeviceBatch& b, int enc, int& site) const {
    const auto self_parts = attn_parts(b, Span::Target);
    const auto cross_parts = attn_parts(b, Span::Cross);
    int x = t.embedding(tgt_embed_, b.target_in, int(b.tgt_positions()), emb_spans(b, false), std::sqrt(float(d_)),
                        pe_dev_, b.tgt_segs);
    x = maybe_dropout(t, x, site);
    // cross K/V of every decoder layer from the encoder output in one GEMM
    // (model.cpp:262-263 per layer; same dot products, batched)
    const int ckv_all = dec_.empty() ? -1 : t.linear(enc, cross_kv_w_, &cross_kv_b_, false);
    int li = 0;
    for (const Layer& l : dec_) {
      const int z = t.layer_norm(x, l.ln1g, l.ln1b);
      const ParamRef bqkv = l.self.bqkv();
      const int qkv = t.linear(z, l.self.wqkv(), &bqkv, false);
      const int a = t.attention(qkv, 0, qkv, d_, 2 * d_, d_, heads_, self_parts, true);
      x = residual(t, a, l.self.wo, &l.self.bo, false, x, site);
      const int z2 = t.layer_norm(x, l.ln2g, l.ln2b);
      const int cq = t.linear(z2, l.cross.wq, &l.cross.bq, false);
      const int kc = 2 * d_ * li++;
      const int ca = t.attention(cq, 0, ckv_all, kc, kc + d_, d_, heads_, cross_parts, false);
      x = residual(t, ca, l.cross.wo, &l.cross.bo, false, x, site);
      const int z3 = t.layer_norm(x, l.ln3g, l.ln3b);
      const int h = t.linear(z3, l.w1, &l.b1, true);
      x = residual(t, h, l.w2, &l.b2, false, x, site);
    }
    x = t.layer_norm(x, dec_lng_, dec_lnb_);
    return t.logits(x, out_proj_);
  }
};

void set_model_position_table(ModelBase& m, const float* dev) {
  if (auto* t = dynamic_cast<TransformerModel*>(&m)) t->set_position_table(dev);
}

// ------------------------------------------------------------------ criterions
// criterions.cpp:10-54: gold = target_out, active = gold != pad, SUM reduction
class XentCriterion : public CriterionBase {
 public:
  explicit XentCriterion(double eps) : eps_(float(eps)) {
    if (eps < 0.0 || eps >= 1.0) throw ConfigError("label_smoothed_cross_entropy: epsilon must be in [0, 1)");
  }
  CriterionOutput compute(ModelBase& model, const DeviceBatch& b, DeviceTape& tape) override {
    const int logits = model.forward_to_logits(tape, b);
    CriterionOutput out;
    out.loss_node = tape.softmax_xent(logits, b.target_out, eps_);
    return out;
  }

 private:
  float eps_;
};

// ------------------------------------------------------------------ optimizers
class AdamOptimizer : public OptimizerBase {
 public:
  AdamOptimizer(int64_t n, double b1, double b2, double eps) : n_(n), b1_(b1), b2_(b2), eps_(eps) {
    if (n < 0) throw ConfigError("adam: negative parameter count");
    if (b1 < 0 || b1 >= 1 || b2 < 0 || b2 >= 1) throw ConfigError("adam: betas must be in [0, 1)");
    if (eps <= 0) throw ConfigError("adam: eps must be positive");
  }
  ~AdamOptimizer() override {
    cudaFree(m_);
    cudaFree(v_);
  }
  void apply(float* master, void* shadow, int shadow_dtype, const void* grad, int grad_dtype, int64_t n, double lr,
             const GradPrep& prep, void* stream) override {
    if (n != n_) throw ShapeError("adam: moment/parameter length mismatch");
    ensure(static_cast<cudaStream_t>(stream));
    ++t_;
    const double bc1 = 1.0 - std::pow(b1_, double(t_));
    const double bc2 = 1.0 - std::pow(b2_, double(t_));
    if (!prep.ranges) {
      sfk_check(sfk_adam(grad_dtype, master, shadow, shadow_dtype, grad, m_, v_, n, lr, b1_, b2_, eps_, bc1, bc2,
                         prep.scale, prep.unscale ? 1 : 0, prep.ntokens, prep.skip, stream),
                "adam");
      return;
    }
    const size_t gs = grad_dtype == SFK_F32 ? 4 : 2, ss = shadow_dtype == SFK_F32 ? 4 : 2;
    for (size_t i = 0; i < prep.ranges->size(); ++i) {
      const auto [off, cnt] = (*prep.ranges)[i];
      sfk_check(sfk_adam(grad_dtype, master + off, shadow ? static_cast<char*>(shadow) + off * ss : nullptr,
                         shadow_dtype, static_cast<const char*>(grad) + off * gs, m_ + off, v_ + off, cnt, lr, b1_, b2_,
                         eps_, bc1, bc2, prep.scale, prep.unscale ? 1 : 0, prep.ntokens, prep.skip, stream),
                "adam");
      if (prep.range_done)
        cuda_check(cudaEventRecord((*prep.range_done)[i], static_cast<cudaStream_t>(stream)), "adam range event");
    }
  }
  int64_t step_count() const override { return t_; }
  void set_step_count(int64_t t) override { t_ = t; }
  std::vector<std::pair<std::string, std::vector<float>>> state_blobs() const override {
    std::vector<float> m(size_t(n_), 0.f), v(size_t(n_), 0.f);
    if (m_) {
      // the update may still be running on a trainer stream: join the device
      cuda_check(cudaDeviceSynchronize(), "adam state");
      cuda_check(cudaMemcpy(m.data(), m_, size_t(n_) * 4, cudaMemcpyDeviceToHost), "adam state");
      cuda_check(cudaMemcpy(v.data(), v_, size_t(n_) * 4, cudaMemcpyDeviceToHost), "adam state");
    }
    return {{"adam.m", m}, {"adam.v", v}};
  }
  void load_state_blobs(const std::vector<std::pair<std::string, std::vector<float>>>& blobs) override {
    bool gm = false, gv = false;
    // no pending update may land after the load; the legacy-stream copies
    // below are joined before any trainer stream reads the moments
    cuda_check(cudaDeviceSynchronize(), "adam load");
    ensure(nullptr);
    for (const auto& [name, data] : blobs) {
      if (data.size() != size_t(n_)) throw IntegrityError("adam: moment size mismatch");
      if (name == "adam.m") {
        cuda_check(cudaMemcpy(m_, data.data(), size_t(n_) * 4, cudaMemcpyHostToDevice), "adam load");
        gm = true;
      } else if (name == "adam.v") {
        cuda_check(cudaMemcpy(v_, data.data(), size_t(n_) * 4, cudaMemcpyHostToDevice), "adam load");
        gv = true;
      } else {
        throw IntegrityError("adam: unknown state blob '" + name + "'");
      }
    }
    cuda_check(cudaDeviceSynchronize(), "adam load");
    if (!gm || !gv) throw IntegrityError("adam: missing moment blobs");
  }

 private:
  int64_t n_;
  double b1_, b2_, eps_;
  int64_t t_ = 0;
  float* m_ = nullptr;
  float* v_ = nullptr;
  // zeroed on the stream the first update runs on (or joined when called
  // outside a step), so the update never reads uncleared moments
  void ensure(cudaStream_t s) {
    if (m_) return;
    cuda_check(cudaMalloc(&m_, size_t(std::max<int64_t>(n_, 1)) * 4), "adam m");
    cuda_check(cudaMalloc(&v_, size_t(std::max<int64_t>(n_, 1)) * 4), "adam v");
    cuda_check(cudaMemsetAsync(m_, 0, size_t(n_) * 4, s), "adam m");
    cuda_check(cudaMemsetAsync(v_, 0, size_t(n_) * 4, s), "adam v");
    if (!s) cuda_check(cudaDeviceSynchronize(), "adam zero");
  }
};

class SgdOptimizer : public OptimizerBase {
 public:
  void apply(float* master, void* shadow, int shadow_dtype, const void* grad, int grad_dtype, int64_t n, double lr,
             const GradPrep& prep, void* stream) override {
    sfk_check(sfk_sgd(grad_dtype, master, shadow, shadow_dtype, grad, n, lr, prep.scale, prep.unscale ? 1 : 0,
                      prep.ntokens, prep.skip, stream),
              "sgd");
    ++t_;
  }
  int64_t step_count() const override { return t_; }
  void set_step_count(int64_t t) override { t_ = t; }
  std::vector<std::pair<std::string, std::vector<float>>> state_blobs() const override { return {}; }
  void load_state_blobs(const std::vector<std::pair<std::string, std::vector<float>>>& b) override {
    if (!b.empty()) throw IntegrityError("sgd: unexpected optimizer state blobs");
  }

 private:
  int64_t t_ = 0;
};

// ------------------------------------------------------------------ schedulers (optim.cpp:75-137)
class FixedSchedule : public SchedulerBase {
 public:
  explicit FixedSchedule(double lr) : lr_(lr) {
    if (lr <= 0) throw ConfigError("scheduler: base lr must be positive");
  }
  double lr(int64_t) const override { return lr_; }

 private:
  double lr_;
};

class InverseSqrtSchedule : public SchedulerBase {
 public:
  InverseSqrtSchedule(double base, int64_t warmup, double init) : base_(base), init_(init), warmup_(warmup) {
    if (base <= 0) throw ConfigError("scheduler: base lr must be positive");
    if (warmup < 0) throw ConfigError("inverse_sqrt: warmup must be >= 0");
    if (init < 0) throw ConfigError("inverse_sqrt: warmup_init_lr must be >= 0");
  }
  double lr(int64_t step) const override {
    if (step < 1) throw BoundsError("scheduler: step must be >= 1");
    if (step <= warmup_) return init_ + (base_ - init_) * double(step) / double(warmup_);
    const double w = double(warmup_ > 0 ? warmup_ : 1);
    return base_ * std::sqrt(w / double(step));
  }

 private:
  double base_, init_;
  int64_t warmup_;
};

class CosineRestartSchedule : public SchedulerBase {
 public:
  CosineRestartSchedule(double base, double eta_min, int64_t period, double t_mult)
      : base_(base), eta_min_(eta_min), t_mult_(t_mult), period_(period) {
    if (base <= 0) throw ConfigError("scheduler: base lr must be positive");
    if (eta_min < 0 || eta_min > base) throw ConfigError("cosine_restart: eta_min must be in [0, base_lr]");
    if (period < 1) throw ConfigError("cosine_restart: period must be >= 1");
    if (t_mult < 1) throw ConfigError("cosine_restart: t_mult must be >= 1");
  }
  double lr(int64_t step) const override {
    if (step < 1) throw BoundsError("scheduler: step must be >= 1");
    double cur = double(step - 1), len = double(period_);
    while (cur >= len) {
      cur -= len;
      len *= t_mult_;
    }
    return eta_min_ + 0.5 * (base_ - eta_min_) * (1.0 + std::cos(3.14159265358979323846 * cur / len));
  }

 private:
  double base_, eta_min_, t_mult_;
  int64_t period_;
};

// ------------------------------------------------------------------ tasks
// "synthetic": the WMT-shaped generator of SURVEY §8(d), in memory
class SyntheticTask : public TaskBase {
 public:
  explicit SyntheticTask(const Config& cfg) {
    sv_ = int(cfg.get_int("src_vocab"));
    tv_ = int(cfg.get_int("tgt_vocab"));
    if (sv_ == 0 || tv_ == 0) throw ConfigError("synthetic: src_vocab and tgt_vocab must be set");
    const int64_t n = cfg.get_int("synthetic_pairs");
    if (n <= 0) throw ConfigError("synthetic: synthetic_pairs must be positive");
    pairs_ = synthetic_corpus(int(n), sv_, tv_, cfg.get_real("zipf_s"), uint64_t(cfg.get_int("seed")));
  }
  int source_vocab() const override { return sv_; }
  int target_vocab() const override { return tv_; }
  const std::vector<SequencePair>& train_pairs() const override { return pairs_; }

 private:
  int sv_, tv_;
  std::vector<SequencePair> pairs_;
};

void register_builtins(Registry& r) {
  r.register_model(
      "transformer",
      [](const Config& cfg, uint64_t seed) -> std::unique_ptr<ModelBase> {
        return std::make_unique<TransformerModel>(cfg, seed);
      },
      transformer_default_config());

  auto arch = [&](const char* name, std::vector<std::pair<std::string, ConfigValue>> ov) {
    ArchitectureDef a;
    a.name = name;
    a.base_model = "transformer";
    a.overrides = std::move(ov);
    r.register_architecture(std::move(a));
  };
  // builtins.cpp:21-30
  arch("tiny_transformer", {{"d_model", int64_t{16}},
                            {"heads", int64_t{2}},
                            {"enc_layers", int64_t{1}},
                            {"dec_layers", int64_t{1}},
                            {"d_ffn", int64_t{32}},
                            {"max_positions", int64_t{64}},
                            {"share_embeddings", true}});
  // BASELINE.json configs C1-C5 over the same pre-norm transformer
  auto bench = [&](const char* name, int64_t d, int64_t h, int64_t L, int64_t f) {
    arch(name, {{"d_model", d},
                {"heads", h},
                {"enc_layers", L},
                {"dec_layers", L},
                {"d_ffn", f},
                {"max_positions", int64_t{256}},
                {"share_embeddings", false}});
  };
  bench("transformer_base_defaults", 64, 4, 2, 128);
  bench("transformer_iwslt_de_en", 512, 4, 6, 1024);
  bench("transformer_wmt_en_de", 512, 8, 6, 2048);
  bench("transformer_vaswani_wmt_en_de_big", 1024, 16, 6, 4096);

  r.register_criterion("cross_entropy",
                       [](const Config&) -> std::unique_ptr<CriterionBase> { return std::make_unique<XentCriterion>(0.0); });
  r.register_criterion("label_smoothed_cross_entropy", [](const Config& cfg) -> std::unique_ptr<CriterionBase> {
    return std::make_unique<XentCriterion>(cfg.get_real("label_smoothing"));
  });
  r.register_task("translation",
                  [](const Config& cfg) -> std::unique_ptr<TaskBase> { return std::make_unique<TranslationTask>(cfg); });
  r.register_task("synthetic",
                  [](const Config& cfg) -> std::unique_ptr<TaskBase> { return std::make_unique<SyntheticTask>(cfg); });
  r.register_optimizer("sgd", [](const Config&, int64_t) -> std::unique_ptr<OptimizerBase> {
    return std::make_unique<SgdOptimizer>();
  });
  r.register_optimizer("adam", [](const Config& cfg, int64_t n) -> std::unique_ptr<OptimizerBase> {
    return std::make_unique<AdamOptimizer>(n, cfg.get_real("adam_beta1"), cfg.get_real("adam_beta2"),
                                           cfg.get_real("adam_eps"));
  });
  r.register_scheduler("fixed", [](const Config& cfg) -> std::unique_ptr<SchedulerBase> {
    return std::make_unique<FixedSchedule>(cfg.get_real("lr"));
  });
  r.register_scheduler("inverse_sqrt", [](const Config& cfg) -> std::unique_ptr<SchedulerBase> {
    return std::make_unique<InverseSqrtSchedule>(cfg.get_real("lr"), cfg.get_int("warmup"),
                                                 cfg.get_real("warmup_init_lr"));
  });
  r.register_scheduler("cosine_restart", [](const Config& cfg) -> std::unique_ptr<SchedulerBase> {
    return std::make_unique<CosineRestartSchedule>(cfg.get_real("lr"), cfg.get_real("eta_min"),
                                                   cfg.get_int("cosine_period"), cfg.get_real("cosine_t_mult"));
  });
}

Registry& global_registry() {
  static Registry reg = [] {
    Registry r;
    register_builtins(r);
    return r;
  }();
  return reg;
}

}  // namespace sqf

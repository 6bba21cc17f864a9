#include "device_tape.hpp"

#include <algorithm>
#include <tuple>
#include <cstdlib>
#include <cstring>

namespace sqf {

// Measured scheduling knobs (defaults are the measured-best settings; see
// DESIGN.md §5): SQF_WGRAD_TILE=0 restores the wave-efficiency tile choice for
// the side-stream weight-gradient GEMMs.
static int tile_env() {
  static const int v = [] {
    const char* e = std::getenv("SQF_WGRAD_TILE");
    return e ? std::atoi(e) : 1;
  }();
  return v;
}

// SQF_LN_FUSED=1: one-pass LN backward (dx + gamma/beta partials on the main stream)
// SQF_ABLATE (measurement only, results are wrong): bit mask of kernel
// classes whose launches are skipped, to read each class's share of the real
// concurrent step from the step-time difference. 1 LN fwd, 2 LN dx, 4 LN
// gamma/beta, 8 attention fwd, 16 attention bwd, 32 xent.
int ablate_mask() {
  static const int m = [] {
    const char* e = std::getenv("SQF_ABLATE");
    return e ? std::atoi(e) : 0;
  }();
  return m;
}

static bool ln_fused_env() {
  static const bool v = [] {
    const char* e = std::getenv("SQF_LN_FUSED");
    return e && std::atoi(e) != 0;
  }();
  return v;
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}
void sfk_check(int status, const char* what) {
  if (status != SFK_OK) throw DeviceError(std::string(what) + " failed: " + sfk_last_error());
}

// ------------------------------------------------------------------ arena
Arena::~Arena() {
  for (auto& c : chunks_) cudaFree(c.base);
}

void* Arena::alloc(size_t bytes) {
  bytes = (bytes + 255) & ~size_t(255);
  while (cur_ < chunks_.size() && chunks_[cur_].used + bytes > chunks_[cur_].size) ++cur_;
  if (cur_ == chunks_.size()) {
    size_t sz = std::max(bytes, size_t(256) << 20);
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, sz), "arena cudaMalloc");
    chunks_.push_back({static_cast<char*>(p), sz, 0});
  }
  Chunk& c = chunks_[cur_];
  void* out = c.base + c.used;
  c.used += bytes;
  return out;
}

void Arena::reset() {
  // A sub-batch that needed more than one chunk means the arena is still
  // growing: merge everything into one chunk of the combined size, so a
  // workload settles after a few sub-batches instead of allocating whenever
  // the (first-fit, forward-only) cursor skips past a chunk. cudaFree waits
  // for the device, so no in-flight kernel still uses the old chunks.
  if (chunks_.size() > 1) {
    size_t total = 0;
    for (auto& c : chunks_) total += c.size;
    for (auto& c : chunks_) cuda_check(cudaFree(c.base), "arena cudaFree");
    chunks_.clear();
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, total), "arena cudaMalloc");
    chunks_.push_back({static_cast<char*>(p), total, 0});
  }
  for (auto& c : chunks_) c.used = 0;
  cur_ = 0;
}

size_t Arena::capacity() const {
  size_t s = 0;
  for (const auto& c : chunks_) s += c.size;
  return s;
}

// ------------------------------------------------------------------ profiler
const char* Profiler::name(int c) {
  static const char* n[] = {"gemm_fwd", "gemm_dgrad", "gemm_wgrad", "attn_fwd", "attn_bwd",
                            "layernorm", "xent", "embed", "bias_grad", "optim"};
  return c >= 0 && c < kCats ? n[c] : "?";
}
Profiler::~Profiler() {
  for (auto e : pool_) cudaEventDestroy(e);
}
cudaEvent_t Profiler::get() {
  if (next_ == pool_.size()) {
    cudaEvent_t e;
    cuda_check(cudaEventCreate(&e), "profiler event");
    pool_.push_back(e);
  }
  return pool_[next_++];
}
void Profiler::begin(cudaStream_t s) {
  open_ = get();
  cuda_check(cudaEventRecord(open_, s), "profiler record");
}
void Profiler::end(cudaStream_t s, int cat, double fl, double by) {
  cudaEvent_t b = get();
  cuda_check(cudaEventRecord(b, s), "profiler record");
  pending_.push_back({open_, b, cat, fl, by, s});
}
void Profiler::mark_base(cudaStream_t s) {
  base_ = get();
  cuda_check(cudaEventRecord(base_, s), "profiler record");
}
void Profiler::collect() {
  for (const Rec& r : pending_) {
    cuda_check(cudaEventSynchronize(r.b), "profiler sync");
    float t = 0.f;
    cuda_check(cudaEventElapsedTime(&t, r.a, r.b), "profiler elapsed");
    if (base_) {
      int si = 0;
      while (si < int(streams.size()) && streams[size_t(si)] != r.s) ++si;
      if (si == int(streams.size())) streams.push_back(r.s);
      float t0 = 0.f, t1 = 0.f;
      cuda_check(cudaEventElapsedTime(&t0, base_, r.a), "profiler elapsed");
      cuda_check(cudaEventElapsedTime(&t1, base_, r.b), "profiler elapsed");
      spans.push_back({si, r.cat, t0, t1});
    }
    ms[r.cat] += t;
    flops[r.cat] += r.flops;
    bytes[r.cat] += r.bytes;
    count[r.cat] += 1;
  }
  pending_.clear();
  next_ = 0;
  base_ = nullptr;
}
void Profiler::reset() {
  pending_.clear();
  spans.clear();
  base_ = nullptr;
  next_ = 0;
  for (int c = 0; c < kCats; ++c) ms[c] = flops[c] = bytes[c] = 0, count[c] = 0;
}

// ------------------------------------------------------------------ batch packing
namespace {
// recording-order segments for the embedding backward: unique ids ascending,
// each with its rows in ascending (= recording) order
void build_segments(const std::vector<int>& ids, std::vector<int32_t>& uniq, std::vector<int32_t>& off,
                    std::vector<int32_t>& rows) {
  std::vector<int32_t> order(ids.size());
  for (size_t i = 0; i < ids.size(); ++i) order[i] = int32_t(i);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return ids[a] < ids[b]; });
  uniq.clear();
  off.clear();
  rows.assign(order.begin(), order.end());
  for (size_t i = 0; i < order.size(); ++i) {
    if (i == 0 || ids[order[i]] != ids[order[i - 1]]) {
      uniq.push_back(ids[order[i]]);
      off.push_back(int32_t(i));
    }
  }
  off.push_back(int32_t(order.size()));
}

// chunk tables of sfk_embed_bwd_chunked: segments cut into <= 16-row chunks
void build_chunks(const std::vector<int32_t>& uniq, const std::vector<int32_t>& off, std::vector<int32_t>& chunks,
                  std::vector<int32_t>& multi, int& nslots) {
  constexpr int kChunk = 16;
  chunks.clear();
  multi.clear();
  nslots = 0;
  for (size_t u = 0; u < uniq.size(); ++u) {
    const int s0 = off[u], s1 = off[u + 1];
    const int n = (s1 - s0 + kChunk - 1) / kChunk;
    if (n == 1) {
      chunks.insert(chunks.end(), {uniq[u], s0, s1, -1});
      continue;
    }
    multi.insert(multi.end(), {uniq[u], nslots, n, 0});
    for (int c = 0; c < n; ++c) chunks.insert(chunks.end(), {uniq[u], s0 + c * kChunk, std::min(s1, s0 + (c + 1) * kChunk), nslots++});
  }
}
}  // namespace

PackedBatch PackedBatch::pack(const MiniBatch& b) {
  PackedBatch p;
  p.rows = b.rows;
  p.src_width = b.src_width;
  p.tgt_width = b.tgt_width;
  p.ntokens = b.ntokens;
  p.parts = b.parts;
  std::vector<int32_t> su, so, sr, tu, to, tr;
  build_segments(b.source, su, so, sr);
  build_segments(b.target_in, tu, to, tr);
  std::vector<int32_t> sc, sm, tc, tm;
  build_chunks(su, so, sc, sm, p.n_ss);
  build_chunks(tu, to, tc, tm, p.n_ts);
  auto put = [&](const auto& v) {
    const size_t at = p.blob.size();
    p.blob.insert(p.blob.end(), v.begin(), v.end());
    while (p.blob.size() % 4) p.blob.push_back(0);  // 16-byte aligned sections
    return at;
  };
  p.off_source = put(b.source);
  p.off_tin = put(b.target_in);
  p.off_tout = put(b.target_out);
  p.off_slens = put(b.src_lens);
  p.off_su = put(su);
  p.off_so = put(so);
  p.off_sr = put(sr);
  p.off_tu = put(tu);
  p.off_to = put(to);
  p.off_tr = put(tr);
  p.off_sc = put(sc);
  p.off_sm = put(sm);
  p.off_tc = put(tc);
  p.off_tm = put(tm);
  p.n_su = int(su.size());
  p.n_tu = int(tu.size());
  p.n_sc = int(sc.size() / 4);
  p.n_sm = int(sm.size() / 4);
  p.n_tc = int(tc.size() / 4);
  p.n_tm = int(tm.size() / 4);
  return p;
}

int64_t DeviceBatch::src_positions() const {
  int64_t n = 0;
  for (int k = 0; k < parts(); ++k) n += int64_t(get_part(k).rows) * get_part(k).src_width;
  return n;
}

int64_t DeviceBatch::tgt_positions() const {
  int64_t n = 0;
  for (int k = 0; k < parts(); ++k) n += int64_t(get_part(k).rows) * get_part(k).tgt_width;
  return n;
}

DeviceBatch PackedBatch::bind(const int32_t* d) const {
  DeviceBatch b;
  b.rows = rows;
  b.src_width = src_width;
  b.tgt_width = tgt_width;
  b.ntokens = ntokens;
  b.source = d + off_source;
  b.target_in = d + off_tin;
  b.target_out = d + off_tout;
  b.src_lens = d + off_slens;
  b.src_segs = {d + off_su, d + off_so, d + off_sr, n_su, d + off_sc, d + off_sm, n_sc, n_sm, n_ss};
  b.tgt_segs = {d + off_tu, d + off_to, d + off_tr, n_tu, d + off_tc, d + off_tm, n_tc, n_tm, n_ts};
  if (parts.size() > 1) {
    if (parts.size() > size_t(DeviceBatch::kMaxParts)) throw ShapeError("packed batch: too many parts");
    b.nparts = int(parts.size());
    int row = 0;
    int64_t sp = 0, tp = 0;
    for (size_t k = 0; k < parts.size(); ++k) {
      const auto& [r, sw, tw] = parts[k];
      b.part[k] = DeviceBatch::Part{r, sw, tw, sp, tp, b.src_lens + row};
      row += r;
      sp += int64_t(r) * sw;
      tp += int64_t(r) * tw;
    }
  }
  return b;
}

// ------------------------------------------------------------------ tape
DeviceTape::DeviceTape(Arena& arena, const DeviceParams& params, int dtype, cudaStream_t stream)
    : arena_(arena), params_(params), dtype_(dtype), esize_(dtype == SFK_F32 ? 4 : 2), stream_(stream), cur_(stream) {}

int DeviceTape::embedding(ParamRef table, const int32_t* ids, int rows, int width, float scale, const float* pe,
                          const DeviceBatch::Segs& segs) {
  return embedding(table, ids, rows, {EmbSpan{0, rows, width}}, scale, pe, segs);
}

int DeviceTape::embedding(ParamRef table, const int32_t* ids, int rows, const std::vector<EmbSpan>& spans, float scale,
                          const float* pe, const DeviceBatch::Segs& segs) {
  int64_t covered = 0;
  for (const EmbSpan& sp : spans) {
    if (sp.row0 != covered || sp.width <= 0 || sp.rows % sp.width) throw ShapeError("embedding: span layout mismatch");
    covered += sp.rows;
  }
  if (covered != rows) throw ShapeError("embedding: span layout mismatch");
  Node n;
  n.kind = Kind::Embedding;
  n.p0 = table;
  n.ids = ids;
  n.rows = rows;
  n.cols = table.cols;
  n.width = spans.size() == 1 ? spans[0].width : 0;
  n.espans = spans;
  n.scale = scale;
  n.segs = segs;
  n.out = alloc_elems(int64_t(rows) * n.cols);
  for (const EmbSpan& sp : spans) {
    pbegin();
    sfk_check(sfk_embed_fwd(dtype_, ids + sp.row0, sp.rows, sp.width, n.cols, pptr(table), pe, scale,
                            static_cast<char*>(n.out) + sp.row0 * n.cols * int64_t(esize_), cur_),
              "embed_fwd");
    pend(Profiler::Embed, 0, double(sp.rows) * n.cols * (2.0 * esize_ + 4));
    ++launches_;
  }
  nodes_.push_back(n);
  return int(nodes_.size()) - 1;
}

int DeviceTape::layer_norm(int x, ParamRef gamma, ParamRef beta) {
  const Node& in = nodes_[x];
  if (gamma.cols != in.cols || beta.cols != in.cols) throw ShapeError("layer_norm: affine parameter length mismatch");
  Node n;
  n.kind = Kind::LayerNorm;
  n.in0 = x;
  n.p0 = gamma;
  n.p1 = beta;
  n.rows = in.rows;
  n.cols = in.cols;
  n.out = alloc_elems(int64_t(n.rows) * n.cols);
  n.stats = static_cast<float*>(arena_.alloc(size_t(n.rows) * 8));
  pbegin();
  if (!(ablate_mask() & 1))
  sfk_check(sfk_layernorm_fwd(dtype_, in.out, n.rows, n.cols, pptr(gamma), pptr(beta), n.out, n.stats, cur_),
            "layernorm_fwd");
  pend(Profiler::LayerNorm, 0, double(n.rows) * (2.0 * n.cols * esize_ + 8));
  ++launches_;
  nodes_.push_back(n);
  return int(nodes_.size()) - 1;
}

void DeviceTape::gemm(int cat, int m, int n, int k, const void* a, int64_t lda, bool a_kmajor, const void* b,
                      int64_t ldb, bool b_kmajor, void* c, int64_t ldc, int flags, const void* bias, const void* res,
                      int64_t ldr, const void* mask, int64_t ldm, void* bias_grad) {
  sfk_gemm_args g{};
  g.m = m;
  g.n = n;
  g.k = k;
  g.dtype = dtype_;
  g.a = a;
  g.lda = lda;
  g.a_kmajor = a_kmajor;
  g.b = b;
  g.ldb = ldb;
  g.b_kmajor = b_kmajor;
  g.c = c;
  g.ldc = ldc;
  g.bias = bias;
  g.res = res;
  g.ldr = ldr;
  g.mask = mask;
  g.ldm = ldm;
  g.flags = flags;
  g.bias_grad = bias_grad;
  // parameter-gradient GEMMs run on the side stream, concurrently with the
  // activation-gradient chain: what counts there is work per SM-cycle, not
  // latency, so they always take the widest (most operand-efficient) tile
  if (cat == Profiler::GemmWgrad && cur_ == side_ && side_ && tile_env() != 0) g.tile_n = 256;
  // weight gradients take CTA-pair tiles too (the fused bias gradient works in
  // both kernels; measured 119.6 vs 121.6 ms/step on C4; SQF_WGRAD_PAIR=0 off)
  static const int wpair_env = [] {
    const char* e = std::getenv("SQF_WGRAD_PAIR");
    return e ? std::atoi(e) : 1;
  }();
  if (wpair_env && cat == Profiler::GemmWgrad && m >= 512 && dtype_ != SFK_F32) {
    g.pair = 1;
    g.tile_n = 256;
  }
  // CTA-pair (cta_group::2, 256 x 256) tiles for the main-stream GEMMs: half
  // the per-SM operand traffic of 128 x 256 (measured 128.1 vs 131.1 ms/step
  // on C4); SQF_PAIR=0 switches back to single-CTA tiles
  static const int pair_env = [] {
    const char* e = std::getenv("SQF_PAIR");
    return e ? std::atoi(e) : 1;
  }();
  // SQF_PAIR_BN: 256 (default) always 256-wide pair tiles; -S picks 128 when its
  // wave efficiency beats 256's by more than S percent (0: any gain)
  static const int pair_bn = [] {
    const char* e = std::getenv("SQF_PAIR_BN");
    return e ? std::atoi(e) : 256;
  }();
  if (pair_env && cat != Profiler::GemmWgrad && m >= 512 && dtype_ != SFK_F32) {
    g.pair = 1;
    g.tile_n = pair_bn;
  }
  // SQF_SIDE_MAX_SMS / SQF_MAIN_MAX_SMS: cap the SMs a GEMM's persistent
  // tile loop takes on the side stream / on the stream the tape records
  // on (forward-ahead or main), leaving SMs to the other streams (0 = all)
  static const int side_max = [] {
    const char* e = std::getenv("SQF_SIDE_MAX_SMS");
    return e ? std::atoi(e) : 0;
  }();
  static const int main_max = [] {
    const char* e = std::getenv("SQF_MAIN_MAX_SMS");
    return e ? std::atoi(e) : 0;
  }();
  g.max_sms = cur_ == side_ && side_ ? side_max : main_max;
  float* ws = cur_ == stream_ ? ws_main_ : cur_ == side_ ? ws_side_ : nullptr;
  static const int sk_mode = [] {
    const char* v = std::getenv("SQF_GEMM_STREAM_K");  // 0 off (default), 1 auto, 2 force
    return v ? std::atoi(v) : 0;
  }();
  const int sk = sk_override_ ? sk_override_ : sk_mode;
  // SQF_PAIR_SK=1: CTA-pair GEMMs may split the last wave stream-K style
  // (sfk_gemm decides per shape). Off by default: measured slower on every
  // C4 shape so far (fp32 partial round trips cost more than the idle tail)
  static const int pair_sk = [] {
    const char* v = std::getenv("SQF_PAIR_SK");
    return v ? std::atoi(v) : 0;
  }();
  if (ws && ctr_base_ && (sk > 0 || (g.pair > 0 && pair_sk))) {
    g.stream_k = sk > 1 ? 1 : 0;
    g.workspace = ws;
    g.workspace_floats = ws_floats_;
    g.n_counters = 2 * 148;
    g.counters = counters(g.n_counters);
  }
  pbegin();
  sfk_check(sfk_gemm(&g, cur_), "gemm");
  pend(cat, 2.0 * m * n * k, double(esize_) * (double(m) * k + double(n) * k + double(m) * n));
  ++launches_;
}

int DeviceTape::logits(int x, ParamRef w) {
  const Node& in = nodes_[x];
  if (in.cols != w.cols) throw ShapeError("matmul_nt: inner dimension mismatch");
  Node n;
  n.kind = Kind::Linear;
  n.in0 = x;
  n.p0 = w;
  n.rows = in.rows;
  n.cols = w.rows;
  n.ld = dtype_ == SFK_F32 ? n.cols : (int64_t(n.cols) + 7) / 8 * 8;
  n.out = alloc_elems(int64_t(n.rows) * n.ld);
  gemm(Profiler::GemmFwd, n.rows, n.cols, in.cols, in.out, in.cols, true, pptr(w), w.cols, true, n.out, n.ld,
       SFK_EPI_PREROUND);
  nodes_.push_back(n);
  return int(nodes_.size()) - 1;
}

int DeviceTape::linear(int x, ParamRef w, const ParamRef* bias, bool relu, int residual) {
  const Node& in = nodes_[x];
  if (in.cols != w.cols) throw ShapeError("matmul_nt: inner dimension mismatch");
  if (bias && (bias->cols != w.rows || bias->rows != 1)) throw ShapeError("add_bias: bias length mismatch");
  Node n;
  n.kind = Kind::Linear;
  n.in0 = x;
  n.in1 = residual;
  n.p0 = w;
  if (bias) n.p1 = *bias;
  n.has_bias = bias != nullptr;
  n.relu = relu;
  n.rows = in.rows;
  n.cols = w.rows;
  n.ld = n.cols;
  if (residual >= 0 && (nodes_[residual].rows != n.rows || nodes_[residual].cols != n.cols))
    throw ShapeError("add: shape mismatch");
  n.out = alloc_elems(int64_t(n.rows) * n.cols);
  int flags = SFK_EPI_PREROUND;
  if (bias) flags |= SFK_EPI_BIAS;
  if (relu) flags |= SFK_EPI_RELU;
  if (residual >= 0) flags |= SFK_EPI_RESIDUAL;
  gemm(Profiler::GemmFwd, n.rows, n.cols, in.cols, in.out, in.cols, true, pptr(w), w.cols, true, n.out, n.cols, flags,
       bias ? pptr(*bias) : nullptr, residual >= 0 ? nodes_[residual].out : nullptr, n.cols);
  nodes_.push_back(n);
  return int(nodes_.size()) - 1;
}

namespace {
double attn_flops(int batch, int qw, int kw, const int32_t* /*k_len device*/, int d, bool causal, bool bwd) {
  // padded-span upper bound: every query row of sentence b against its key span
  const double pairs = causal ? double(batch) * qw * (qw + 1) / 2.0 : double(batch) * qw * kw;
  return (bwd ? 8.0 : 4.0) * pairs * d;
}
}  // namespace

int DeviceTape::external(const void* data, int rows, int cols) {
  Node n;
  n.kind = Kind::External;
  n.rows = rows;
  n.cols = cols;
  n.ld = cols;
  n.out = const_cast<void*>(data);
  nodes_.push_back(n);
  return int(nodes_.size()) - 1;
}

int DeviceTape::attention(int q, int q_col, int kv, int k_col, int v_col, int d, int heads, int batch, int q_width,
                          int k_width, bool causal, const int32_t* k_len) {
  if (nodes_[q].rows != batch * q_width || nodes_[kv].rows != batch * k_width)
    throw ShapeError("attention: span layout mismatch");
  return attention(q, q_col, kv, k_col, v_col, d, heads, {AttnPart{batch, q_width, k_width, 0, 0, k_len}}, causal);
}

int DeviceTape::attention(int q, int q_col, int kv, int k_col, int v_col, int d, int heads,
                          const std::vector<AttnPart>& parts, bool causal) {
  if (heads <= 0 || d % heads != 0) throw ShapeError("attention: d_model not divisible by heads");
  const Node& qn = nodes_[q];
  const Node& kn = nodes_[kv];
  int64_t qrows = 0;
  for (const AttnPart& pt : parts) {
    if (pt.q_row0 != qrows || pt.k_row0 + int64_t(pt.batch) * pt.k_width > kn.rows)
      throw ShapeError("attention: span layout mismatch");
    qrows += int64_t(pt.batch) * pt.q_width;
  }
  if (parts.empty() || qrows != qn.rows) throw ShapeError("attention: span layout mismatch");
  Node n;
  n.kind = Kind::Attention;
  n.in0 = q;
  n.in1 = kv;
  n.q_col = q_col;
  n.k_col = k_col;
  n.v_col = v_col;
  n.heads = heads;
  n.aparts = parts;
  n.causal = causal;
  n.rows = qn.rows;
  n.cols = d;
  n.out = alloc_elems(int64_t(n.rows) * d);
  n.stats = static_cast<float*>(arena_.alloc(size_t(n.rows) * heads * 8));
  // one call for all parts: the parts of one width class share a launch
  std::vector<sfk_attn_args> args;
  double flops = 0, bytes = 0;
  for (const AttnPart& pt : parts) {
    sfk_attn_args a{};
    a.dtype = dtype_;
    a.batch = pt.batch;
    a.q_width = pt.q_width;
    a.k_width = pt.k_width;
    a.heads = heads;
    a.dh = d / heads;
    a.causal = causal;
    a.k_len = pt.k_len;
    a.q = static_cast<const char*>(qn.out) + (pt.q_row0 * qn.cols + q_col) * int64_t(esize_);
    a.ldq = qn.cols;
    a.k = static_cast<const char*>(kn.out) + (pt.k_row0 * kn.cols + k_col) * int64_t(esize_);
    a.ldk = kn.cols;
    a.v = static_cast<const char*>(kn.out) + (pt.k_row0 * kn.cols + v_col) * int64_t(esize_);
    a.ldv = kn.cols;
    a.o = static_cast<char*>(n.out) + pt.q_row0 * d * int64_t(esize_);
    a.ldo = d;
    a.stats = n.stats + pt.q_row0 * heads * 2;
    args.push_back(a);
    flops += attn_flops(pt.batch, pt.q_width, pt.k_width, pt.k_len, d, causal, false);
    bytes += double(esize_) * d * (2.0 * pt.batch * pt.q_width + 2.0 * pt.batch * pt.k_width);
  }
  pbegin();
  if (!(ablate_mask() & 8))
    sfk_check(sfk_attention_fwd_parts(args.data(), int(args.size()), cur_), "attention_fwd");
  pend(Profiler::AttnFwd, flops, bytes);
  launches_ += sfk_attention_last_launches();
  nodes_.push_back(n);
  return int(nodes_.size()) - 1;
}

int DeviceTape::softmax_xent(int logits, const int32_t* gold, float epsilon) {
  if (epsilon < 0.f || epsilon >= 1.f) throw ConfigError("softmax_xent: epsilon must be in [0, 1)");
  Node n;
  n.kind = Kind::Xent;
  n.in0 = logits;
  n.gold = gold;
  n.eps = epsilon;
  n.rows = nodes_[logits].rows;
  n.cols = 1;
  n.row_out = static_cast<float*>(arena_.alloc(size_t(n.rows) * 16));
  nodes_.push_back(n);
  return int(nodes_.size()) - 1;
}

int DeviceTape::dropout(int x, float p, uint64_t seed, uint64_t stream, int residual) {
  const Node& in = nodes_[x];
  if (residual >= 0 && (nodes_[residual].rows != in.rows || nodes_[residual].cols != in.cols))
    throw ShapeError("add: shape mismatch");
  Node n;
  n.kind = Kind::Dropout;
  n.in0 = x;
  n.in1 = residual;
  n.p = p;
  n.seed = seed;
  n.rng_stream = stream;
  n.rows = in.rows;
  n.cols = in.cols;
  n.out = alloc_elems(int64_t(n.rows) * n.cols);
  const int64_t cnt = int64_t(n.rows) * n.cols;
  pbegin();
  sfk_check(sfk_dropout_fwd(dtype_, in.out, residual >= 0 ? nodes_[residual].out : nullptr, n.out, cnt, p, seed, stream,
                            cur_),
            "dropout_fwd");
  pend(Profiler::LayerNorm, 0, double(cnt) * esize_ * (residual >= 0 ? 3.0 : 2.0));
  ++launches_;
  nodes_.push_back(n);
  return int(nodes_.size()) - 1;
}

std::pair<void*, bool> DeviceTape::grad_of(int id) {
  Node& n = nodes_[id];
  if (n.grad) return {n.grad, false};
  n.grad = alloc_elems(int64_t(n.rows) * n.cols);
  return {n.grad, true};
}

std::pair<void*, const void*> DeviceTape::acc_target(int id) {
  Node& n = nodes_[id];
  if (!n.grad) {
    n.grad = alloc_elems(int64_t(n.rows) * n.cols);
    return {n.grad, nullptr};
  }
  // default: wait for the reader and accumulate in place (measured 118.6 vs
  // 120.5 ms/step on C4 for out of place: the extra buffers and the unthrottled
  // main stream cost more than the waits); SQF_ACC_INPLACE=0 goes out of place
  static const bool inplace = [] {
    const char* e = std::getenv("SQF_ACC_INPLACE");
    return !(e && std::atoi(e) == 0);
  }();
  if (inplace) {
    wait_side_reader(n.grad);
    return {n.grad, n.grad};
  }
  for (const auto& r : side_readers_)
    if (r.first == n.grad) {
      const void* old = n.grad;
      n.grad = alloc_elems(int64_t(n.rows) * n.cols);
      return {n.grad, old};
    }
  return {n.grad, n.grad};
}

void DeviceTape::run_xent(Node& n, float seed, bool with_grad, double* stats_acc) {
  Node& lg = nodes_[n.in0];
  // the logits buffer becomes its own gradient (dlogits written in place)
  pbegin();
  if (!(ablate_mask() & 32))
  sfk_check(sfk_xent_fwd_bwd(dtype_, lg.out, lg.rows, lg.cols, lg.ld ? lg.ld : lg.cols, n.gold, kPad, n.eps, seed,
                             with_grad ? lg.out : nullptr, n.row_out, cur_),
            "xent");
  sfk_check(sfk_xent_reduce(n.row_out, n.rows, stats_acc, cur_), "xent_reduce");
  pend(Profiler::Xent, 0, double(lg.rows) * lg.cols * esize_ * (with_grad ? 2.0 : 1.0));
  launches_ += 2;
  if (with_grad) lg.grad = lg.out;
}

void DeviceTape::finish(int loss_node, double* stats_acc) {
  Node& n = nodes_.at(loss_node);
  if (n.kind != Kind::Xent) throw ShapeError("finish: loss node must be a softmax_xent node");
  run_xent(n, 0.f, false, stats_acc);
}

void DeviceTape::backward(int loss_node, float seed, double* stats_acc, bool join) {
  if (loss_node < 0 || loss_node >= int(nodes_.size())) throw BoundsError("backward: bad node id");
  Node& n = nodes_[loss_node];
  if (n.kind != Kind::Xent) throw ShapeError("backward: loss node must be a softmax_xent node");
  run_xent(n, seed, true, stats_acc);
  for (int i = loss_node - 1; i >= 0; --i) backward_node(i);
  if (!ln_folds_.empty()) {
    // the partials were written on the side stream (or the main stream when
    // there is none): fold them there, behind everything already enqueued
    if (side_) cur_ = side_;
    flush_ln_folds();
    if (side_) {
      cudaEvent_t done = event();
      cuda_check(cudaEventRecord(done, side_), "event record");
      side_last_ = done;
      cur_ = stream_;
    }
  }
  if (join) join_side();
}

void DeviceTape::flush_ln_folds() {
  if (ln_folds_.empty()) return;
  pbegin();
  sfk_check(sfk_layernorm_bwd_params_fold(dtype_, ln_folds_.data(), int(ln_folds_.size()), cur_),
            "layernorm_bwd_params_fold");
  double bytes = 0;
  for (const auto& j : ln_folds_) bytes += double(j.nparts) * j.d * 8.0;
  pend(Profiler::LayerNorm, 0, bytes);
  ++launches_;
  ln_folds_.clear();
}

cudaEvent_t DeviceTape::event() {
  if (!evpool_) throw DeviceError("device tape: no event pool");
  if (ev_next_ == evpool_->size()) {
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event create");
    evpool_->push_back(e);
  }
  return (*evpool_)[ev_next_++];
}

void DeviceTape::wait_side_reader(const void* buf) {
  for (auto it = side_readers_.rbegin(); it != side_readers_.rend(); ++it)
    if (it->first == buf) {
      cuda_check(cudaStreamWaitEvent(stream_, it->second, 0), "stream wait");
      return;
    }
}

void DeviceTape::join_side() {
  if (side_last_) cuda_check(cudaStreamWaitEvent(stream_, side_last_, 0), "stream join");
}

void DeviceTape::bias_grad(const void* dy, int rows, int cols, int64_t ld, void* out) {
  // sfk_colsum scratch: min(512 * cols, 4M) floats
  const size_t part_floats = std::min<size_t>(size_t(512) * cols, size_t(4) << 20);
  float* part = static_cast<float*>(arena_.alloc(part_floats * 4));
  pbegin();
  sfk_check(sfk_colsum(dtype_, dy, rows, cols, ld, part, counters((cols + 255) / 256), out, cur_), "colsum");
  pend(Profiler::BiasGrad, 0, double(rows) * cols * esize_);
  launches_ += 1;
}

std::vector<std::pair<int64_t, int64_t>> DeviceTape::planned_grad_writes() const {
  // mirrors backward_node: reverse recording order, same per-kind write order
  std::vector<std::pair<int64_t, int64_t>> w;
  auto put = [&](const ParamRef& p) { w.emplace_back(p.offset, int64_t(p.rows) * p.cols); };
  for (int i = int(nodes_.size()) - 1; i >= 0; --i) {
    const Node& n = nodes_[size_t(i)];
    switch (n.kind) {
      case Kind::Embedding: put(n.p0); break;
      case Kind::LayerNorm: put(n.p0); put(n.p1); break;
      case Kind::Linear:
        if (n.has_bias) put(n.p1);
        put(n.p0);
        break;
      default: break;
    }
  }
  return w;
}

void DeviceTape::backward_node(int id) {
  Node& n = nodes_[id];
  if (!n.grad) return;  // no consumer contributed (e.g. unused branch)
  switch (n.kind) {
    case Kind::Xent:
      return;
    case Kind::Embedding: {
      // a tied output projection's wgrad (side stream) writes the same
      // parameter rows: only then wait for the side stream here
      for (const Node& o : nodes_)
        if (o.kind == Kind::Linear && o.p0.offset == n.p0.offset) {
          join_side();
          break;
        }
      pbegin();
      if (dtype_ != SFK_F32 && n.segs.chunks) {
        float* scratch = n.segs.nslots ? static_cast<float*>(arena_.alloc(size_t(n.segs.nslots) * n.cols * 4)) : nullptr;
        sfk_check(sfk_embed_bwd_chunked(dtype_, n.segs.chunks, n.segs.nchunks, n.segs.multi, n.segs.nmulti,
                                        n.segs.rows, n.cols, n.grad, n.scale, scratch, gptr(n.p0), cur_),
                  "embed_bwd");
        launches_ += n.segs.nmulti ? 1 : 0;
      } else {
        sfk_check(sfk_embed_bwd(dtype_, n.segs.uniq, n.segs.off, n.segs.rows, n.segs.n, n.cols, n.grad, n.scale,
                                gptr(n.p0), cur_),
                  "embed_bwd");
      }
      pend(Profiler::Embed, 0, double(n.rows) * n.cols * esize_ + 2.0 * n.segs.n * n.cols * esize_);
      ++launches_;
      grad_done(n.p0);
      return;
    }
    case Kind::LayerNorm: {
      const Node& in = nodes_[n.in0];
      const int max_parts = 4 * 148;  // sfk_layernorm_bwd_fused: <= 592 row blocks
      float* part = static_cast<float*>(arena_.alloc(size_t(2) * max_parts * n.cols * 4));
      const bool split = dtype_ != SFK_F32 && n.cols % 8 == 0 && n.cols <= 1024;
      // 16-bit split path: accumulate out of place when a wgrad may still read
      // the old gradient; other paths accumulate in place after waiting for it
      void* dxw = nullptr;
      const void* acc = nullptr;
      if (split && !ln_fused_env()) {
        std::tie(dxw, acc) = acc_target(n.in0);
      }
      auto [dx, fresh] = grad_of(n.in0);
      if (!dxw && !fresh) wait_side_reader(dx);
      // SQF_LN_FUSED=1: one-pass dx + gamma/beta partials on the main stream
      // (measured slower on C4, 121.1 vs 119.3 ms/step: the longer
      // critical-path kernel costs more than the side-stream pass it saves)
      if (ln_fused_env() && dtype_ != SFK_F32 && n.cols % 8 == 0 && n.cols <= 1024) {
        // dx and the gamma/beta column partials in one pass over x and dy on
        // the main stream; only the small fold of the partials is side work
        float* lpart = static_cast<float*>(arena_.alloc(size_t(2) * ((n.rows + 15) / 16) * n.cols * 4));
        int nparts = 0;
        pbegin();
        sfk_check(sfk_layernorm_bwd_dx_part(dtype_, in.out, n.grad, n.rows, n.cols, pptr(n.p0), n.stats, dx,
                                            fresh ? 0 : 1, lpart, &nparts, cur_),
                  "layernorm_bwd_dx_part");
        pend(Profiler::LayerNorm, 0, double(n.rows) * n.cols * esize_ * (fresh ? 3.0 : 4.0));
        if (side_) {
          cudaEvent_t ready = event();
          cuda_check(cudaEventRecord(ready, stream_), "event record");
          cuda_check(cudaStreamWaitEvent(side_, ready, 0), "stream wait");
          cur_ = side_;
        }
        pbegin();
        sfk_check(sfk_layernorm_bwd_fold(dtype_, lpart, nparts, n.cols, gptr(n.p0), gptr(n.p1), cur_),
                  "layernorm_bwd_fold");
        pend(Profiler::LayerNorm, 0, double(nparts) * n.cols * 8.0);
        grad_done(n.p0);
        grad_done(n.p1);
        if (side_) {
          cudaEvent_t done = event();
          cuda_check(cudaEventRecord(done, side_), "event record");
          side_last_ = done;
          cur_ = stream_;
        }
        launches_ += 2;
        return;
      }
      if (dtype_ != SFK_F32 && n.cols % 8 == 0 && n.cols <= 1024) {
        // gamma/beta gradients are parameter work: side stream, after dy is
        // ready (SQF_LN_PARAMS_MAIN=1 keeps them on the main stream)
        static const bool ln_main = [] {
          const char* e = std::getenv("SQF_LN_PARAMS_MAIN");
          return e && std::atoi(e) != 0;
        }();
        if (side_ && !ln_main) {
          cudaEvent_t ready = event();
          cuda_check(cudaEventRecord(ready, stream_), "event record");
          cuda_check(cudaStreamWaitEvent(side_, ready, 0), "stream wait");
          cur_ = side_;
        }
        // column partials now; the folds of all LayerNorm nodes of the
        // sub-batch share one launch at the end of backward (per node when a
        // gradient hook needs each parameter's completion in order)
        pbegin();
        int nparts = 0;
        if (!(ablate_mask() & 4))
          sfk_check(sfk_layernorm_bwd_params_partial(dtype_, in.out, n.grad, n.rows, n.cols, n.stats, part, &nparts,
                                                     cur_),
                    "layernorm_bwd_params_partial");
        pend(Profiler::LayerNorm, 0, double(n.rows) * n.cols * esize_ * 2.0);
        if (nparts > 0) ln_folds_.push_back({part, gptr(n.p0), gptr(n.p1), nparts, n.cols});
        if (hook_ || ln_folds_.size() == size_t(SFK_LN_FOLD_MAX_JOBS)) flush_ln_folds();
        grad_done(n.p0);
        grad_done(n.p1);
        if (side_ && !ln_main) {
          cudaEvent_t done = event();
          cuda_check(cudaEventRecord(done, side_), "event record");
          side_readers_.emplace_back(n.grad, done);
          side_last_ = done;
          cur_ = stream_;
        }
        pbegin();
        if (!(ablate_mask() & 2))
        sfk_check(sfk_layernorm_bwd_dx_acc(dtype_, in.out, n.grad, n.rows, n.cols, pptr(n.p0), n.stats, acc, dxw,
                                           cur_),
                  "layernorm_bwd_dx");
        pend(Profiler::LayerNorm, 0, double(n.rows) * n.cols * esize_ * (acc ? 4.0 : 3.0));
        launches_ += 2;
        return;
      }
      pbegin();
      sfk_check(sfk_layernorm_bwd_fused(dtype_, in.out, n.grad, n.rows, n.cols, pptr(n.p0), n.stats, dx,
                                        fresh ? 0 : 1, part, counters(1), gptr(n.p0), gptr(n.p1), cur_),
                "layernorm_bwd");
      pend(Profiler::LayerNorm, 0, double(n.rows) * n.cols * esize_ * (fresh ? 3.0 : 4.0));
      launches_ += 1;
      grad_done(n.p0);
      grad_done(n.p1);
      return;
    }
    case Kind::Linear: {
      const Node& in = nodes_[n.in0];
      void* dy = n.grad;
      // residual add: the residual input receives dy unchanged; alias when fresh
      if (n.in1 >= 0) {
        Node& r = nodes_[n.in1];
        if (r.grad) throw ShapeError("linear: residual input already has a gradient (unsupported fan-out)");
        r.grad = dy;
      }
      // parameter gradients (bias column sums + wgrad dW += dy^T x) only feed
      // the optimizer: they run on the side stream, ordered after dy is ready
      if (side_) {
        cudaEvent_t ready = event();
        cuda_check(cudaEventRecord(ready, stream_), "event record");
        cuda_check(cudaStreamWaitEvent(side_, ready, 0), "stream wait");
        cur_ = side_;
      }
      // 16-bit: the bias gradient rides in the weight-gradient GEMM (its
      // epilogue warps sum dY out of the A tiles in shared memory)
      const bool fused_db = n.has_bias && dtype_ != SFK_F32;
      const int64_t ldy = n.ld ? n.ld : n.cols;
      if (n.has_bias && !fused_db) bias_grad(dy, n.rows, n.cols, ldy, gptr(n.p1));
      gemm(Profiler::GemmWgrad, n.cols, in.cols, n.rows, dy, ldy, false, in.out, in.cols, false, gptr(n.p0),
             n.p0.cols, SFK_EPI_ACCUM, nullptr, nullptr, 0, nullptr, 0, fused_db ? gptr(n.p1) : nullptr);
      if (n.has_bias) grad_done(n.p1);
      grad_done(n.p0);
      if (side_) {
        cudaEvent_t done = event();
        cuda_check(cudaEventRecord(done, side_), "event record");
        side_readers_.emplace_back(dy, done);
        side_last_ = done;
        cur_ = stream_;
      }
      // dgrad into the input; a relu input gets the masked (pre-activation) grad
      Node& inm = nodes_[n.in0];
      const bool relu_in = inm.kind == Kind::Linear && inm.relu;
      if (relu_in && inm.grad) throw ShapeError("linear: relu output with several consumers is unsupported");
      // an accumulation whose old buffer a side-stream wgrad may still read
      // goes out of place: new = q(old + dY W) via the residual epilogue
      auto [dx, acc] = dtype_ != SFK_F32 ? acc_target(n.in0) : std::pair<void*, const void*>{nullptr, nullptr};
      bool fresh = true;
      if (!dx) {
        auto g = grad_of(n.in0);
        dx = g.first;
        fresh = g.second;
        acc = fresh ? nullptr : dx;
        if (!fresh) wait_side_reader(dx);
      }
      int flags = acc == nullptr ? 0 : acc == dx ? SFK_EPI_ACCUM : SFK_EPI_RESIDUAL;
      const void* mask = nullptr;
      if (relu_in) {
        flags = SFK_EPI_MASK;
        mask = inm.out;
        inm.grad_masked = true;
      }
      gemm(Profiler::GemmDgrad, n.rows, in.cols, n.cols, dy, ldy, true, pptr(n.p0), n.p0.cols, false, dx, in.cols,
           flags, nullptr, flags == SFK_EPI_RESIDUAL ? acc : nullptr, in.cols, mask, in.cols);
      return;
    }
    case Kind::Dropout: {
      void* dy = n.grad;
      if (n.in1 >= 0) {  // the fused residual add passes dy through unchanged
        Node& r = nodes_[n.in1];
        if (r.grad) throw ShapeError("dropout: residual input already has a gradient (unsupported fan-out)");
        r.grad = dy;
      }
      auto [dx, fresh] = grad_of(n.in0);
      if (!fresh) wait_side_reader(dx);
      const int64_t cnt = int64_t(n.rows) * n.cols;
      pbegin();
      sfk_check(sfk_dropout_bwd(dtype_, dy, dx, cnt, n.p, n.seed, n.rng_stream, fresh ? 0 : 1, cur_), "dropout_bwd");
      pend(Profiler::LayerNorm, 0, double(cnt) * esize_ * (fresh ? 2.0 : 3.0));
      ++launches_;
      return;
    }
    case Kind::External:
      break;
    case Kind::Attention: {
      const Node& qn = nodes_[n.in0];
      const Node& kn = nodes_[n.in1];
      auto [dq, fq] = grad_of(n.in0);
      auto [dkv, fkv] = grad_of(n.in1);
      // q is private to this node; a K/V node may feed several attention nodes
      // through disjoint column slices (the stacked cross K/V of all decoder
      // layers): each backward writes only its own slice
      if (!fq) throw ShapeError("attention: the query input must not have other consumers");
      (void)fkv;
      float* scratch = static_cast<float*>(arena_.alloc(size_t(n.rows) * n.heads * 4));
      std::vector<sfk_attn_args> args;
      double flops = 0, bytes = 0;
      for (const AttnPart& pt : n.aparts) {
        sfk_attn_args a{};
        a.dtype = dtype_;
        a.batch = pt.batch;
        a.q_width = pt.q_width;
        a.k_width = pt.k_width;
        a.heads = n.heads;
        a.dh = n.cols / n.heads;
        a.causal = n.causal;
        a.k_len = pt.k_len;
        const int64_t qo = pt.q_row0 * qn.cols, ko = pt.k_row0 * kn.cols, oo = pt.q_row0 * n.cols;
        a.q = static_cast<const char*>(qn.out) + (qo + n.q_col) * int64_t(esize_);
        a.ldq = qn.cols;
        a.k = static_cast<const char*>(kn.out) + (ko + n.k_col) * int64_t(esize_);
        a.ldk = kn.cols;
        a.v = static_cast<const char*>(kn.out) + (ko + n.v_col) * int64_t(esize_);
        a.ldv = kn.cols;
        a.o = static_cast<char*>(n.out) + oo * int64_t(esize_);
        a.ldo = n.cols;
        a.stats = n.stats + pt.q_row0 * n.heads * 2;
        a.dout = static_cast<char*>(n.grad) + oo * int64_t(esize_);
        a.lddo = n.cols;
        a.dq = static_cast<char*>(dq) + (qo + n.q_col) * int64_t(esize_);
        a.lddq = qn.cols;
        a.dk = static_cast<char*>(dkv) + (ko + n.k_col) * int64_t(esize_);
        a.lddk = kn.cols;
        a.dv = static_cast<char*>(dkv) + (ko + n.v_col) * int64_t(esize_);
        a.lddv = kn.cols;
        a.scratch = scratch + pt.q_row0 * n.heads;
        args.push_back(a);
        flops += attn_flops(pt.batch, pt.q_width, pt.k_width, pt.k_len, n.cols, n.causal, true);
        bytes += double(esize_) * n.cols * (4.0 * pt.batch * pt.q_width + 4.0 * pt.batch * pt.k_width);
      }
      pbegin();
      if (!(ablate_mask() & 16))
        sfk_check(sfk_attention_bwd_parts(args.data(), int(args.size()), cur_), "attention_bwd");
      pend(Profiler::AttnBwd, flops, bytes);
      launches_ += sfk_attention_last_launches();
      return;
    }
  }
}

}  // namespace sqf

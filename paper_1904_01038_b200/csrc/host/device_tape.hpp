// Device tape: records the forward of one sub-batch as sm_100a kernel launches
// and replays the exact reverse order for backward, mirroring the reference's
// Tape contract (tape.hpp:63-108): node outputs are kept for backward,
// activation gradients accumulate per node, parameter gradients accumulate
// into a caller-owned flat buffer that the tape never zeroes (the basis of
// `accum`/update_freq delayed updates).
#pragma once

#include <functional>

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <array>
#include <vector>

#include "../../../include/sqf_kernels.h"
#include "plugins.hpp"

namespace sqf {

void cuda_check(cudaError_t e, const char* what);
void sfk_check(int status, const char* what);

// Bump allocator over a few large cudaMalloc chunks; reset() once per
// sub-batch. Allocation order is deterministic so steady state never grows.
class Arena {
 public:
  ~Arena();
  void* alloc(size_t bytes);
  void reset();
  size_t capacity() const;

 private:
  struct Chunk {
    char* base;
    size_t size, used;
  };
  std::vector<Chunk> chunks_;
  size_t cur_ = 0;
};

// One sub-batch resident on the device (ids, lengths, embedding-backward segments).
struct DeviceBatch {
  int rows = 0, src_width = 0, tgt_width = 0;
  int64_t ntokens = 0;
  const int32_t* source = nullptr;      // rows x S
  const int32_t* target_in = nullptr;   // rows x T
  const int32_t* target_out = nullptr;  // rows x T
  const int32_t* src_lens = nullptr;    // rows
  struct Segs {
    const int32_t* uniq = nullptr;
    const int32_t* off = nullptr;
    const int32_t* rows = nullptr;
    int n = 0;
    // <= 16-row chunks {id, s0, s1, slot} and multi-chunk folds {id, first_slot, nslots, 0}
    const int32_t* chunks = nullptr;
    const int32_t* multi = nullptr;
    int nchunks = 0, nmulti = 0, nslots = 0;
  } src_segs, tgt_segs;
  // A pass over several packed batches of one update (sub-batch pairing,
  // trainer.cpp pack_local): part k's sentences keep their own widths; its
  // source / target positions start at src_pos0 / tgt_pos0 of the
  // concatenated id arrays. nparts == 0: one part, rows x src_width / tgt_width.
  struct Part {
    int rows = 0, src_width = 0, tgt_width = 0;
    int64_t src_pos0 = 0, tgt_pos0 = 0;
    const int32_t* src_lens = nullptr;
  };
  static constexpr int kMaxParts = 16;
  int nparts = 0;
  Part part[kMaxParts];
  int parts() const { return nparts > 0 ? nparts : 1; }
  Part get_part(int k) const {
    return nparts > 0 ? part[k] : Part{rows, src_width, tgt_width, 0, 0, src_lens};
  }
  int64_t src_positions() const;
  int64_t tgt_positions() const;
};

// Host-side packing of a MiniBatch into one int32 blob (uploaded with a single
// cudaMemcpyAsync); returns the element count. bind() turns a device copy of
// the blob into a DeviceBatch.
struct PackedBatch {
  std::vector<int32_t> blob;
  int rows = 0, src_width = 0, tgt_width = 0;
  int64_t ntokens = 0;
  size_t off_source = 0, off_tin = 0, off_tout = 0, off_slens = 0;
  size_t off_su = 0, off_so = 0, off_sr = 0, off_tu = 0, off_to = 0, off_tr = 0;
  size_t off_sc = 0, off_sm = 0, off_tc = 0, off_tm = 0;
  int n_su = 0, n_tu = 0;
  int n_sc = 0, n_sm = 0, n_ss = 0, n_tc = 0, n_tm = 0, n_ts = 0;
  std::vector<std::array<int, 3>> parts;  // (rows, src_width, tgt_width) per part; empty: one part
  static PackedBatch pack(const MiniBatch& b);
  DeviceBatch bind(const int32_t* dev_blob) const;
};

// Optional per-launch CUDA-event timing (bench/profiling pass only): every
// launch the tape issues is bracketed by an event pair on the tape's stream
// and attributed to a kernel class with its algorithmic flops and bytes.
class Profiler {
 public:
  enum Cat { GemmFwd, GemmDgrad, GemmWgrad, AttnFwd, AttnBwd, LayerNorm, Xent, Embed, BiasGrad, Optim, kCats };
  static const char* name(int c);
  ~Profiler();
  void begin(cudaStream_t s);
  void end(cudaStream_t s, int cat, double flops, double bytes);
  // resolves all pending events (synchronises)
  void collect();
  void reset();
  double ms[kCats] = {}, flops[kCats] = {}, bytes[kCats] = {};
  int64_t count[kCats] = {};
  // Timeline mode: the trainer keeps its concurrent schedule (side stream,
  // overlapped optimizer) and every launch's [start, end] is kept relative to
  // the base event of the step (ms), with the stream it ran on.
  bool concurrent = false;
  struct Span {
    int stream, cat;
    float t0, t1;
  };
  std::vector<Span> spans;
  std::vector<cudaStream_t> streams;  // index = Span::stream
  void mark_base(cudaStream_t s);

 private:
  struct Rec {
    cudaEvent_t a, b;
    int cat;
    double flops, bytes;
    cudaStream_t s;
  };
  cudaEvent_t base_ = nullptr;
  std::vector<cudaEvent_t> pool_;
  size_t next_ = 0;
  std::vector<Rec> pending_;
  cudaEvent_t open_ = nullptr;
  cudaEvent_t get();
};

struct DeviceParams {
  float* master = nullptr;   // fp32 master (device order)
  void* compute = nullptr;   // parameters the kernels read (== master in fp32 mode)
  void* grad = nullptr;      // flat gradient accumulator (caller owned)
  int64_t n = 0;
};

class DeviceTape {
 public:
  enum class Kind { Embedding, LayerNorm, Linear, Attention, Xent, Dropout, External };

  DeviceTape(Arena& arena, const DeviceParams& params, int dtype, cudaStream_t stream);

  // a8: out = q(q(E[ids]) * scale) + q(pe[pos]) ; rows = batch*width
  int embedding(ParamRef table, const int32_t* ids, int rows, int width, float scale, const float* pe,
                const DeviceBatch::Segs& segs);
  // the same over consecutive spans of positions with their own widths
  // (a multi-part pass): span k covers rows [row0, row0 + rows), positions
  // counted from row0
  struct EmbSpan {
    int64_t row0;
    int rows, width;
  };
  int embedding(ParamRef table, const int32_t* ids, int rows, const std::vector<EmbSpan>& spans, float scale,
                const float* pe, const DeviceBatch::Segs& segs);
  // a14
  int layer_norm(int x, ParamRef gamma, ParamRef beta);
  // a9 (+a11 bias, a12 relu, a13 residual add): y = [res +] [relu](x W^T [+ b])
  int linear(int x, ParamRef w, const ParamRef* bias, bool relu, int residual = -1);
  // the output projection: like linear(x, w, nullptr, false) but the logits
  // rows get a leading dimension rounded up to 8 elements, so a vocabulary of
  // any size keeps the 16-byte row alignment the tensor-core GEMMs (dgrad,
  // wgrad read dlogits through TMA) and the vectorised xent need
  int logits(int x, ParamRef w);
  // a16: q/k/v are column slices [q_col, q_col+d) of node q and [k_col..), [v_col..) of node kv
  int attention(int q, int q_col, int kv, int k_col, int v_col, int d, int heads, int batch, int q_width,
                int k_width, bool causal, const int32_t* k_len);
  // the same over parts with their own widths (a multi-part pass): part k's
  // queries are rows q_row0 + [0, batch*q_width) of q, its keys/values rows
  // k_row0 + [0, batch*k_width) of kv; one launch per part into one output
  struct AttnPart {
    int batch, q_width, k_width;
    int64_t q_row0, k_row0;
    const int32_t* k_len;
  };
  int attention(int q, int q_col, int kv, int k_col, int v_col, int d, int heads, const std::vector<AttnPart>& parts,
                bool causal);
  // a leaf over caller-owned device memory (rows x cols, row-major, tape
  // dtype): the incremental decoder's K/V caches; never differentiated
  int external(const void* data, int rows, int cols);
  cudaStream_t stream() const { return stream_; }
  // backward on another stream than the forward was recorded on (the caller
  // orders the two streams); no side-stream work may be pending
  void set_main_stream(cudaStream_t s) {
    stream_ = s;
    cur_ = s;
  }
  // a18: records the loss node; stats are produced when backward()/finish() runs
  int softmax_xent(int logits, const int32_t* gold, float epsilon);
  // Tape::dropout (tape.cpp:109-121) with the mask drawn from RngStream(seed,
  // stream); residual >= 0 fuses the following Tape::add: out = q(res + q(x*m))
  int dropout(int x, float p, uint64_t seed, uint64_t stream, int residual = -1);

  // Seeds d(loss_row) = seed on active rows (tape.cpp:506-516), runs the fused
  // xent fwd+bwd and sweeps nodes in exact reverse order.
  // join_side = false leaves the side-stream parameter-gradient work running
  // past the return (the caller orders it before reusing the arena)
  void backward(int loss_node, float seed, double* stats_acc, bool join_side = true);
  // forward-only loss statistics (evaluate)
  void finish(int loss_node, double* stats_acc);

  int dtype() const { return dtype_; }
  size_t size() const { return nodes_.size(); }
  int rows(int id) const { return nodes_[id].rows; }
  int cols(int id) const { return nodes_[id].cols; }
  const void* out(int id) const { return nodes_[id].out; }
  // number of our kernels launched so far (bench evidence)
  int64_t launches() const { return launches_; }
  void set_profiler(Profiler* p) { prof_ = p; }
  // second stream for parameter-gradient work (wgrad GEMM + bias grad) that is
  // off the critical path of the backward sweep; events order it against the
  // main stream (see backward_node). The tape joins it before returning.
  void set_side_stream(cudaStream_t s, std::vector<cudaEvent_t>* event_pool) {
    side_ = s;
    evpool_ = event_pool;
  }
  // pool of zeroed int32 counters for single-launch deterministic reductions
  // (each user re-arms its slots to 0); handed out round-robin
  // parameter-gradient completion hook, called right after the launch that
  // writes a parameter range's gradient contribution is enqueued (on `stream`);
  // the trainer uses it to start bucket all-reduces while backward continues
  using GradHook = std::function<void(int64_t offset, int64_t numel, cudaStream_t stream)>;
  // called before a launch reads parameters [offset, offset + numel) on `stream` (the
  // trainer makes the stream wait for that range's optimizer update)
  using UseHook = std::function<void(int64_t offset, int64_t numel, cudaStream_t stream)>;
  void set_use_hook(UseHook h) { use_hook_ = std::move(h); }
  void set_grad_hook(GradHook h) { hook_ = std::move(h); }
  // every parameter-gradient write backward() makes, as (offset, numel), in the
  // order the hook will report them
  std::vector<std::pair<int64_t, int64_t>> planned_grad_writes() const;
  cudaStream_t side_stream() const { return side_; }
  // stream-K GEMM workspaces, one per stream (concurrent GEMMs must not share)
  // 2 = force stream-K on every eligible GEMM (decoding: M = a few dozen
  // rows, so plain tiles would leave most SMs idle); 0 = SQF_GEMM_STREAM_K
  void set_stream_k(int mode) { sk_override_ = mode; }
  void set_gemm_workspace(float* main_ws, float* side_ws, int64_t floats) {
    ws_main_ = main_ws;
    ws_side_ = side_ws;
    ws_floats_ = floats;
  }
  void set_counters(int32_t* base, int64_t n, int64_t* cursor) {
    ctr_base_ = base;
    ctr_n_ = n;
    ctr_cursor_ = cursor;
  }

 private:
  struct Node {
    Kind kind;
    int in0 = -1, in1 = -1, in2 = -1;
    ParamRef p0{}, p1{};
    bool has_bias = false, relu = false, causal = false;
    int rows = 0, cols = 0;
    int64_t ld = 0;  // row stride of out/grad (== cols except for padded logits)
    void* out = nullptr;
    void* grad = nullptr;
    bool grad_masked = false;  // relu node: grad already holds d(pre-activation)
    float* stats = nullptr;    // LN: (mean,rstd); attention: (max,1/sum)
    // embedding
    const int32_t* ids = nullptr;
    int width = 0;
    float scale = 1.f;
    DeviceBatch::Segs segs;
    std::vector<EmbSpan> espans;  // multi-part pass (empty: one span of `width`)
    // attention
    int q_col = 0, k_col = 0, v_col = 0, heads = 0;
    std::vector<AttnPart> aparts;
    // xent
    const int32_t* gold = nullptr;
    float eps = 0.f;
    // dropout
    float p = 0.f;
    uint64_t seed = 0, rng_stream = 0;
    float* row_out = nullptr;
  };

  Arena& arena_;
  DeviceParams params_;
  int dtype_;
  int sk_override_ = 0;
  size_t esize_;
  cudaStream_t stream_;
  std::vector<Node> nodes_;
  int64_t launches_ = 0;
  Profiler* prof_ = nullptr;
  int32_t* ctr_base_ = nullptr;
  int64_t ctr_n_ = 0;
  int64_t* ctr_cursor_ = nullptr;
  int32_t* counters(int k) {
    if (!ctr_base_ || k > ctr_n_) throw DeviceError("device tape: no counter pool");
    if (*ctr_cursor_ + k > ctr_n_) *ctr_cursor_ = 0;
    int32_t* p = ctr_base_ + *ctr_cursor_;
    *ctr_cursor_ += k;
    return p;
  }
  GradHook hook_;
  UseHook use_hook_;
  float* ws_main_ = nullptr;
  float* ws_side_ = nullptr;
  int64_t ws_floats_ = 0;
  void grad_done(const ParamRef& p) {
    if (hook_) hook_(p.offset, int64_t(p.rows) * p.cols, cur_);
  }
  cudaStream_t cur_ = nullptr;  // stream the next launches go to (main or side)
  cudaStream_t side_ = nullptr;
  std::vector<cudaEvent_t>* evpool_ = nullptr;
  size_t ev_next_ = 0;
  std::vector<std::pair<const void*, cudaEvent_t>> side_readers_;  // grad buffer -> last side reader
  cudaEvent_t side_last_ = nullptr;
  cudaEvent_t event();
  void wait_side_reader(const void* buf);
  void join_side();
  void pbegin() {
    if (prof_) prof_->begin(cur_);
  }
  void pend(int cat, double flops, double bytes) {
    if (prof_) prof_->end(cur_, cat, flops, bytes);
  }

  void* alloc_elems(int64_t n) { return arena_.alloc(size_t(n) * esize_); }
  void* pptr(const ParamRef& p) const {
    if (use_hook_) use_hook_(p.offset, int64_t(p.rows) * p.cols, cur_);
    return static_cast<char*>(params_.compute) + p.offset * esize_;
  }
  void* gptr(const ParamRef& p) const { return static_cast<char*>(params_.grad) + p.offset * esize_; }
  // gradient buffer of node `id`: returns {ptr, fresh}; allocates on first use
  std::pair<void*, bool> grad_of(int id);
  // accumulation target for node id's gradient: (buffer to write, buffer to
  // accumulate from or nullptr when fresh). If a side-stream reader may still
  // be reading the current buffer, the sum goes to a new buffer instead of
  // making the main stream wait for it.
  std::pair<void*, const void*> acc_target(int id);
  void backward_node(int id);
  std::vector<sfk_ln_fold_job> ln_folds_;  // LayerNorm gamma/beta folds not yet launched
  void flush_ln_folds();
  void run_xent(Node& n, float seed, bool with_grad, double* stats_acc);
  void gemm(int cat, int m, int n, int k, const void* a, int64_t lda, bool a_kmajor, const void* b, int64_t ldb,
            bool b_kmajor, void* c, int64_t ldc, int flags, const void* bias = nullptr, const void* res = nullptr,
            int64_t ldr = 0, const void* mask = nullptr, int64_t ldm = 0, void* bias_grad = nullptr);
  void bias_grad(const void* dy, int rows, int cols, int64_t ld, void* out);
};

}  // namespace sqf

// Device-side candidate selection for beam search (reference
// generate.cpp:220-262): per decoder row (fp32 / fp16 / bf16 logits), the log-partition lse, the eos
// log-probability, and the kk best continuations under the reference's order
// -- key = cum (double) + lp (float), lp = logit - lse, key descending, token
// ascending on ties -- so the host merges rows * kk candidates instead of
// rows * V (V = 32k for the WMT models). One CTA per row; kk passes over the
// row, each taking the best candidate strictly after the previous one in that
// total order (no membership sets). The row stays in L2 between passes.
// With cum == nullptr (top-k sampling, generate.cpp:353-383) the order is the
// raw logit descending, token ascending, and lp returns the raw logits.
#include <cfloat>

#include "common.cuh"

namespace sfk {
namespace {

constexpr int kThreads = 256;

struct Best {
  double key;
  int tok;
};

__device__ __forceinline__ bool before(const Best& a, const Best& b) {
  return a.key > b.key || (a.key == b.key && a.tok < b.tok);
}

__device__ __forceinline__ Best warp_best(Best b) {
  for (int o = 16; o; o >>= 1) {
    Best x{__shfl_xor_sync(0xffffffffu, b.key, o), __shfl_xor_sync(0xffffffffu, b.tok, o)};
    if (before(x, b)) b = x;
  }
  return b;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) beam_topk_k(const T* __restrict__ logits, int64_t ld, int V,
                                                       const double* __restrict__ cum, int kk, int eos,
                                                       float* __restrict__ lse_out, float* __restrict__ eos_lp,
                                                       int32_t* __restrict__ tok_out, float* __restrict__ lp_out) {
  const int row = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T* xr = logits + int64_t(row) * ld;
  auto x = [xr](int v) { return Num<T>::ld(xr + v); };
  __shared__ float red[kThreads / 32];
  __shared__ Best bred[kThreads / 32];
  __shared__ Best prev;

  float m = -FLT_MAX;
  for (int v = threadIdx.x; v < V; v += kThreads) m = fmaxf(m, x(v));
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red[warp] = m;
  __syncthreads();
  m = red[0];
  for (int w = 1; w < kThreads / 32; ++w) m = fmaxf(m, red[w]);
  __syncthreads();
  float s = 0.f;
  for (int v = threadIdx.x; v < V; v += kThreads) s += expf(x(v) - m);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  s = 0.f;
  for (int w = 0; w < kThreads / 32; ++w) s += red[w];
  const float lse = m + logf(s);
  const bool raw = cum == nullptr;  // sampling: rank raw logits, return them
  const double c = raw ? 0.0 : cum[row];
  if (threadIdx.x == 0) {
    lse_out[row] = lse;
    eos_lp[row] = x(eos) - lse;
    prev = Best{DBL_MAX, -1};
  }
  __syncthreads();

  for (int j = 0; j < kk; ++j) {
    const Best p = prev;
    // -inf keys still rank (ties to the lower token), as in the reference's
    // stable sort of every (hypothesis, token) candidate; only NaN never does
    Best b{-INFINITY, 0x7fffffff};
    for (int v = threadIdx.x; v < V; v += kThreads) {
      const Best cnd{raw ? double(x(v)) : c + double(x(v) - lse), v};
      if (before(p, cnd) && before(cnd, b)) b = cnd;
    }
    b = warp_best(b);
    if (lane == 0) bred[warp] = b;
    __syncthreads();
    if (threadIdx.x == 0) {
      Best w = bred[0];
      for (int i = 1; i < kThreads / 32; ++i)
        if (before(bred[i], w)) w = bred[i];
      const int t = w.tok < V ? w.tok : eos;  // non-finite row: nothing ranks
      tok_out[int64_t(row) * kk + j] = t;
      lp_out[int64_t(row) * kk + j] = raw ? x(t) : x(t) - lse;
      prev = w;
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace sfk

using namespace sfk;

extern "C" int sfk_beam_topk(int dtype, const void* logits, int64_t ld, int rows, int vocab, const double* cum, int kk,
                             int eos, float* lse, float* eos_lp, int32_t* tok, float* lp, void* stream) {
  if (rows < 0 || vocab < 1 || kk < 1 || kk > vocab || ld < vocab || eos < 0 || eos >= vocab ||
      (rows && (!logits || !lse || !eos_lp || !tok || !lp))) {
    set_error("sfk_beam_topk: bad arguments (1 <= kk <= vocab, eos < vocab)");
    return SFK_EINVAL;
  }
  if (rows == 0) return SFK_OK;
  SFK_DISPATCH(dtype, T,
               beam_topk_k<T><<<rows, kThreads, 0, as_stream(stream)>>>(static_cast<const T*>(logits), ld, vocab, cum,
                                                                       kk, eos, lse, eos_lp, tok, lp));
  return check_launch("sfk_beam_topk");
}

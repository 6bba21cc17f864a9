// Multi-head attention over ragged per-sentence key spans (reference
// tape.cpp:229-258 forward, 426-480 backward; kernels.cpp:47-78), covering the
// three span shapes of model.cpp:168-187, 241-249: encoder self (keys of the
// same sentence, src_len_b of them), decoder causal self (t+1 keys) and
// cross attention (src_len_b encoder keys).
//
// Version 1 (SIMT): one warp per (query row, head) for the forward and the
// query-side backward, one warp per (key row, head) for the key-side
// backward. The fp32 softmax statistics {max, 1/sum} are saved per
// (row, head) so the backward recomputes the reference's exact probabilities
// p = exp(s - max) * (1/sum) from the same dot products instead of storing
// the probability matrix.
#include <cstdlib>

#include "common.cuh"

namespace sfk {
namespace attn {

constexpr int kWarps = 4;
constexpr int kMaxDhPerLane = 4;  // dh <= 128

struct P {
  int batch, qw, kw, heads, dh, causal;
  const int32_t* klen;
  float sc;
};

__device__ __forceinline__ int key_count(const P& p, int b, int t) { return p.causal ? t + 1 : p.klen[b]; }

// q row fragment (lane owns columns lane + 32*i) dotted with a key row
template <typename T>
__device__ __forceinline__ float dot_row(const float (&qf)[kMaxDhPerLane], const T* krow, int dh, int lane) {
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < kMaxDhPerLane; ++i) {
    const int c = lane + 32 * i;
    if (c < dh) acc = fmaf(qf[i], Num<T>::ld(krow + c), acc);
  }
  return warp_sum(acc);
}

template <typename T>
__global__ void __launch_bounds__(kWarps * 32) fwd_k(P p, const T* __restrict__ q, int64_t ldq, const T* __restrict__ k,
                                                     int64_t ldk, const T* __restrict__ v, int64_t ldv, T* __restrict__ o,
                                                     int64_t ldo, float2* __restrict__ stats) {
  extern __shared__ float sbuf[];
  const int wid = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t gw = int64_t(blockIdx.x) * kWarps + wid;
  const int64_t total = int64_t(p.batch) * p.qw * p.heads;
  if (gw >= total) return;
  float* s = sbuf + wid * p.kw;
  const int h = int(gw % p.heads);
  const int64_t row = gw / p.heads;
  const int b = int(row / p.qw), t = int(row % p.qw);
  const int n = key_count(p, b, t);
  const int64_t kb = int64_t(b) * p.kw;
  T* orow = o + row * ldo + h * p.dh;
  if (n <= 0) {
    for (int c = lane; c < p.dh; c += 32) Num<T>::st(orow + c, 0.f);
    if (lane == 0) stats[gw] = make_float2(0.f, 0.f);
    return;
  }
  float qf[kMaxDhPerLane];
#pragma unroll
  for (int i = 0; i < kMaxDhPerLane; ++i) {
    const int c = lane + 32 * i;
    qf[i] = c < p.dh ? Num<T>::ld(q + row * ldq + h * p.dh + c) : 0.f;
  }
  float mx = -INFINITY;
  for (int j = 0; j < n; ++j) {
    const float sj = __fmul_rn(p.sc, dot_row<T>(qf, k + (kb + j) * ldk + h * p.dh, p.dh, lane));
    if (lane == 0) s[j] = sj;
    mx = fmaxf(mx, sj);
  }
  __syncwarp();
  float sum = 0.f;
  for (int j = lane; j < n; j += 32) {
    const float e = expf(__fsub_rn(s[j], mx));
    s[j] = e;
    sum += e;
  }
  sum = warp_sum(sum);
  const float inv = __fdiv_rn(1.0f, sum);
  for (int j = lane; j < n; j += 32) s[j] = __fmul_rn(s[j], inv);
  __syncwarp();
  float acc[kMaxDhPerLane] = {};
  for (int j = 0; j < n; ++j) {
    const float pj = s[j];
    const T* vrow = v + (kb + j) * ldv + h * p.dh;
#pragma unroll
    for (int i = 0; i < kMaxDhPerLane; ++i) {
      const int c = lane + 32 * i;
      if (c < p.dh) acc[i] = fmaf(pj, Num<T>::ld(vrow + c), acc[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < kMaxDhPerLane; ++i) {
    const int c = lane + 32 * i;
    if (c < p.dh) Num<T>::st(orow + c, acc[i]);
  }
  if (lane == 0) stats[gw] = make_float2(mx, inv);
}

// query side: dq = sc * sum_j ds_j k_j, with D = sum_j p_j dp_j saved for the key side
template <typename T>
__global__ void __launch_bounds__(kWarps * 32) bwd_q_k(P p, const T* __restrict__ q, int64_t ldq,
                                                       const T* __restrict__ k, int64_t ldk, const T* __restrict__ v,
                                                       int64_t ldv, const T* __restrict__ dout, int64_t lddo,
                                                       const float2* __restrict__ stats, T* __restrict__ dq,
                                                       int64_t lddq, float* __restrict__ dsum) {
  extern __shared__ float sbuf[];
  const int wid = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t gw = int64_t(blockIdx.x) * kWarps + wid;
  const int64_t total = int64_t(p.batch) * p.qw * p.heads;
  if (gw >= total) return;
  float* pr = sbuf + wid * 2 * p.kw;
  float* dp = pr + p.kw;
  const int h = int(gw % p.heads);
  const int64_t row = gw / p.heads;
  const int b = int(row / p.qw), t = int(row % p.qw);
  const int n = key_count(p, b, t);
  const int64_t kb = int64_t(b) * p.kw;
  const float2 st = stats[gw];
  float qf[kMaxDhPerLane], gf[kMaxDhPerLane];
#pragma unroll
  for (int i = 0; i < kMaxDhPerLane; ++i) {
    const int c = lane + 32 * i;
    qf[i] = c < p.dh ? Num<T>::ld(q + row * ldq + h * p.dh + c) : 0.f;
    gf[i] = c < p.dh ? Num<T>::ld(dout + row * lddo + h * p.dh + c) : 0.f;
  }
  float D = 0.f;
  for (int j = 0; j < n; ++j) {
    const float sj = __fmul_rn(p.sc, dot_row<T>(qf, k + (kb + j) * ldk + h * p.dh, p.dh, lane));
    const float pj = __fmul_rn(expf(__fsub_rn(sj, st.x)), st.y);
    const float dpj = dot_row<T>(gf, v + (kb + j) * ldv + h * p.dh, p.dh, lane);
    if (lane == 0) {
      pr[j] = pj;
      dp[j] = dpj;
    }
    D = fmaf(pj, dpj, D);
  }
  __syncwarp();
  float acc[kMaxDhPerLane] = {};
  for (int j = 0; j < n; ++j) {
    const float dsj = __fmul_rn(pr[j], __fsub_rn(dp[j], D));
    const T* krow = k + (kb + j) * ldk + h * p.dh;
#pragma unroll
    for (int i = 0; i < kMaxDhPerLane; ++i) {
      const int c = lane + 32 * i;
      if (c < p.dh) acc[i] = fmaf(dsj, Num<T>::ld(krow + c), acc[i]);
    }
  }
  T* dqr = dq + row * lddq + h * p.dh;
#pragma unroll
  for (int i = 0; i < kMaxDhPerLane; ++i) {
    const int c = lane + 32 * i;
    if (c < p.dh) Num<T>::st(dqr + c, __fmul_rn(p.sc, acc[i]));
  }
  if (lane == 0) dsum[gw] = D;
}

// key side: for key j of sentence b, every query row i attending it
template <typename T>
__global__ void __launch_bounds__(kWarps * 32) bwd_kv_k(P p, const T* __restrict__ q, int64_t ldq,
                                                        const T* __restrict__ k, int64_t ldk, const T* __restrict__ v,
                                                        int64_t ldv, const T* __restrict__ dout, int64_t lddo,
                                                        const float2* __restrict__ stats, const float* __restrict__ dsum,
                                                        T* __restrict__ dk, int64_t lddk, T* __restrict__ dv,
                                                        int64_t lddv) {
  const int wid = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t gw = int64_t(blockIdx.x) * kWarps + wid;
  const int64_t total = int64_t(p.batch) * p.kw * p.heads;
  if (gw >= total) return;
  const int h = int(gw % p.heads);
  const int64_t krow_i = gw / p.heads;
  const int b = int(krow_i / p.kw), j = int(krow_i % p.kw);
  float kf[kMaxDhPerLane], vf[kMaxDhPerLane], ak[kMaxDhPerLane] = {}, av[kMaxDhPerLane] = {};
#pragma unroll
  for (int i = 0; i < kMaxDhPerLane; ++i) {
    const int c = lane + 32 * i;
    kf[i] = c < p.dh ? Num<T>::ld(k + krow_i * ldk + h * p.dh + c) : 0.f;
    vf[i] = c < p.dh ? Num<T>::ld(v + krow_i * ldv + h * p.dh + c) : 0.f;
  }
  const bool live = p.causal ? true : j < p.klen[b];
  if (live) {
    for (int t = p.causal ? j : 0; t < p.qw; ++t) {
      const int64_t qrow = int64_t(b) * p.qw + t;
      const int64_t sidx = qrow * p.heads + h;
      float qf[kMaxDhPerLane], gf[kMaxDhPerLane];
#pragma unroll
      for (int i = 0; i < kMaxDhPerLane; ++i) {
        const int c = lane + 32 * i;
        qf[i] = c < p.dh ? Num<T>::ld(q + qrow * ldq + h * p.dh + c) : 0.f;
        gf[i] = c < p.dh ? Num<T>::ld(dout + qrow * lddo + h * p.dh + c) : 0.f;
      }
      // identical arithmetic to the forward's score (dot of q fragment with k row)
      const float sj = __fmul_rn(p.sc, dot_row<T>(qf, k + krow_i * ldk + h * p.dh, p.dh, lane));
      const float2 st = stats[sidx];
      const float pj = __fmul_rn(expf(__fsub_rn(sj, st.x)), st.y);
      const float dpj = dot_row<T>(gf, v + krow_i * ldv + h * p.dh, p.dh, lane);
      const float dsj = __fmul_rn(pj, __fsub_rn(dpj, dsum[sidx]));
      const float sds = __fmul_rn(p.sc, dsj);
#pragma unroll
      for (int i = 0; i < kMaxDhPerLane; ++i) {
        ak[i] = fmaf(sds, qf[i], ak[i]);
        av[i] = fmaf(pj, gf[i], av[i]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kMaxDhPerLane; ++i) {
    const int c = lane + 32 * i;
    if (c < p.dh) {
      Num<T>::st(dk + krow_i * lddk + h * p.dh + c, ak[i]);
      Num<T>::st(dv + krow_i * lddv + h * p.dh + c, av[i]);
    }
  }
  (void)kf;
  (void)vf;
}

}  // namespace attn
}  // namespace sfk

namespace sfk {
int attention_mma(const sfk_attn_args* s, int n, bool bwd, cudaStream_t st);
void set_last_launches(int n);
}

using namespace sfk;

static int check_attn(const sfk_attn_args* a) {
  if (!a || a->batch < 0 || a->q_width < 0 || a->k_width <= 0 || a->heads <= 0 || a->dh <= 0 ||
      a->dh > 32 * attn::kMaxDhPerLane || (!a->causal && !a->k_len) || (a->causal && a->k_width < a->q_width)) {
    set_error("sfk_attention: bad arguments (dh <= 128, causal needs k_width >= q_width)");
    return SFK_EINVAL;
  }
  return SFK_OK;
}

extern "C" int sfk_attention_fwd(const sfk_attn_args* a, void* stream) {
  set_last_launches(0);
  if (int e = check_attn(a)) return e;
  if (a->batch * a->q_width == 0) return SFK_OK;
  // fp16/bf16: tensor-core flash kernel; fp32 parity mode: exact SIMT kernel below
  if (a->dtype != SFK_F32) return attention_mma(a, 1, false, as_stream(stream));
  set_last_launches(1);
  attn::P p{a->batch, a->q_width, a->k_width, a->heads, a->dh, a->causal, a->k_len, 1.0f / sqrtf(float(a->dh))};
  const int64_t warps = int64_t(a->batch) * a->q_width * a->heads;
  if (warps == 0) return SFK_OK;
  const int blocks = int((warps + attn::kWarps - 1) / attn::kWarps);
  const size_t smem = size_t(attn::kWarps) * a->k_width * sizeof(float);
  SFK_DISPATCH(a->dtype, T,
               attn::fwd_k<T><<<blocks, attn::kWarps * 32, smem, as_stream(stream)>>>(
                   p, static_cast<const T*>(a->q), a->ldq, static_cast<const T*>(a->k), a->ldk,
                   static_cast<const T*>(a->v), a->ldv, static_cast<T*>(a->o), a->ldo,
                   reinterpret_cast<float2*>(a->stats)));
  return check_launch("sfk_attention_fwd");
}

extern "C" int sfk_attention_bwd(const sfk_attn_args* a, void* stream) {
  set_last_launches(0);
  if (int e = check_attn(a)) return e;
  if (a->batch * a->q_width == 0) return SFK_OK;
  if (a->dtype != SFK_F32) return attention_mma(a, 1, true, as_stream(stream));
  set_last_launches(2);
  attn::P p{a->batch, a->q_width, a->k_width, a->heads, a->dh, a->causal, a->k_len, 1.0f / sqrtf(float(a->dh))};
  const int64_t qwarps = int64_t(a->batch) * a->q_width * a->heads;
  const int64_t kwarps = int64_t(a->batch) * a->k_width * a->heads;
  if (qwarps == 0) return SFK_OK;
  cudaStream_t s = as_stream(stream);
  const size_t smem = size_t(attn::kWarps) * 2 * a->k_width * sizeof(float);
  SFK_DISPATCH(a->dtype, T, {
    attn::bwd_q_k<T><<<int((qwarps + attn::kWarps - 1) / attn::kWarps), attn::kWarps * 32, smem, s>>>(
        p, static_cast<const T*>(a->q), a->ldq, static_cast<const T*>(a->k), a->ldk, static_cast<const T*>(a->v),
        a->ldv, static_cast<const T*>(a->dout), a->lddo, reinterpret_cast<const float2*>(a->stats),
        static_cast<T*>(a->dq), a->lddq, a->scratch);
    attn::bwd_kv_k<T><<<int((kwarps + attn::kWarps - 1) / attn::kWarps), attn::kWarps * 32, 0, s>>>(
        p, static_cast<const T*>(a->q), a->ldq, static_cast<const T*>(a->k), a->ldk, static_cast<const T*>(a->v),
        a->ldv, static_cast<const T*>(a->dout), a->lddo, reinterpret_cast<const float2*>(a->stats), a->scratch,
        static_cast<T*>(a->dk), a->lddk, static_cast<T*>(a->dv), a->lddv);
  });
  return check_launch("sfk_attention_bwd");
}

// several attention problems of one pass (the parts of a multi-part batch):
// the fp16/bf16 kernels serve all parts of one width class in one launch;
// fp32 runs them one by one
static int attn_parts(const sfk_attn_args* a, int n, bool bwd, void* stream) {
  set_last_launches(0);
  if (!a || n < 0) {
    set_error("sfk_attention_parts: bad arguments");
    return SFK_EINVAL;
  }
  bool all16 = true;
  for (int i = 0; i < n; ++i) {
    if (int e = check_attn(a + i)) return e;
    all16 = all16 && a[i].dtype != SFK_F32;
  }
  // SQF_ATTN_PARTS=0: one launch per part (for A/B measurements)
  static const bool joint = [] {
    const char* e = std::getenv("SQF_ATTN_PARTS");
    return !(e && std::atoi(e) == 0);
  }();
  if (n > 0 && all16 && joint) return attention_mma(a, n, bwd, as_stream(stream));
  int launched = 0;
  for (int i = 0; i < n; ++i) {
    if (int e = bwd ? sfk_attention_bwd(a + i, stream) : sfk_attention_fwd(a + i, stream)) return e;
    launched += sfk_attention_last_launches();
  }
  set_last_launches(launched);
  return SFK_OK;
}

extern "C" int sfk_attention_fwd_parts(const sfk_attn_args* a, int n, void* stream) {
  return attn_parts(a, n, false, stream);
}

extern "C" int sfk_attention_bwd_parts(const sfk_attn_args* a, int n, void* stream) {
  return attn_parts(a, n, true, stream);
}

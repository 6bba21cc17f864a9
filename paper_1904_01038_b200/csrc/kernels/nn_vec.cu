// 16-byte vectorised variants of the memory-bound kernels for 16-bit storage
// (fp16/bf16) with widths that are multiples of 8: embedding front/backward,
// layer norm forward/backward, bias-grad column partials. Same arithmetic
// and rounding points as the scalar kernels in nn.cu (which remain the fp32
// parity-mode path); only the memory access pattern differs.
#include "common.cuh"

namespace sfk {
namespace vec {

template <typename T>
struct V8 {
  static __device__ __forceinline__ void load(const T* p, float (&f)[8]) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if constexpr (std::is_same<T, __half>::value) {
        const float2 t = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
      } else {
        const float2 t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
      }
    }
  }
  static __device__ __forceinline__ void store(T* p, const float (&f)[8]) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if constexpr (std::is_same<T, __half>::value) {
        __half2 h = __floats2half2_rn(f[2 * i], f[2 * i + 1]);
        w[i] = *reinterpret_cast<uint32_t*>(&h);
      } else {
        __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
        w[i] = *reinterpret_cast<uint32_t*>(&h);
      }
    }
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  }
};

// warp per row; lane owns 8-wide chunks lane, lane+32, ...
template <typename T>
__global__ void __launch_bounds__(256) embed_fwd_v(const int32_t* __restrict__ ids, int rows, int width, int d,
                                                  const T* __restrict__ table, const float* __restrict__ pe,
                                                  float scale, T* __restrict__ out) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  if (r >= rows) return;
  const T* e = table + int64_t(ids[r]) * d;
  const float* p = pe + int64_t(r % width) * d;
  T* o = out + int64_t(r) * d;
  for (int c = lane * 8; c < d; c += 256) {
    float f[8];
    V8<T>::load(e + c, f);
    const float4 p0 = *reinterpret_cast<const float4*>(p + c), p1 = *reinterpret_cast<const float4*>(p + c + 4);
    const float pv[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = __fadd_rn(Num<T>::rnd(__fmul_rn(scale, f[i])), Num<T>::rnd(pv[i]));
    V8<T>::store(o + c, f);
  }
}

template <typename T>
__global__ void __launch_bounds__(128) embed_bwd_v(const int32_t* __restrict__ uniq, const int32_t* __restrict__ off,
                                                  const int32_t* __restrict__ srows, int d, const T* __restrict__ dx,
                                                  float scale, T* __restrict__ grad) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  const int u = blockIdx.x;
  const int s0 = off[u], s1 = off[u + 1];
  T* g = grad + int64_t(uniq[u]) * d;
  for (int c = threadIdx.x * 8; c < d; c += blockDim.x * 8) {
    float acc[8];
    V8<T>::load(g + c, acc);
    for (int s = s0; s < s1; ++s) {
      float f[8];
      V8<T>::load(dx + int64_t(srows[s]) * d + c, f);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = __fadd_rn(acc[i], Num<T>::rnd(__fmul_rn(scale, f[i])));
    }
    V8<T>::store(g + c, acc);
  }
}

constexpr int kMaxCh = 4;  // d <= 32 lanes * 4 chunks * 8 = 1024

template <typename T>
__global__ void __launch_bounds__(256) ln_fwd_v(const T* __restrict__ x, int rows, int d, const T* __restrict__ g,
                                               const T* __restrict__ b, T* __restrict__ y,
                                               float2* __restrict__ stats) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  if (r >= rows) return;
  const T* xr = x + int64_t(r) * d;
  float v[kMaxCh][8];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kMaxCh; ++i) {
    const int c = (lane + 32 * i) * 8;
    if (c < d) {
      V8<T>::load(xr + c, v[i]);
#pragma unroll
      for (int e = 0; e < 8; ++e) s += v[i][e];
    }
  }
  const float mean = __fdiv_rn(warp_sum(s), float(d));
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < kMaxCh; ++i) {
    const int c = (lane + 32 * i) * 8;
    if (c < d)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float t = __fsub_rn(v[i][e], mean);
        q = __fadd_rn(q, __fmul_rn(t, t));
      }
  }
  const float var = __fdiv_rn(warp_sum(q), float(d));
  const float rstd = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, 1e-5f)));
  T* yr = y + int64_t(r) * d;
#pragma unroll
  for (int i = 0; i < kMaxCh; ++i) {
    const int c = (lane + 32 * i) * 8;
    if (c < d) {
      float gg[8], bb[8], o[8];
      V8<T>::load(g + c, gg);
      V8<T>::load(b + c, bb);
#pragma unroll
      for (int e = 0; e < 8; ++e)
        o[e] = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(v[i][e], mean), rstd), gg[e]), bb[e]);
      V8<T>::store(yr + c, o);
    }
  }
  if (lane == 0) stats[r] = make_float2(mean, rstd);
}

// 8 warps per block over a contiguous row chunk; per-block column partials
// of dy*xhat (gamma) and dy (beta) are reduced through shared memory into
// part[0|1][blockIdx][d]
template <typename T>
__device__ __forceinline__ void ln_bwd_body(const T* __restrict__ x, const T* __restrict__ dy, int rows, int d,
                                            const T* __restrict__ g, const float2* __restrict__ stats,
                                            T* __restrict__ dx, int accumulate, int rpb, float* __restrict__ part,
                                            int nblk);

template <typename T>
__global__ void __launch_bounds__(256) ln_bwd_v(const T* __restrict__ x, const T* __restrict__ dy, int rows, int d,
                                               const T* __restrict__ g, const float2* __restrict__ stats,
                                               T* __restrict__ dx, int accumulate, int rpb, float* __restrict__ part,
                                               int nblk) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  ln_bwd_body<T>(x, dy, rows, d, g, stats, dx, accumulate, rpb, part, nblk);
}

template <typename T>
__device__ __forceinline__ void ln_bwd_body(const T* __restrict__ x, const T* __restrict__ dy, int rows, int d,
                                            const T* __restrict__ g, const float2* __restrict__ stats,
                                            T* __restrict__ dx, int accumulate, int rpb, float* __restrict__ part,
                                            int nblk) {
  extern __shared__ float red[];  // [2][8][d]
  const int wid = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int r0 = blockIdx.x * rpb, r1 = min(rows, r0 + rpb);
  float pg[kMaxCh][8], pb[kMaxCh][8];
#pragma unroll
  for (int i = 0; i < kMaxCh; ++i)
#pragma unroll
    for (int e = 0; e < 8; ++e) pg[i][e] = pb[i][e] = 0.f;
  const float inv_n = __fdiv_rn(1.0f, float(d));
  for (int r = r0 + wid; r < r1; r += 8) {
    const float2 st = stats[r];
    float xh[kMaxCh][8], gy[kMaxCh][8];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < kMaxCh; ++i) {
      const int c = (lane + 32 * i) * 8;
      if (c < d) {
        float gg[8];
        V8<T>::load(x + int64_t(r) * d + c, xh[i]);
        V8<T>::load(dy + int64_t(r) * d + c, gy[i]);
        V8<T>::load(g + c, gg);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          xh[i][e] = __fmul_rn(__fsub_rn(xh[i][e], st.x), st.y);
          const float dxh = __fmul_rn(gy[i][e], gg[e]);
          s1 += dxh;
          s2 += dxh * xh[i][e];
        }
      }
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    const float m1 = __fmul_rn(s1, inv_n), m2 = __fmul_rn(s2, inv_n);
#pragma unroll
    for (int i = 0; i < kMaxCh; ++i) {
      const int c = (lane + 32 * i) * 8;
      if (c < d) {
        float gg[8], o[8];
        V8<T>::load(g + c, gg);
        if (accumulate) V8<T>::load(dx + int64_t(r) * d + c, o);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float dxh = __fmul_rn(gy[i][e], gg[e]);
          const float v = __fmul_rn(st.y, __fsub_rn(__fsub_rn(dxh, m1), __fmul_rn(xh[i][e], m2)));
          o[e] = accumulate ? __fadd_rn(o[e], v) : v;
          pg[i][e] += gy[i][e] * xh[i][e];
          pb[i][e] += gy[i][e];
        }
        V8<T>::store(dx + int64_t(r) * d + c, o);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kMaxCh; ++i) {
    const int c = (lane + 32 * i) * 8;
    if (c < d)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        red[(0 * 8 + wid) * d + c + e] = pg[i][e];
        red[(1 * 8 + wid) * d + c + e] = pb[i][e];
      }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float sg = 0.f, sb = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      sg += red[w * d + c];
      sb += red[(8 + w) * d + c];
    }
    part[int64_t(blockIdx.x) * d + c] = sg;
    part[int64_t(nblk + blockIdx.x) * d + c] = sb;
  }
}

// The last block to finish (ticket == nblk-1) folds the per-block partials in
// block order: out[c] = q(out[c] + sum_p part[p][c]) — one launch, deterministic.
// The counter is re-armed to 0 by that block.
template <typename T>
__device__ __forceinline__ void fold_if_last(const float* part, int nblk, int n, T* out, int32_t* counter) {
  __shared__ int last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1) == nblk - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    float s = 0.f;
    for (int p = 0; p < nblk; ++p) s += __ldcg(part + int64_t(p) * n + c);
    Num<T>::st(out + c, Num<T>::ld(out + c) + s);
  }
  if (threadIdx.x == 0) *counter = 0;
}

template <typename T>
__global__ void __launch_bounds__(256) ln_bwd_fused_v(const T* __restrict__ x, const T* __restrict__ dy, int rows,
                                                     int d, const T* __restrict__ g, const float2* __restrict__ stats,
                                                     T* __restrict__ dx, int accumulate, int rpb,
                                                     float* __restrict__ part, int nblk, int32_t* counter,
                                                     T* __restrict__ dgamma, T* __restrict__ dbeta) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  ln_bwd_body<T>(x, dy, rows, d, g, stats, dx, accumulate, rpb, part, nblk);
  // partials for gamma then beta are contiguous: fold them as one 2d-wide vector
  __shared__ int last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1) == nblk - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float sg = 0.f, sb = 0.f;
    for (int p = 0; p < nblk; ++p) {
      sg += __ldcg(part + int64_t(p) * d + c);
      sb += __ldcg(part + int64_t(nblk + p) * d + c);
    }
    Num<T>::st(dgamma + c, Num<T>::ld(dgamma + c) + sg);
    Num<T>::st(dbeta + c, Num<T>::ld(dbeta + c) + sb);
  }
  if (threadIdx.x == 0) *counter = 0;
}

template <typename T>
__global__ void colsum_fused_v(const T* __restrict__ x, int rows, int n, int64_t ld, int rpb, float* __restrict__ part,
                               int nblk, int32_t* counter, T* __restrict__ out) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (c < n) {
    const int r0 = blockIdx.y * rpb, r1 = min(rows, r0 + rpb);
    float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int r = r0; r < r1; ++r) {
      float f[8];
      V8<T>::load(x + int64_t(r) * ld + c, f);
#pragma unroll
      for (int e = 0; e < 8; ++e) s[e] += f[e];
    }
    float* o = part + int64_t(blockIdx.y) * n + c;
    *reinterpret_cast<float4*>(o) = make_float4(s[0], s[1], s[2], s[3]);
    *reinterpret_cast<float4*>(o + 4) = make_float4(s[4], s[5], s[6], s[7]);
  }
  // one counter per column block: the last row-chunk block of this column
  // block folds its columns
  __shared__ int last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter + blockIdx.x, 1) == nblk - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int cb0 = blockIdx.x * blockDim.x * 8, cb1 = min(n, cb0 + int(blockDim.x) * 8);
  for (int cc = cb0 + threadIdx.x; cc < cb1; cc += blockDim.x) {
    float sum = 0.f;
    for (int p = 0; p < nblk; ++p) sum += __ldcg(part + int64_t(p) * n + cc);
    Num<T>::st(out + cc, Num<T>::ld(out + cc) + sum);
  }
  if (threadIdx.x == 0) counter[blockIdx.x] = 0;
}

template <typename T>
__global__ void colsum_partial_v(const T* __restrict__ x, int rows, int n, int64_t ld, int rpb,
                                 float* __restrict__ part) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (c >= n) return;
  const int r0 = blockIdx.y * rpb, r1 = min(rows, r0 + rpb);
  float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int r = r0; r < r1; ++r) {
    float f[8];
    V8<T>::load(x + int64_t(r) * ld + c, f);
#pragma unroll
    for (int e = 0; e < 8; ++e) s[e] += f[e];
  }
  float* o = part + int64_t(blockIdx.y) * n + c;
  *reinterpret_cast<float4*>(o) = make_float4(s[0], s[1], s[2], s[3]);
  *reinterpret_cast<float4*>(o + 4) = make_float4(s[4], s[5], s[6], s[7]);
}

}  // namespace vec

namespace {
inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
}

// vector-path launchers; return SFK_EUNSUP when the shape/alignment does not fit
int embed_fwd_vec(int dtype, const int32_t* ids, int rows, int width, int d, const void* table, const float* pe,
                  float scale, void* out, cudaStream_t s) {
  if (dtype == SFK_F32 || d % 8 || !al16(table) || !al16(out) || !al16(pe)) return SFK_EUNSUP;
  const int blocks = (rows + 7) / 8;
  if (dtype == SFK_F16)
    launch_pdl(vec::embed_fwd_v<__half>, blocks, 256, 0, s, ids, rows, width, d, static_cast<const __half*>(table), pe, scale,
                                                    static_cast<__half*>(out));
  else
    launch_pdl(vec::embed_fwd_v<__nv_bfloat16>, blocks, 256, 0, s, ids, rows, width, d,
                                                           static_cast<const __nv_bfloat16*>(table), pe, scale,
                                                           static_cast<__nv_bfloat16*>(out));
  return check_launch("sfk_embed_fwd(vec)");
}

int embed_bwd_vec(int dtype, const int32_t* uniq, const int32_t* off, const int32_t* rows, int nuniq, int d,
                  const void* dx, float scale, void* grad, cudaStream_t s) {
  if (dtype == SFK_F32 || d % 8 || !al16(dx) || !al16(grad)) return SFK_EUNSUP;
  const int threads = std::min(128, std::max(32, d / 8));
  if (dtype == SFK_F16)
    launch_pdl(vec::embed_bwd_v<__half>, nuniq, threads, 0, s, uniq, off, rows, d, static_cast<const __half*>(dx), scale,
                                                       static_cast<__half*>(grad));
  else
    launch_pdl(vec::embed_bwd_v<__nv_bfloat16>, nuniq, threads, 0, s, uniq, off, rows, d,
                                                              static_cast<const __nv_bfloat16*>(dx), scale,
                                                              static_cast<__nv_bfloat16*>(grad));
  return check_launch("sfk_embed_bwd(vec)");
}

int ln_fwd_vec(int dtype, const void* x, int rows, int d, const void* g, const void* b, void* y, float* stats,
               cudaStream_t s) {
  if (dtype == SFK_F32 || d % 8 || d > 1024 || !al16(x) || !al16(y) || !al16(g) || !al16(b)) return SFK_EUNSUP;
  const int blocks = (rows + 7) / 8;
  if (dtype == SFK_F16)
    launch_pdl(vec::ln_fwd_v<__half>, blocks, 256, 0, s, static_cast<const __half*>(x), rows, d,
                                                 static_cast<const __half*>(g), static_cast<const __half*>(b),
                                                 static_cast<__half*>(y), reinterpret_cast<float2*>(stats));
  else
    launch_pdl(vec::ln_fwd_v<__nv_bfloat16>, blocks, 256, 0, s, 
        static_cast<const __nv_bfloat16*>(x), rows, d, static_cast<const __nv_bfloat16*>(g),
        static_cast<const __nv_bfloat16*>(b), static_cast<__nv_bfloat16*>(y), reinterpret_cast<float2*>(stats));
  return check_launch("sfk_layernorm_fwd(vec)");
}

int ln_bwd_vec(int dtype, const void* x, const void* dy, int rows, int d, const void* g, const float* stats, void* dx,
               int accumulate, float* part, int* nparts, cudaStream_t s) {
  if (dtype == SFK_F32 || d % 8 || d > 1024 || !al16(x) || !al16(dy) || !al16(dx) || !al16(g)) return SFK_EUNSUP;
  int nblk = (rows + 31) / 32;
  nblk = std::max(1, std::min(nblk, 296));
  const int rpb = (rows + nblk - 1) / nblk;
  *nparts = nblk;
  const size_t smem = size_t(2) * 8 * d * sizeof(float);
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(vec::ln_bwd_v<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(vec::ln_bwd_v<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cfg = true;
  }
  if (dtype == SFK_F16)
    launch_pdl(vec::ln_bwd_v<__half>, nblk, 256, smem, s, static_cast<const __half*>(x), static_cast<const __half*>(dy), rows,
                                                  d, static_cast<const __half*>(g),
                                                  reinterpret_cast<const float2*>(stats), static_cast<__half*>(dx),
                                                  accumulate, rpb, part, nblk);
  else
    launch_pdl(vec::ln_bwd_v<__nv_bfloat16>, nblk, 256, smem, s, 
        static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(dy), rows, d,
        static_cast<const __nv_bfloat16*>(g), reinterpret_cast<const float2*>(stats),
        static_cast<__nv_bfloat16*>(dx), accumulate, rpb, part, nblk);
  return check_launch("sfk_layernorm_bwd(vec)");
}

int colsum_partial_vec(int dtype, const void* x, int rows, int n, int64_t ld, float* part, int* nparts,
                       cudaStream_t s);

// Fold of `nparts` column partials with 8 independent accumulators per thread
// (the loads of a column no longer serialise behind one add chain); up to two
// vectors (gamma and beta) per launch. Fixed association order: deterministic.
template <typename T>
__global__ void fold_k(const float* __restrict__ pa, const float* __restrict__ pb, int nparts, int n,
                       T* __restrict__ oa, T* __restrict__ ob) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const bool second = blockIdx.y == 1;
  if (c >= n) return;
  const float* p = second ? pb : pa;
  T* o = second ? ob : oa;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int q = 0;
  for (; q + 8 <= nparts; q += 8)
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] += p[int64_t(q + u) * n + c];
  for (; q < nparts; ++q) acc[q & 7] += p[int64_t(q) * n + c];
  const float s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  Num<T>::st(o + c, Num<T>::ld(o + c) + s);
}

int ln_bwd_fused_vec(int dtype, const void* x, const void* dy, int rows, int d, const void* g, const float* stats,
                     void* dx, int accumulate, float* part, int32_t* /*counter*/, void* dgamma, void* dbeta,
                     cudaStream_t s) {
  if (dtype == SFK_F32 || d % 8 || d > 1024 || !al16(x) || !al16(dy) || !al16(dx) || !al16(g)) return SFK_EUNSUP;
  int nparts = 0;
  if (int e = ln_bwd_vec(dtype, x, dy, rows, d, g, stats, dx, accumulate, part, &nparts, s)) return e;
  dim3 grid((d + 127) / 128, 2);
  if (dtype == SFK_F16)
    launch_pdl(fold_k<__half>, grid, 128, 0, s, part, part + size_t(nparts) * d, nparts, d, static_cast<__half*>(dgamma),
                                        static_cast<__half*>(dbeta));
  else
    launch_pdl(fold_k<__nv_bfloat16>, grid, 128, 0, s, part, part + size_t(nparts) * d, nparts, d,
                                               static_cast<__nv_bfloat16*>(dgamma),
                                               static_cast<__nv_bfloat16*>(dbeta));
  return check_launch("sfk_layernorm_bwd_fused(fold)");
}

int colsum_fused_vec(int dtype, const void* x, int rows, int n, int64_t ld, float* part, int32_t* /*counters*/,
                     void* out, cudaStream_t s) {
  if (dtype == SFK_F32 || n % 8 || ld % 8 || !al16(x)) return SFK_EUNSUP;
  int nparts = 0;
  if (int e = colsum_partial_vec(dtype, x, rows, n, ld, part, &nparts, s)) return e;
  dim3 grid((n + 127) / 128, 1);
  if (dtype == SFK_F16)
    launch_pdl(fold_k<__half>, grid, 128, 0, s, part, nullptr, nparts, n, static_cast<__half*>(out), nullptr);
  else
    launch_pdl(fold_k<__nv_bfloat16>, grid, 128, 0, s, part, nullptr, nparts, n, static_cast<__nv_bfloat16*>(out), nullptr);
  return check_launch("sfk_colsum(fold)");
}

int colsum_partial_vec(int dtype, const void* x, int rows, int n, int64_t ld, float* part, int* nparts,
                       cudaStream_t s) {
  if (dtype == SFK_F32 || n % 8 || ld % 8 || !al16(x)) return SFK_EUNSUP;
  // enough row chunks to fill the machine: ~4 blocks of 128 threads per SM
  const int col_blocks = (n / 8 + 127) / 128;
  int nblk = std::max(1, std::min(64, (148 * 4) / std::max(1, col_blocks)));
  nblk = std::min(nblk, std::max(1, rows / 16));
  const int rpb = (rows + nblk - 1) / nblk;
  *nparts = nblk;
  dim3 grid(col_blocks, nblk);
  if (dtype == SFK_F16)
    launch_pdl(vec::colsum_partial_v<__half>, grid, 128, 0, s, static_cast<const __half*>(x), rows, n, ld, rpb, part);
  else
    launch_pdl(vec::colsum_partial_v<__nv_bfloat16>, grid, 128, 0, s, static_cast<const __nv_bfloat16*>(x), rows, n, ld, rpb,
                                                              part);
  return check_launch("sfk_colsum_partial(vec)");
}

}  // namespace sfk

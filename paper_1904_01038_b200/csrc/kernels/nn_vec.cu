// 16-byte vectorised variants of the memory-bound kernels for 16-bit storage
// (fp16/bf16) with widths that are multiples of 8: embedding front/backward,
// layer norm forward/backward, bias-grad column partials. Same arithmetic
// and rounding points as the scalar kernels in nn.cu (which remain the fp32
// parity-mode path); only the memory access pattern differs.
#include <cstdlib>

#include "common.cuh"

namespace sfk {
namespace vec {

template <typename T>
struct V8 {
  static __device__ __forceinline__ void load(const T* p, float (&f)[8]) { unpack(*reinterpret_cast<const uint4*>(p), f); }
  static __device__ __forceinline__ void unpack(const uint4& u, float (&f)[8]) {
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
    int s = s0;
    // rows are added strictly in recording order; only the loads run ahead
    for (; s + 4 <= s1; s += 4) {
      float f[4][8];
#pragma unroll
      for (int u = 0; u < 4; ++u) V8<T>::load(dx + int64_t(srows[s + u]) * d + c, f[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = __fadd_rn(acc[i], Num<T>::rnd(__fmul_rn(scale, f[u][i])));
    }
    for (; s < s1; ++s) {
      float f[8];
      V8<T>::load(dx + int64_t(srows[s]) * d + c, f);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = __fadd_rn(acc[i], Num<T>::rnd(__fmul_rn(scale, f[i])));
    }
    V8<T>::store(g + c, acc);
  }
}

// Chunked embedding backward: one block per <= 16-row chunk of an id's
// recording-order segment (all loads in flight), then one block per id with
// several chunks folding the chunk sums in chunk order.
constexpr int kEmbChunk = 16;
template <typename T>
__global__ void __launch_bounds__(128) embed_bwd_chunk_v(const int4* __restrict__ chunks,
                                                        const int32_t* __restrict__ srows, int d,
                                                        const T* __restrict__ dx, float scale,
                                                        float* __restrict__ scratch, T* __restrict__ grad) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  const int4 ch = chunks[blockIdx.x];  // {id, s0, s1, slot}
  const int n = ch.z - ch.y;
  for (int c = threadIdx.x * 8; c < d; c += blockDim.x * 8) {
    uint4 u[kEmbChunk];
#pragma unroll
    for (int j = 0; j < kEmbChunk; ++j)
      if (j < n) u[j] = *reinterpret_cast<const uint4*>(dx + int64_t(srows[ch.y + j]) * d + c);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (ch.w < 0) V8<T>::load(grad + int64_t(ch.x) * d + c, acc);
#pragma unroll
    for (int j = 0; j < kEmbChunk; ++j) {
      if (j >= n) break;
      float f[8];
      V8<T>::unpack(u[j], f);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = __fadd_rn(acc[i], Num<T>::rnd(__fmul_rn(scale, f[i])));
    }
    if (ch.w < 0) {
      V8<T>::store(grad + int64_t(ch.x) * d + c, acc);
    } else {
      float* o = scratch + int64_t(ch.w) * d + c;
      *reinterpret_cast<float4*>(o) = make_float4(acc[0], acc[1], acc[2], acc[3]);
      *reinterpret_cast<float4*>(o + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(128) embed_bwd_fold_v(const int4* __restrict__ multi, int d,
                                                       const float* __restrict__ scratch, T* __restrict__ grad) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  const int4 m = multi[blockIdx.x];  // {id, first_slot, nslots, 0}
  for (int c = threadIdx.x * 8; c < d; c += blockDim.x * 8) {
    float acc[8];
    V8<T>::load(grad + int64_t(m.x) * d + c, acc);
    int k = 0;
    for (; k + 4 <= m.z; k += 4) {
      float4 q[4][2];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float* p = scratch + int64_t(m.y + k + j) * d + c;
        q[j][0] = __ldcg(reinterpret_cast<const float4*>(p));
        q[j][1] = __ldcg(reinterpret_cast<const float4*>(p + 4));
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[0] += q[j][0].x, acc[1] += q[j][0].y, acc[2] += q[j][0].z, acc[3] += q[j][0].w;
        acc[4] += q[j][1].x, acc[5] += q[j][1].y, acc[6] += q[j][1].z, acc[7] += q[j][1].w;
      }
    }
    for (; k < m.z; ++k) {
      const float* p = scratch + int64_t(m.y + k) * d + c;
      const float4 a = __ldcg(reinterpret_cast<const float4*>(p)), b = __ldcg(reinterpret_cast<const float4*>(p + 4));
      acc[0] += a.x, acc[1] += a.y, acc[2] += a.z, acc[3] += a.w;
      acc[4] += b.x, acc[5] += b.y, acc[6] += b.z, acc[7] += b.w;
    }
    V8<T>::store(grad + int64_t(m.x) * d + c, acc);
  }
}

constexpr int kMaxCh = 4;  // d <= 32 lanes * 4 chunks * 8 = 1024

// One warp per RW rows (rows w, w + nw, ... of the block). Every global load
// of the rows and of gamma/beta is issued up front (one memory round trip per
// warp), x is converted to fp32 once and kept in registers, and the rows'
// reductions interleave. RW = 1 with 256-thread blocks (default: 24 warps per
// SM at C4 shapes) or RW = 2 with 128-thread blocks (SQF_LN_FWD_ROWS=2).
template <typename T, int RW>
__global__ void __launch_bounds__(RW == 1 ? 256 : 128) ln_fwd_v(const T* __restrict__ x, int rows, int d,
                                                              const T* __restrict__ g, const T* __restrict__ b,
                                                              T* __restrict__ y, float2* __restrict__ stats) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  const int r0 = blockIdx.x * nw * RW + warp;
  if (r0 >= rows) return;
  int rr[RW];
  bool ok[RW];
#pragma unroll
  for (int k = 0; k < RW; ++k) {
    rr[k] = r0 + k * nw;
    ok[k] = rr[k] < rows;
  }
  float xf[RW][kMaxCh][8];
  {
    uint4 xu[RW][kMaxCh];
#pragma unroll
    for (int i = 0; i < kMaxCh; ++i) {
      const int c = (lane + 32 * i) * 8;
#pragma unroll
      for (int k = 0; k < RW; ++k)
        if (c < d && ok[k]) xu[k][i] = *reinterpret_cast<const uint4*>(x + int64_t(rr[k]) * d + c);
    }
#pragma unroll
    for (int i = 0; i < kMaxCh; ++i) {
      const int c = (lane + 32 * i) * 8;
#pragma unroll
      for (int k = 0; k < RW; ++k) {
        if (c < d && ok[k]) V8<T>::unpack(xu[k][i], xf[k][i]);
        else
#pragma unroll
          for (int e = 0; e < 8; ++e) xf[k][i][e] = 0.f;
      }
    }
  }
  float mean[RW], rstd[RW];
  {
    float sm[RW];
#pragma unroll
    for (int k = 0; k < RW; ++k) {
      sm[k] = 0.f;
#pragma unroll
      for (int i = 0; i < kMaxCh; ++i)
#pragma unroll
        for (int e = 0; e < 8; ++e) sm[k] += xf[k][i][e];
    }
#pragma unroll
    for (int k = 0; k < RW; ++k) mean[k] = __fdiv_rn(warp_sum(sm[k]), float(d));
    float q[RW];
#pragma unroll
    for (int k = 0; k < RW; ++k) {
      q[k] = 0.f;
#pragma unroll
      for (int i = 0; i < kMaxCh; ++i) {
        const int c = (lane + 32 * i) * 8;
        if (c < d)
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float t = __fsub_rn(xf[k][i][e], mean[k]);
            q[k] = __fadd_rn(q[k], __fmul_rn(t, t));
          }
      }
    }
#pragma unroll
    for (int k = 0; k < RW; ++k) {
      const float var = __fdiv_rn(warp_sum(q[k]), float(d));
      rstd[k] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, 1e-5f)));
    }
  }
#pragma unroll
  for (int i = 0; i < kMaxCh; ++i) {
    const int c = (lane + 32 * i) * 8;
    if (c < d) {
      float gg[8], bb[8];
      V8<T>::unpack(__ldg(reinterpret_cast<const uint4*>(g + c)), gg);
      V8<T>::unpack(__ldg(reinterpret_cast<const uint4*>(b + c)), bb);
#pragma unroll
      for (int k = 0; k < RW; ++k) {
        if (!ok[k]) continue;
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e)
          o[e] = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(xf[k][i][e], mean[k]), rstd[k]), gg[e]), bb[e]);
        V8<T>::store(y + int64_t(rr[k]) * d + c, o);
      }
    }
  }
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < RW; ++k)
      if (ok[k]) stats[rr[k]] = make_float2(mean[k], rstd[k]);
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
  // x and dy stay packed (16-bit) between the two passes over the row; only
  // the per-column gamma/beta partials live in fp32 registers
  for (int r = r0 + wid; r < r1; r += 8) {
    const float2 st = stats[r];
    uint4 xr[kMaxCh], gr[kMaxCh], dxo[kMaxCh];
#pragma unroll
    for (int i = 0; i < kMaxCh; ++i) {
      const int c = (lane + 32 * i) * 8;
      if (c < d) {
        xr[i] = *reinterpret_cast<const uint4*>(x + int64_t(r) * d + c);
        gr[i] = *reinterpret_cast<const uint4*>(dy + int64_t(r) * d + c);
        if (accumulate) dxo[i] = *reinterpret_cast<const uint4*>(dx + int64_t(r) * d + c);
      }
    }
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < kMaxCh; ++i) {
      const int c = (lane + 32 * i) * 8;
      if (c < d) {
        float gg[8], xh[8], gy[8];
        V8<T>::load(g + c, gg);
        V8<T>::unpack(xr[i], xh);
        V8<T>::unpack(gr[i], gy);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float xhat = __fmul_rn(__fsub_rn(xh[e], st.x), st.y);
          const float dxh = __fmul_rn(gy[e], gg[e]);
          s1 += dxh;
          s2 += dxh * xhat;
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
        float gg[8], xh[8], gy[8], o[8];
        V8<T>::load(g + c, gg);
        V8<T>::unpack(xr[i], xh);
        V8<T>::unpack(gr[i], gy);
        if (accumulate) V8<T>::unpack(dxo[i], o);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float xhat = __fmul_rn(__fsub_rn(xh[e], st.x), st.y);
          const float dxh = __fmul_rn(gy[e], gg[e]);
          const float v = __fmul_rn(st.y, __fsub_rn(__fsub_rn(dxh, m1), __fmul_rn(xhat, m2)));
          o[e] = accumulate ? __fadd_rn(o[e], v) : v;
          pg[i][e] += gy[e] * xhat;
          pb[i][e] += gy[e];
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
  int r = r0;
  for (; r + 4 <= r1; r += 4) {  // 4 loads in flight, sums still in row order
    uint4 u[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) u[j] = *reinterpret_cast<const uint4*>(x + int64_t(r + j) * ld + c);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float f[8];
      V8<T>::unpack(u[j], f);
#pragma unroll
      for (int e = 0; e < 8; ++e) s[e] += f[e];
    }
  }
  for (; r < r1; ++r) {
    float f[8];
    V8<T>::load(x + int64_t(r) * ld + c, f);
#pragma unroll
    for (int e = 0; e < 8; ++e) s[e] += f[e];
  }
  float* o = part + int64_t(blockIdx.y) * n + c;
  *reinterpret_cast<float4*>(o) = make_float4(s[0], s[1], s[2], s[3]);
  *reinterpret_cast<float4*>(o + 4) = make_float4(s[4], s[5], s[6], s[7]);
}

// LN backward split for the B200 schedule: the activation gradient (critical
// path) is one warp per row with no column state; the gamma/beta gradients
// (parameter work, run on the side stream) are a column reduction over rows.
template <typename T>
__global__ void __launch_bounds__(128) ln_dx_v(const T* __restrict__ x, const T* __restrict__ dy, int rows, int d,
                                              const T* __restrict__ g, const float2* __restrict__ stats,
                                              T* dx, const T* acc) {
  // acc: nullptr (dx = contribution), dx (in place) or another buffer (out of place).
  // All loads of the row (x, dy, acc, gamma, stats) are issued before any math.
  const int accumulate = acc != nullptr;
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  if (r >= rows) return;
  const float2 st = stats[r];
  const float inv_n = __fdiv_rn(1.0f, float(d));
  uint4 xr[kMaxCh], gr[kMaxCh], dxo[kMaxCh], gu[kMaxCh];
#pragma unroll
  for (int i = 0; i < kMaxCh; ++i) {
    const int c = (lane + 32 * i) * 8;
    if (c < d) {
      xr[i] = *reinterpret_cast<const uint4*>(x + int64_t(r) * d + c);
      gr[i] = *reinterpret_cast<const uint4*>(dy + int64_t(r) * d + c);
      if (accumulate) dxo[i] = *reinterpret_cast<const uint4*>(acc + int64_t(r) * d + c);
      gu[i] = __ldg(reinterpret_cast<const uint4*>(g + c));
    }
  }
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int i = 0; i < kMaxCh; ++i) {
    const int c = (lane + 32 * i) * 8;
    if (c < d) {
      float gg[8], xh[8], gy[8];
      V8<T>::unpack(gu[i], gg);
      V8<T>::unpack(xr[i], xh);
      V8<T>::unpack(gr[i], gy);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float dxh = __fmul_rn(gy[e], gg[e]);
        s1 += dxh;
        s2 += dxh * __fmul_rn(__fsub_rn(xh[e], st.x), st.y);
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
      float gg[8], xh[8], gy[8], o[8];
      V8<T>::unpack(gu[i], gg);
      V8<T>::unpack(xr[i], xh);
      V8<T>::unpack(gr[i], gy);
      if (accumulate) V8<T>::unpack(dxo[i], o);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float xhat = __fmul_rn(__fsub_rn(xh[e], st.x), st.y);
        const float v = __fmul_rn(st.y, __fsub_rn(__fsub_rn(__fmul_rn(gy[e], gg[e]), m1), __fmul_rn(xhat, m2)));
        o[e] = accumulate ? __fadd_rn(o[e], v) : v;
      }
      V8<T>::store(dx + int64_t(r) * d + c, o);
    }
  }
}

// LN backward, activation gradient + gamma/beta column partials in one pass:
// warp w of block b handles rows b*16 + 2w, +1 (same arithmetic as ln_dx_v),
// and keeps per-lane column sums of dy*xhat and dy over its rows; the 8 warp
// sums are combined in warp order in shared memory and block b writes
// part[0][b][:] (dgamma) and part[1][b][:] (dbeta). A fold over the nblk
// partials (fold_k, fixed order) finishes dgamma/dbeta off the critical path.
constexpr int kLnRowsPerWarp = 2;
template <typename T>
__global__ void __launch_bounds__(256) ln_dx_part_v(const T* __restrict__ x, const T* __restrict__ dy, int rows, int d,
                                                   const T* __restrict__ g, const float2* __restrict__ stats,
                                                   T* __restrict__ dx, int accumulate, float* __restrict__ part,
                                                   int nblk) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  extern __shared__ float red[];  // [8][d]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const float inv_n = __fdiv_rn(1.0f, float(d));
  float pg[kMaxCh][8], pb[kMaxCh][8];
#pragma unroll
  for (int i = 0; i < kMaxCh; ++i)
#pragma unroll
    for (int e = 0; e < 8; ++e) pg[i][e] = pb[i][e] = 0.f;
#pragma unroll 1
  for (int j = 0; j < kLnRowsPerWarp; ++j) {
    const int r = blockIdx.x * (8 * kLnRowsPerWarp) + warp * kLnRowsPerWarp + j;
    if (r >= rows) break;
    const float2 st = stats[r];
    uint4 xr[kMaxCh], gr[kMaxCh], dxo[kMaxCh];
#pragma unroll
    for (int i = 0; i < kMaxCh; ++i) {
      const int c = (lane + 32 * i) * 8;
      if (c < d) {
        xr[i] = *reinterpret_cast<const uint4*>(x + int64_t(r) * d + c);
        gr[i] = *reinterpret_cast<const uint4*>(dy + int64_t(r) * d + c);
        if (accumulate) dxo[i] = *reinterpret_cast<const uint4*>(dx + int64_t(r) * d + c);
      }
    }
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < kMaxCh; ++i) {
      const int c = (lane + 32 * i) * 8;
      if (c < d) {
        float gg[8], xh[8], gy[8];
        V8<T>::load(g + c, gg);
        V8<T>::unpack(xr[i], xh);
        V8<T>::unpack(gr[i], gy);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float dxh = __fmul_rn(gy[e], gg[e]);
          const float xhat = __fmul_rn(__fsub_rn(xh[e], st.x), st.y);
          s1 += dxh;
          s2 += dxh * xhat;
          pg[i][e] += gy[e] * xhat;
          pb[i][e] += gy[e];
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
        float gg[8], xh[8], gy[8], o[8];
        V8<T>::load(g + c, gg);
        V8<T>::unpack(xr[i], xh);
        V8<T>::unpack(gr[i], gy);
        if (accumulate) V8<T>::unpack(dxo[i], o);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float xhat = __fmul_rn(__fsub_rn(xh[e], st.x), st.y);
          const float v = __fmul_rn(st.y, __fsub_rn(__fsub_rn(__fmul_rn(gy[e], gg[e]), m1), __fmul_rn(xhat, m2)));
          o[e] = accumulate ? __fadd_rn(o[e], v) : v;
        }
        V8<T>::store(dx + int64_t(r) * d + c, o);
      }
    }
  }
  // block partials, one vector at a time through the [8][d] buffer
#pragma unroll
  for (int v = 0; v < 2; ++v) {
#pragma unroll
    for (int i = 0; i < kMaxCh; ++i) {
      const int c = (lane + 32 * i) * 8;
      if (c < d) {
        float* o = red + warp * d + c;
        const float(&src)[8] = v == 0 ? pg[i] : pb[i];
        *reinterpret_cast<float4*>(o) = make_float4(src[0], src[1], src[2], src[3]);
        *reinterpret_cast<float4*>(o + 4) = make_float4(src[4], src[5], src[6], src[7]);
      }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += red[w * d + c];
      part[(int64_t(v) * nblk + blockIdx.x) * d + c] = t;
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void __launch_bounds__(128) ln_dgb_partial_v(const T* __restrict__ x, const T* __restrict__ dy, int rows,
                                                       int d, const float2* __restrict__ stats, int rpb,
                                                       float* __restrict__ part, int nblk) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (c >= d) return;
  const int r0 = blockIdx.y * rpb, r1 = min(rows, r0 + rpb);
  float pg[8] = {0, 0, 0, 0, 0, 0, 0, 0}, pb[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int r = r0;
  for (; r + 2 <= r1; r += 2) {
    uint4 xu[2], gu[2];
    float2 st[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      xu[j] = *reinterpret_cast<const uint4*>(x + int64_t(r + j) * d + c);
      gu[j] = *reinterpret_cast<const uint4*>(dy + int64_t(r + j) * d + c);
      st[j] = stats[r + j];
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      float xh[8], gy[8];
      vec::V8<T>::unpack(xu[j], xh);
      vec::V8<T>::unpack(gu[j], gy);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        pg[e] += gy[e] * __fmul_rn(__fsub_rn(xh[e], st[j].x), st[j].y);
        pb[e] += gy[e];
      }
    }
  }
  for (; r < r1; ++r) {
    float xh[8], gy[8];
    V8<T>::load(x + int64_t(r) * d + c, xh);
    V8<T>::load(dy + int64_t(r) * d + c, gy);
    const float2 st = stats[r];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      pg[e] += gy[e] * __fmul_rn(__fsub_rn(xh[e], st.x), st.y);
      pb[e] += gy[e];
    }
  }
  float* og = part + int64_t(blockIdx.y) * d + c;
  float* ob = part + int64_t(nblk + blockIdx.y) * d + c;
  *reinterpret_cast<float4*>(og) = make_float4(pg[0], pg[1], pg[2], pg[3]);
  *reinterpret_cast<float4*>(og + 4) = make_float4(pg[4], pg[5], pg[6], pg[7]);
  *reinterpret_cast<float4*>(ob) = make_float4(pb[0], pb[1], pb[2], pb[3]);
  *reinterpret_cast<float4*>(ob + 4) = make_float4(pb[4], pb[5], pb[6], pb[7]);
}

// LayerNorm gamma/beta partials: block (b, s) sums rows [b*rpb, (b+1)*rpb) of
// dy*xhat (gamma) and dy (beta) over the 512-column slice s. Warp w takes rows
// w, w+8, ... two at a time (all loads of both rows in flight), every lane keeps
// the column sums of its two 16-byte chunks, and the 8 warp sums are combined
// in warp order through shared memory into part[b][0|1][d]. Fixed
// association: deterministic.
constexpr int kGbCh = 2;  // 16-byte chunks per lane: 32 lanes x 2 x 8 = 512 columns
template <typename T>
__global__ void __launch_bounds__(256) ln_gb_part_k(const T* __restrict__ x, const T* __restrict__ dy,
                                                   const float2* __restrict__ stats, int rows, int d, int rpb,
                                                   float* __restrict__ part) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  __shared__ __align__(16) float red[8][512];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int r0 = blockIdx.x * rpb, r1 = min(rows, r0 + rpb), c0 = blockIdx.y * 512;
  float pg[kGbCh][8], pb[kGbCh][8];
#pragma unroll
  for (int i = 0; i < kGbCh; ++i)
#pragma unroll
    for (int e = 0; e < 8; ++e) pg[i][e] = pb[i][e] = 0.f;
  for (int r = r0 + warp; r < r1; r += 16) {
    const bool two = r + 8 < r1;
    uint4 xu[2][kGbCh], gu[2][kGbCh];
    float2 st[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (j == 1 && !two) break;
      const int64_t row = r + 8 * j;
      st[j] = stats[row];
#pragma unroll
      for (int i = 0; i < kGbCh; ++i) {
        const int c = c0 + (lane + 32 * i) * 8;
        if (c < d) {
          xu[j][i] = *reinterpret_cast<const uint4*>(x + row * d + c);
          gu[j][i] = *reinterpret_cast<const uint4*>(dy + row * d + c);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (j == 1 && !two) break;
#pragma unroll
      for (int i = 0; i < kGbCh; ++i) {
        const int c = c0 + (lane + 32 * i) * 8;
        if (c < d) {
          float xh[8], gy[8];
          V8<T>::unpack(xu[j][i], xh);
          V8<T>::unpack(gu[j][i], gy);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            pg[i][e] += gy[e] * __fmul_rn(__fsub_rn(xh[e], st[j].x), st[j].y);
            pb[i][e] += gy[e];
          }
        }
      }
    }
  }
  const int width = min(512, d - c0);
#pragma unroll
  for (int v = 0; v < 2; ++v) {
#pragma unroll
    for (int i = 0; i < kGbCh; ++i) {
      const int cl = (lane + 32 * i) * 8;
      if (cl < width) {
        float* o = &red[warp][cl];
        const float(&src)[8] = v == 0 ? pg[i] : pb[i];
        *reinterpret_cast<float4*>(o) = make_float4(src[0], src[1], src[2], src[3]);
        *reinterpret_cast<float4*>(o + 4) = make_float4(src[4], src[5], src[6], src[7]);
      }
    }
    __syncthreads();
    for (int cl = threadIdx.x; cl < width; cl += blockDim.x) {
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += red[w][cl];
      part[(int64_t(blockIdx.x) * 2 + v) * d + c0 + cl] = t;
    }
    __syncthreads();
  }
}

// Batched fold of gamma/beta partials for many LayerNorm nodes. Block
// (chunk, vec, job) owns 32 columns of one vector of one job; warp w sums the
// contiguous partial range [w*P/8, (w+1)*P/8) for its lane's column (all loads
// independent), the 8 warp sums are added in warp order, then
// out = q(out + sum). Fixed association: deterministic.
struct LnFoldBatch {
  sfk_ln_fold_job job[SFK_LN_FOLD_MAX_JOBS];
};
template <typename T>
__global__ void __launch_bounds__(256) ln_gb_fold_k(const __grid_constant__ LnFoldBatch B) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  __shared__ float red[8][32];
  const sfk_ln_fold_job& jb = B.job[blockIdx.z];
  const int v = blockIdx.y, warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int c = blockIdx.x * 32 + lane;
  if (blockIdx.x * 32 >= jb.d) return;
  const int p0 = warp * jb.nparts / 8, p1 = (warp + 1) * jb.nparts / 8;
  float acc = 0.f;
  if (c < jb.d) {
    const float* p = jb.part + int64_t(v) * jb.d + c;
    const int64_t stride = int64_t(2) * jb.d;
    float a[4] = {0.f, 0.f, 0.f, 0.f};
    int q = p0;
    for (; q + 4 <= p1; q += 4)
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] += __ldcg(p + (q + u) * stride);
    for (; q < p1; ++q) a[0] += __ldcg(p + q * stride);
    acc = (a[0] + a[1]) + (a[2] + a[3]);
  }
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && c < jb.d) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][lane];
    T* o = static_cast<T*>(v == 0 ? jb.dgamma : jb.dbeta) + c;
    Num<T>::st(o, Num<T>::ld(o) + t);
  }
}

// Fused label-smoothed cross entropy fwd+bwd for one vocabulary row per
// block (tape.cpp:259-290, 481-502): the row is staged in shared memory with
// 16-byte loads; pass 1 computes max / first argmax / sum-exp online,
// pass 2 writes dlogits = q(seed*(softmax - target)) with 16-byte stores and
// accumulates the smoothing sum of (lse - l).
template <typename T>
__global__ void __launch_bounds__(512) xent_v(const T* __restrict__ logits, int V, int64_t ld,
                                             const int32_t* __restrict__ gold, int pad, float eps, float seed,
                                             T* __restrict__ dlogits, float* __restrict__ row_out) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  extern __shared__ uint4 xrow[];
  __shared__ float rm[16], rs[16];
  __shared__ int ri[16];
  const int r = blockIdx.x, tid = threadIdx.x, lane = tid % 32, wid = tid / 32, nw = blockDim.x / 32;
  const int gid = gold[r];
  const int nch = V / 8;
  const T* src = logits + int64_t(r) * ld;
  T* dst = dlogits ? dlogits + int64_t(r) * ld : nullptr;
  if (gid == pad) {
    if (dst)
      for (int ch = tid; ch < nch; ch += blockDim.x) reinterpret_cast<uint4*>(dst)[ch] = make_uint4(0, 0, 0, 0);
    if (tid == 0) reinterpret_cast<float4*>(row_out)[r] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  // log2 domain: every exponential is one FFMA + one SFU ex2 (ftz: terms
  // below 2^-126 of the row max contribute nothing at fp32 precision anyway)
  const float L2E = 1.4426950408889634f;
  auto ex2 = [](float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
  };
  float m = -INFINITY, s = 0.f, sf = 0.f;  // sf: sum of logits (label-smoothing term)
  int mi = 0x7fffffff;
  // four 16-byte loads in flight per thread before any of them is consumed
  for (int ch0 = tid; ch0 < nch; ch0 += 4 * blockDim.x) {
    uint4 uu[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int ch = ch0 + j * blockDim.x;
      if (ch < nch) uu[j] = reinterpret_cast<const uint4*>(src)[ch];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int ch = ch0 + j * blockDim.x;
      if (ch >= nch) break;
      const uint4 u = uu[j];
      xrow[ch] = u;
      float f[8];
      V8<T>::unpack(u, f);
      float cm = f[0];
      int ci = 0;
#pragma unroll
      for (int e = 1; e < 8; ++e)
        if (f[e] > cm) cm = f[e], ci = e;
      if (cm > m) {
        s *= ex2((m - cm) * L2E);
        m = cm;
        mi = ch * 8 + ci;
      }
      const float nml = -m * L2E;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        s += ex2(fmaf(f[e], L2E, nml));
        sf += f[e];
      }
    }
  }
  // (max, sum, first argmax) combine
  auto comb = [&](float om, float os, int oi) {
    const float M = fmaxf(m, om);
    const float a = m == -INFINITY ? 0.f : s * exp2f((m - M) * L2E);
    const float b = om == -INFINITY ? 0.f : os * exp2f((om - M) * L2E);
    const int idx = (om > m || (om == m && oi < mi)) ? oi : mi;
    m = M;
    s = a + b;
    mi = idx;
  };
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, s, o);
    const int oi = __shfl_xor_sync(0xffffffffu, mi, o);
    comb(om, os, oi);
  }
  if (lane == 0) rm[wid] = m, rs[wid] = s, ri[wid] = mi;
  __syncthreads();
  if (wid == 0) {
    m = lane < nw ? rm[lane] : -INFINITY;
    s = lane < nw ? rs[lane] : 0.f;
    mi = lane < nw ? ri[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, s, o);
      const int oi = __shfl_xor_sync(0xffffffffu, mi, o);
      comb(om, os, oi);
    }
    if (lane == 0) rm[0] = m, rs[0] = s, ri[0] = mi;
  }
  __syncthreads();
  const float lse = __fadd_rn(rm[0], logf(rs[0]));
  const int amax = ri[0];
  __syncthreads();
  const float uni = __fdiv_rn(eps, float(V)), on = __fadd_rn(1.0f - eps, uni);
  if (dst) {
    const float nll2 = -lse * L2E;
    const int gch = gid / 8;
    for (int ch = tid; ch < nch; ch += blockDim.x) {
      float f[8], o[8];
      V8<T>::unpack(xrow[ch], f);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = __fmul_rn(seed, __fsub_rn(ex2(fmaf(f[e], L2E, nll2)), uni));
      if (ch == gch) {  // the gold column's target is (1 - eps) + eps / V
        const int e = gid % 8;
        o[e] = __fmul_rn(seed, __fsub_rn(ex2(fmaf(f[e], L2E, nll2)), on));
      }
      V8<T>::store(dst + ch * 8, o);
    }
  }
  // sum over v of (lse - l_v) = V * lse - sum l_v
  float sm = warp_sum(sf);
  if (lane == 0) rs[wid] = sm;
  __syncthreads();
  if (tid == 0) {
    float tsf = 0.f;
    for (int w = 0; w < nw; ++w) tsf += rs[w];
    const float tot = __fsub_rn(__fmul_rn(float(V), lse), tsf);
    float gl[8];
    V8<T>::unpack(xrow[gid / 8], gl);
    const float nll = __fsub_rn(lse, gl[gid % 8]);
    float loss = nll;
    if (eps != 0.0f) loss = __fadd_rn(__fmul_rn(1.0f - eps, nll), __fmul_rn(__fdiv_rn(eps, float(V)), tot));
    reinterpret_cast<float4*>(row_out)[r] = make_float4(Num<T>::rnd(loss), nll, amax == gid ? 1.f : 0.f, 1.f);
  }
}

}  // namespace vec

int xent_vec(int dtype, void* logits, int rows, int V, int64_t ld, const int32_t* gold, int pad, float eps, float seed,
             void* dlogits, float* row_out, cudaStream_t s) {
  const uintptr_t al = reinterpret_cast<uintptr_t>(logits) | reinterpret_cast<uintptr_t>(dlogits) |
                       reinterpret_cast<uintptr_t>(row_out);
  if (dtype == SFK_F32 || V % 8 || ld % 8 || (al & 15) || size_t(V) * 2 > 200 * 1024) return SFK_EUNSUP;
  const size_t smem = size_t(V) * 2;
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(vec::xent_v<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(vec::xent_v<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cfg = true;
  }
  if (dtype == SFK_F16)
    launch_pdl(vec::xent_v<__half>, dim3(rows), dim3(512), smem, s, static_cast<const __half*>(logits), V, ld, gold,
               pad, eps, seed, static_cast<__half*>(dlogits), row_out);
  else
    launch_pdl(vec::xent_v<__nv_bfloat16>, dim3(rows), dim3(512), smem, s, static_cast<const __nv_bfloat16*>(logits), V,
               ld, gold, pad, eps, seed, static_cast<__nv_bfloat16*>(dlogits), row_out);
  return check_launch("sfk_xent_fwd_bwd(vec)");
}

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

int embed_bwd_chunked_vec(int dtype, const int32_t* chunks, int nchunks, const int32_t* multi, int nmulti,
                          const int32_t* rows, int d, const void* dx, float scale, float* scratch, void* grad,
                          cudaStream_t s) {
  if (dtype == SFK_F32 || d % 8 || !al16(dx) || !al16(grad) || (nmulti && !scratch)) return SFK_EUNSUP;
  const int threads = std::min(128, std::max(32, d / 8));
  auto c4 = reinterpret_cast<const int4*>(chunks);
  auto m4 = reinterpret_cast<const int4*>(multi);
  if (dtype == SFK_F16) {
    launch_pdl(vec::embed_bwd_chunk_v<__half>, nchunks, threads, 0, s, c4, rows, d, static_cast<const __half*>(dx),
               scale, scratch, static_cast<__half*>(grad));
    if (nmulti)
      launch_pdl(vec::embed_bwd_fold_v<__half>, nmulti, threads, 0, s, m4, d, static_cast<const float*>(scratch),
                 static_cast<__half*>(grad));
  } else {
    launch_pdl(vec::embed_bwd_chunk_v<__nv_bfloat16>, nchunks, threads, 0, s, c4, rows, d,
               static_cast<const __nv_bfloat16*>(dx), scale, scratch, static_cast<__nv_bfloat16*>(grad));
    if (nmulti)
      launch_pdl(vec::embed_bwd_fold_v<__nv_bfloat16>, nmulti, threads, 0, s, m4, d,
                 static_cast<const float*>(scratch), static_cast<__nv_bfloat16*>(grad));
  }
  return check_launch("sfk_embed_bwd_chunked");
}

int ln_fwd_vec(int dtype, const void* x, int rows, int d, const void* g, const void* b, void* y, float* stats,
               cudaStream_t s) {
  if (dtype == SFK_F32 || d % 8 || d > 1024 || !al16(x) || !al16(y) || !al16(g) || !al16(b)) return SFK_EUNSUP;
  static const int rw = [] {
    const char* e = std::getenv("SQF_LN_FWD_ROWS");
    return e && std::atoi(e) == 2 ? 2 : 1;
  }();
  auto go = [&](auto tag) {
    using T = decltype(tag);
    const T* xt = static_cast<const T*>(x);
    if (rw == 1)
      launch_pdl(vec::ln_fwd_v<T, 1>, (rows + 7) / 8, 256, 0, s, xt, rows, d, static_cast<const T*>(g),
                 static_cast<const T*>(b), static_cast<T*>(y), reinterpret_cast<float2*>(stats));
    else
      launch_pdl(vec::ln_fwd_v<T, 2>, (rows + 7) / 8, 128, 0, s, xt, rows, d, static_cast<const T*>(g),
                 static_cast<const T*>(b), static_cast<T*>(y), reinterpret_cast<float2*>(stats));
  };
  if (dtype == SFK_F16) go(__half{});
  else go(__nv_bfloat16{});
  return check_launch("sfk_layernorm_fwd(vec)");
}

int ln_bwd_vec(int dtype, const void* x, const void* dy, int rows, int d, const void* g, const float* stats, void* dx,
               int accumulate, float* part, int* nparts, cudaStream_t s) {
  if (dtype == SFK_F32 || d % 8 || d > 1024 || !al16(x) || !al16(dy) || !al16(dx) || !al16(g)) return SFK_EUNSUP;
  int nblk = (rows + 15) / 16;
  nblk = std::max(1, std::min(nblk, 4 * 148));
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

// Fold of `nparts` column partials, up to two vectors (gamma and beta) per
// launch. One block per 8-column slice (so n/8 blocks cover the machine):
// thread (g, c) sums partials g, g+32, ... in two fixed chains, then the 32
// group sums are added in group order. Fixed association order: deterministic.
template <typename T>
__global__ void __launch_bounds__(256) fold_k(const float* __restrict__ pa, const float* __restrict__ pb, int nparts,
                                             int n, T* __restrict__ oa, T* __restrict__ ob) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  __shared__ float red[32][9];
  const int g = threadIdx.x >> 3, cl = threadIdx.x & 7;
  const int c = blockIdx.x * 8 + cl;
  const bool second = blockIdx.y == 1;
  const float* p = second ? pb : pa;
  T* o = second ? ob : oa;
  float a0 = 0.f, a1 = 0.f;
  if (c < n) {
    int q = g;
    for (; q + 32 < nparts; q += 64) {
      a0 += __ldcg(p + int64_t(q) * n + c);
      a1 += __ldcg(p + int64_t(q + 32) * n + c);
    }
    if (q < nparts) a0 += __ldcg(p + int64_t(q) * n + c);
  }
  red[g][cl] = a0 + a1;
  __syncthreads();
  if (g == 0 && c < n) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 32; ++k) s += red[k][cl];
    Num<T>::st(o + c, Num<T>::ld(o + c) + s);
  }
}

// Single-launch column reductions (bias gradient, LayerNorm gamma/beta).
// One block = 8 warps over a 256-column slice and a chunk of rows: warp w sums
// rows w, w+8, ... (four 512-byte warp loads in flight), the 8 warp sums are
// combined in warp order through shared memory into one fp32 partial per
// block, and the last block of each column slice (arrival counter) folds the
// partials in block order into out = q(out + sum) and re-arms the counter.
// Every association is fixed, so the result is deterministic.
// LN: vector 0 = sum dy * xhat (dgamma), vector 1 = sum dy (dbeta).
template <typename T, bool LN>
__global__ void __launch_bounds__(256) colred_k(const T* __restrict__ dy, const T* __restrict__ x,
                                               const float2* __restrict__ stats, int rows, int n, int64_t ld, int rpb,
                                               float* __restrict__ part, int nblk, int32_t* __restrict__ counters,
                                               T* __restrict__ out0, T* __restrict__ out1) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  constexpr int NV = LN ? 2 : 1;
  constexpr int U = LN ? 4 : 8;  // rows in flight per warp
  __shared__ __align__(16) float red[NV][8][256];
  __shared__ int last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cb0 = blockIdx.x * 256, c = cb0 + lane * 8;
  const bool cok = c < n;
  const int r0 = blockIdx.y * rpb, r1 = min(rows, r0 + rpb);
  float sb[8] = {0, 0, 0, 0, 0, 0, 0, 0}, sg[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (cok) {
    for (int r = r0 + warp; r < r1; r += 8 * U) {
      uint4 gu[U], xu[U];
      float2 st[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int rr = r + 8 * j;
        if (rr < r1) {
          gu[j] = *reinterpret_cast<const uint4*>(dy + int64_t(rr) * ld + c);
          if (LN) {
            xu[j] = *reinterpret_cast<const uint4*>(x + int64_t(rr) * ld + c);
            st[j] = stats[rr];
          }
        }
      }
#pragma unroll
      for (int j = 0; j < U; ++j) {
        if (r + 8 * j >= r1) break;
        float gy[8];
        vec::V8<T>::unpack(gu[j], gy);
        if (LN) {
          float xh[8];
          vec::V8<T>::unpack(xu[j], xh);
#pragma unroll
          for (int e = 0; e < 8; ++e) sg[e] += gy[e] * __fmul_rn(__fsub_rn(xh[e], st[j].x), st[j].y);
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) sb[e] += gy[e];
      }
    }
  }
  {
    float* d0 = &red[0][warp][lane * 8];
    *reinterpret_cast<float4*>(d0) = LN ? make_float4(sg[0], sg[1], sg[2], sg[3]) : make_float4(sb[0], sb[1], sb[2], sb[3]);
    *reinterpret_cast<float4*>(d0 + 4) =
        LN ? make_float4(sg[4], sg[5], sg[6], sg[7]) : make_float4(sb[4], sb[5], sb[6], sb[7]);
    if (LN) {
      float* d1 = &red[NV - 1][warp][lane * 8];
      *reinterpret_cast<float4*>(d1) = make_float4(sb[0], sb[1], sb[2], sb[3]);
      *reinterpret_cast<float4*>(d1 + 4) = make_float4(sb[4], sb[5], sb[6], sb[7]);
    }
  }
  __syncthreads();
  const int col = cb0 + threadIdx.x;
  if (col < n) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += red[v][w][threadIdx.x];
      part[(int64_t(v) * nblk + blockIdx.y) * n + col] = t;
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counters + blockIdx.x, 1) == nblk - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // fold: warp w sums partials p = w, w+8, ... for 8 columns per lane (all
  // loads of a thread in flight together), then the 8 warp sums combine in
  // warp order -- a fixed association
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    float f[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (cok) {
      const float* pv = part + int64_t(v) * nblk * n + c;
      for (int p = warp; p < nblk; p += 64) {
        float4 q[8][2];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (p + 8 * j < nblk) {
            q[j][0] = __ldcg(reinterpret_cast<const float4*>(pv + int64_t(p + 8 * j) * n));
            q[j][1] = __ldcg(reinterpret_cast<const float4*>(pv + int64_t(p + 8 * j) * n + 4));
          }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (p + 8 * j < nblk) {
            f[0] += q[j][0].x, f[1] += q[j][0].y, f[2] += q[j][0].z, f[3] += q[j][0].w;
            f[4] += q[j][1].x, f[5] += q[j][1].y, f[6] += q[j][1].z, f[7] += q[j][1].w;
          }
      }
    }
    __syncthreads();
    float* d = &red[0][warp][lane * 8];
    *reinterpret_cast<float4*>(d) = make_float4(f[0], f[1], f[2], f[3]);
    *reinterpret_cast<float4*>(d + 4) = make_float4(f[4], f[5], f[6], f[7]);
    __syncthreads();
    if (col < n) {
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += red[0][w][threadIdx.x];
      T* o = v == 0 ? out0 : out1;
      Num<T>::st(o + col, Num<T>::ld(o + col) + t);
    }
  }
  if (threadIdx.x == 0) counters[blockIdx.x] = 0;
}

// rows per block of colred_k: about two blocks per SM in total
static void colred_grid(int rows, int n, int& col_blocks, int& nblk, int& rpb) {
  col_blocks = (n + 255) / 256;
  nblk = std::max(1, (2 * 148) / col_blocks);
  nblk = std::min(nblk, std::max(1, rows / 16));
  rpb = (rows + nblk - 1) / nblk;
  nblk = (rows + rpb - 1) / rpb;
}

int colred_launch(int dtype, bool ln, const void* dy, const void* x, const float* stats, int rows, int n, int64_t ld,
                  float* part, int32_t* counters, void* out0, void* out1, cudaStream_t s) {
  if (dtype == SFK_F32 || n % 8 || ld % 8 || !al16(dy) || (ln && !al16(x)) || !counters) return SFK_EUNSUP;
  int cbk, nblk, rpb;
  colred_grid(rows, n, cbk, nblk, rpb);
  const dim3 grid(cbk, nblk);
  auto st = reinterpret_cast<const float2*>(stats);
  if (dtype == SFK_F16) {
    auto k = ln ? colred_k<__half, true> : colred_k<__half, false>;
    launch_pdl(k, grid, dim3(256), 0, s, static_cast<const __half*>(dy), static_cast<const __half*>(x), st, rows, n, ld,
               rpb, part, nblk, counters, static_cast<__half*>(out0), static_cast<__half*>(out1));
  } else {
    auto k = ln ? colred_k<__nv_bfloat16, true> : colred_k<__nv_bfloat16, false>;
    launch_pdl(k, grid, dim3(256), 0, s, static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(x),
               st, rows, n, ld, rpb, part, nblk, counters, static_cast<__nv_bfloat16*>(out0),
               static_cast<__nv_bfloat16*>(out1));
  }
  return check_launch(ln ? "sfk_layernorm_bwd_params(colred)" : "sfk_colsum(colred)");
}

// row chunks for a column reduction: about two blocks per SM in total
static int fold_parts(int rows, int col_blocks) {
  int nblk = std::max(1, (148 * 2) / std::max(1, col_blocks));
  nblk = std::min(nblk, std::max(1, rows / 8));
  return nblk;
}

int ln_bwd_fused_vec(int dtype, const void* x, const void* dy, int rows, int d, const void* g, const float* stats,
                     void* dx, int accumulate, float* part, int32_t* /*counter*/, void* dgamma, void* dbeta,
                     cudaStream_t s) {
  if (dtype == SFK_F32 || d % 8 || d > 1024 || !al16(x) || !al16(dy) || !al16(dx) || !al16(g)) return SFK_EUNSUP;
  int nparts = 0;
  if (int e = ln_bwd_vec(dtype, x, dy, rows, d, g, stats, dx, accumulate, part, &nparts, s)) return e;
  dim3 grid((d + 7) / 8, 2);
  if (dtype == SFK_F16)
    launch_pdl(fold_k<__half>, grid, 256, 0, s, part, part + size_t(nparts) * d, nparts, d, static_cast<__half*>(dgamma),
                                        static_cast<__half*>(dbeta));
  else
    launch_pdl(fold_k<__nv_bfloat16>, grid, 256, 0, s, part, part + size_t(nparts) * d, nparts, d,
                                               static_cast<__nv_bfloat16*>(dgamma),
                                               static_cast<__nv_bfloat16*>(dbeta));
  return check_launch("sfk_layernorm_bwd_fused(fold)");
}

int ln_dx_part_vec(int dtype, const void* x, const void* dy, int rows, int d, const void* g, const float* stats,
                   void* dx, int accumulate, float* part, int* nparts, cudaStream_t s) {
  if (dtype == SFK_F32 || d % 8 || d > 1024 || !al16(x) || !al16(dy) || !al16(dx) || !al16(g)) return SFK_EUNSUP;
  const int per = 8 * vec::kLnRowsPerWarp;
  const int nblk = (rows + per - 1) / per;
  *nparts = nblk;
  const size_t smem = size_t(8) * d * sizeof(float);
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(vec::ln_dx_part_v<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(vec::ln_dx_part_v<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cfg = true;
  }
  if (dtype == SFK_F16)
    launch_pdl(vec::ln_dx_part_v<__half>, dim3(nblk), dim3(256), smem, s, static_cast<const __half*>(x),
               static_cast<const __half*>(dy), rows, d, static_cast<const __half*>(g),
               reinterpret_cast<const float2*>(stats), static_cast<__half*>(dx), accumulate, part, nblk);
  else
    launch_pdl(vec::ln_dx_part_v<__nv_bfloat16>, dim3(nblk), dim3(256), smem, s, static_cast<const __nv_bfloat16*>(x),
               static_cast<const __nv_bfloat16*>(dy), rows, d, static_cast<const __nv_bfloat16*>(g),
               reinterpret_cast<const float2*>(stats), static_cast<__nv_bfloat16*>(dx), accumulate, part, nblk);
  return check_launch("sfk_layernorm_bwd_dx_part(vec)");
}

int ln_gb_partial_vec(int dtype, const void* x, const void* dy, int rows, int d, const float* stats, float* part,
                      int* nparts, cudaStream_t s) {
  if (dtype == SFK_F32 || d % 8 || d > 1024 || !al16(x) || !al16(dy)) return SFK_EUNSUP;
  int nb = std::min(148, std::max(1, rows / 16));
  const int rpb = (rows + nb - 1) / nb;
  nb = (rows + rpb - 1) / rpb;
  *nparts = nb;
  const dim3 grid(nb, (d + 511) / 512);
  auto st = reinterpret_cast<const float2*>(stats);
  if (dtype == SFK_F16)
    launch_pdl(vec::ln_gb_part_k<__half>, grid, dim3(256), 0, s, static_cast<const __half*>(x),
               static_cast<const __half*>(dy), st, rows, d, rpb, part);
  else
    launch_pdl(vec::ln_gb_part_k<__nv_bfloat16>, grid, dim3(256), 0, s, static_cast<const __nv_bfloat16*>(x),
               static_cast<const __nv_bfloat16*>(dy), st, rows, d, rpb, part);
  return check_launch("sfk_layernorm_bwd_params_partial");
}

int ln_gb_fold_vec(int dtype, const sfk_ln_fold_job* jobs, int njobs, cudaStream_t s) {
  if (dtype == SFK_F32) return SFK_EUNSUP;
  if (njobs <= 0) return SFK_OK;
  if (njobs > SFK_LN_FOLD_MAX_JOBS) return SFK_EINVAL;
  vec::LnFoldBatch B{};
  int dmax = 0;
  for (int j = 0; j < njobs; ++j) {
    B.job[j] = jobs[j];
    dmax = std::max(dmax, jobs[j].d);
  }
  const dim3 grid((dmax + 31) / 32, 2, njobs);
  if (dtype == SFK_F16)
    launch_pdl(vec::ln_gb_fold_k<__half>, grid, dim3(256), 0, s, B);
  else
    launch_pdl(vec::ln_gb_fold_k<__nv_bfloat16>, grid, dim3(256), 0, s, B);
  return check_launch("sfk_layernorm_bwd_params_fold");
}

int fold2_vec(int dtype, const float* part, int nparts, int d, void* dgamma, void* dbeta, cudaStream_t s) {
  if (dtype == SFK_F32) return SFK_EUNSUP;
  dim3 grid((d + 7) / 8, dbeta ? 2 : 1);
  if (dtype == SFK_F16)
    launch_pdl(fold_k<__half>, grid, 256, 0, s, part, part + size_t(nparts) * d, nparts, d, static_cast<__half*>(dgamma),
               static_cast<__half*>(dbeta));
  else
    launch_pdl(fold_k<__nv_bfloat16>, grid, 256, 0, s, part, part + size_t(nparts) * d, nparts, d,
               static_cast<__nv_bfloat16*>(dgamma), static_cast<__nv_bfloat16*>(dbeta));
  return check_launch("sfk_layernorm_bwd_fold");
}

int ln_dx_acc_vec(int dtype, const void* x, const void* dy, int rows, int d, const void* g, const float* stats,
                  const void* acc, void* dx, cudaStream_t s) {
  if (dtype == SFK_F32 || d % 8 || d > 1024 || !al16(x) || !al16(dy) || !al16(dx) || !al16(g) || (acc && !al16(acc)))
    return SFK_EUNSUP;
  const int blocks = (rows + 3) / 4;
  if (dtype == SFK_F16)
    launch_pdl(vec::ln_dx_v<__half>, dim3(blocks), dim3(128), 0, s, static_cast<const __half*>(x),
               static_cast<const __half*>(dy), rows, d, static_cast<const __half*>(g),
               reinterpret_cast<const float2*>(stats), static_cast<__half*>(dx), static_cast<const __half*>(acc));
  else
    launch_pdl(vec::ln_dx_v<__nv_bfloat16>, dim3(blocks), dim3(128), 0, s, static_cast<const __nv_bfloat16*>(x),
               static_cast<const __nv_bfloat16*>(dy), rows, d, static_cast<const __nv_bfloat16*>(g),
               reinterpret_cast<const float2*>(stats), static_cast<__nv_bfloat16*>(dx),
               static_cast<const __nv_bfloat16*>(acc));
  return check_launch("sfk_layernorm_bwd_dx(vec)");
}

int ln_dx_vec(int dtype, const void* x, const void* dy, int rows, int d, const void* g, const float* stats, void* dx,
              int accumulate, cudaStream_t s) {
  return ln_dx_acc_vec(dtype, x, dy, rows, d, g, stats, accumulate ? dx : nullptr, dx, s);
}

int ln_params_vec(int dtype, const void* x, const void* dy, int rows, int d, const float* stats, float* part,
                  void* dgamma, void* dbeta, cudaStream_t s) {
  if (dtype == SFK_F32 || d % 8 || !al16(x) || !al16(dy)) return SFK_EUNSUP;
  const int col_blocks = (d / 8 + 127) / 128;
  const int nblk = fold_parts(rows, col_blocks);
  const int rpb = (rows + nblk - 1) / nblk;
  if (dtype == SFK_F16)
    launch_pdl(vec::ln_dgb_partial_v<__half>, dim3(col_blocks, nblk), dim3(128), 0, s, static_cast<const __half*>(x),
               static_cast<const __half*>(dy), rows, d, reinterpret_cast<const float2*>(stats), rpb, part, nblk);
  else
    launch_pdl(vec::ln_dgb_partial_v<__nv_bfloat16>, dim3(col_blocks, nblk), dim3(128), 0, s,
               static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(dy), rows, d,
               reinterpret_cast<const float2*>(stats), rpb, part, nblk);
  dim3 grid((d + 7) / 8, 2);
  if (dtype == SFK_F16)
    launch_pdl(fold_k<__half>, grid, 256, 0, s, part, part + size_t(nblk) * d, nblk, d, static_cast<__half*>(dgamma),
               static_cast<__half*>(dbeta));
  else
    launch_pdl(fold_k<__nv_bfloat16>, grid, 256, 0, s, part, part + size_t(nblk) * d, nblk, d,
               static_cast<__nv_bfloat16*>(dgamma), static_cast<__nv_bfloat16*>(dbeta));
  return check_launch("sfk_layernorm_bwd_params(vec)");
}

int colsum_fused_vec(int dtype, const void* x, int rows, int n, int64_t ld, float* part, int32_t* /*counters*/,
                     void* out, cudaStream_t s) {
  if (dtype == SFK_F32 || n % 8 || ld % 8 || !al16(x)) return SFK_EUNSUP;
  int nparts = 0;
  if (int e = colsum_partial_vec(dtype, x, rows, n, ld, part, &nparts, s)) return e;
  dim3 grid((n + 7) / 8, 1);
  if (dtype == SFK_F16)
    launch_pdl(fold_k<__half>, grid, 256, 0, s, part, nullptr, nparts, n, static_cast<__half*>(out), nullptr);
  else
    launch_pdl(fold_k<__nv_bfloat16>, grid, 256, 0, s, part, nullptr, nparts, n, static_cast<__nv_bfloat16*>(out), nullptr);
  return check_launch("sfk_colsum(fold)");
}

int colsum_partial_vec(int dtype, const void* x, int rows, int n, int64_t ld, float* part, int* nparts,
                       cudaStream_t s) {
  if (dtype == SFK_F32 || n % 8 || ld % 8 || !al16(x)) return SFK_EUNSUP;
  // enough row chunks to fill the machine: ~4 blocks of 128 threads per SM
  // enough row chunks for ~4 blocks per SM; partial scratch capped at 4M floats
  const int col_blocks = (n / 8 + 127) / 128;
  int nblk = fold_parts(rows, col_blocks);
  nblk = std::min(nblk, std::max(1, (4 << 20) / std::max(1, n)));
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

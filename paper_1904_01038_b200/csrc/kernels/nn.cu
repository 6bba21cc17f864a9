// Memory-bound kernels of the training step: embedding front (a8), embedding
// backward (scatter-add, a8 bwd), layer norm (a14), bias-grad column sums
// (a11), fused label-smoothed cross entropy fwd+bwd (a18/a19).
// Elementwise arithmetic uses explicit _rn intrinsics where the reference
// evaluates separate IEEE multiplies/adds (no FMA contraction on its x86-64
// build), so rounding points line up with the reference's.
#include <cfloat>

#include "common.cuh"

namespace sfk {

// ------------------------------------------------------------------ embedding
template <typename T>
__global__ void embed_fwd_k(const int32_t* __restrict__ ids, int rows, int width, int d, const T* __restrict__ table,
                            const float* __restrict__ pe, float scale, T* __restrict__ out) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  const int r = blockIdx.x;
  if (r >= rows) return;
  const int64_t id = ids[r];
  const int pos = r % width;
  const T* e = table + id * d;
  const float* p = pe + int64_t(pos) * d;
  T* o = out + int64_t(r) * d;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    // lookup (already on the storage grid) -> q(scale*e) -> + q(pe) -> q()
    const float scaled = Num<T>::rnd(__fmul_rn(scale, Num<T>::ld(e + c)));
    Num<T>::st(o + c, __fadd_rn(scaled, Num<T>::rnd(p[c])));
  }
}

template <typename T>
__global__ void embed_bwd_k(const int32_t* __restrict__ uniq, const int32_t* __restrict__ seg_off,
                            const int32_t* __restrict__ seg_rows, int d, const T* __restrict__ dx, float scale,
                            T* __restrict__ grad) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  const int u = blockIdx.x;
  const int64_t id = uniq[u];
  const int s0 = seg_off[u], s1 = seg_off[u + 1];
  T* g = grad + id * d;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float acc = Num<T>::ld(g + c);
    for (int s = s0; s < s1; ++s) {
      const int64_t r = seg_rows[s];
      acc = __fadd_rn(acc, Num<T>::rnd(__fmul_rn(scale, Num<T>::ld(dx + r * d + c))));
    }
    Num<T>::st(g + c, acc);
  }
}

// ------------------------------------------------------------------ layer norm
constexpr float kLnEps = 1e-5f;  // kernels.hpp:12
constexpr int kLnMaxPerLane = 32;  // d <= 1024

template <typename T>
__global__ void __launch_bounds__(256) ln_fwd_k(const T* __restrict__ x, int rows, int d, const T* __restrict__ g,
                                                const T* __restrict__ b, T* __restrict__ y, float2* __restrict__ stats) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  if (warp >= rows) return;
  const T* xr = x + int64_t(warp) * d;
  float v[kLnMaxPerLane];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kLnMaxPerLane; ++i) {
    const int c = lane + 32 * i;
    v[i] = c < d ? Num<T>::ld(xr + c) : 0.f;
    s += v[i];
  }
  const float mean = __fdiv_rn(warp_sum(s), float(d));
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < kLnMaxPerLane; ++i) {
    const int c = lane + 32 * i;
    if (c < d) {
      const float t = __fsub_rn(v[i], mean);
      q = __fadd_rn(q, __fmul_rn(t, t));
    }
  }
  const float var = __fdiv_rn(warp_sum(q), float(d));
  const float rstd = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, kLnEps)));
  T* yr = y + int64_t(warp) * d;
#pragma unroll
  for (int i = 0; i < kLnMaxPerLane; ++i) {
    const int c = lane + 32 * i;
    if (c < d) {
      const float t = __fmul_rn(__fmul_rn(__fsub_rn(v[i], mean), rstd), Num<T>::ld(g + c));
      Num<T>::st(yr + c, __fadd_rn(t, Num<T>::ld(b + c)));
    }
  }
  if (lane == 0) stats[warp] = make_float2(mean, rstd);
}

// one block = 8 warps handles a contiguous chunk of rows; per-block column
// partials of dy*xhat (gamma) and dy (beta) go to part[0|1][blockIdx][d]
template <typename T>
__global__ void __launch_bounds__(256) ln_bwd_k(const T* __restrict__ x, const T* __restrict__ dy, int rows, int d,
                                                const T* __restrict__ g, const float2* __restrict__ stats,
                                                T* __restrict__ dx, int accumulate, int rows_per_block,
                                                float* __restrict__ part, int nblk) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  __shared__ float red[2][8][kLnMaxPerLane * 32 / 8];  // reused per column slab
  const int wid = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int r0 = blockIdx.x * rows_per_block;
  const int r1 = min(rows, r0 + rows_per_block);
  float pg[kLnMaxPerLane], pb[kLnMaxPerLane];
#pragma unroll
  for (int i = 0; i < kLnMaxPerLane; ++i) pg[i] = pb[i] = 0.f;
  const float inv_n = __fdiv_rn(1.0f, float(d));
  for (int r = r0 + wid; r < r1; r += 8) {
    const float2 st = stats[r];
    const T* xr = x + int64_t(r) * d;
    const T* gr = dy + int64_t(r) * d;
    float xh[kLnMaxPerLane], dxh[kLnMaxPerLane], gy[kLnMaxPerLane];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < kLnMaxPerLane; ++i) {
      const int c = lane + 32 * i;
      if (c < d) {
        xh[i] = __fmul_rn(__fsub_rn(Num<T>::ld(xr + c), st.x), st.y);
        gy[i] = Num<T>::ld(gr + c);
        dxh[i] = __fmul_rn(gy[i], Num<T>::ld(g + c));
        s1 += dxh[i];
        s2 += dxh[i] * xh[i];
      } else {
        xh[i] = dxh[i] = gy[i] = 0.f;
      }
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    const float m1 = __fmul_rn(s1, inv_n), m2 = __fmul_rn(s2, inv_n);
    T* dr = dx + int64_t(r) * d;
#pragma unroll
    for (int i = 0; i < kLnMaxPerLane; ++i) {
      const int c = lane + 32 * i;
      if (c < d) {
        const float v = __fmul_rn(st.y, __fsub_rn(__fsub_rn(dxh[i], m1), __fmul_rn(xh[i], m2)));
        const float old = accumulate ? Num<T>::ld(dr + c) : 0.f;
        Num<T>::st(dr + c, __fadd_rn(old, v));
        pg[i] += gy[i] * xh[i];
        pb[i] += gy[i];
      }
    }
  }
  // reduce the 8 warps' partials column slab by column slab (4 per-lane slots at a time)
  for (int base = 0; base < kLnMaxPerLane; base += 4) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      red[0][wid][j * 32 + lane] = pg[base + j];
      red[1][wid][j * 32 + lane] = pb[base + j];
    }
    __syncthreads();
    if (threadIdx.x < 128) {
      const int j = threadIdx.x / 32, l = threadIdx.x % 32;
      const int c = l + 32 * (base + j);
      float sg = 0.f, sb = 0.f;
      for (int w = 0; w < 8; ++w) {
        sg += red[0][w][j * 32 + l];
        sb += red[1][w][j * 32 + l];
      }
      if (c < d) {
        part[int64_t(blockIdx.x) * d + c] = sg;
        part[int64_t(nblk + blockIdx.x) * d + c] = sb;
      }
    }
    __syncthreads();
    if (32 * (base + 4) >= d) break;
  }
}

// ------------------------------------------------------------------ column sums
template <typename T>
__global__ void colsum_partial_k(const T* __restrict__ x, int rows, int n, int64_t ld, int rows_per_block,
                                 float* __restrict__ part) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int r0 = blockIdx.y * rows_per_block, r1 = min(rows, r0 + rows_per_block);
  float s = 0.f;
  for (int r = r0; r < r1; ++r) s += Num<T>::ld(x + int64_t(r) * ld + c);
  part[int64_t(blockIdx.y) * n + c] = s;
}

template <typename T>
__global__ void colsum_finish_k(const float* __restrict__ part, int nparts, int n, T* __restrict__ out) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  float s = 0.f;
  for (int p = 0; p < nparts; ++p) s += part[int64_t(p) * n + c];
  Num<T>::st(out + c, Num<T>::ld(out + c) + s);
}

// ------------------------------------------------------------------ xent
// Block per row; the row is staged in shared memory once, then three passes:
// (max, first argmax) -> sum exp -> dlogits + smoothing sum. Matches
// kernels.cpp:80-95 / tape.cpp:259-290, 481-502.
template <typename T>
__global__ void __launch_bounds__(1024) xent_k(T* __restrict__ logits, int rows, int V, int64_t ld,
                                               const int32_t* __restrict__ gold, int pad, float eps, float seed,
                                               T* __restrict__ dlogits, float* __restrict__ row_out) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  extern __shared__ uint8_t xs_raw[];
  T* row = reinterpret_cast<T*>(xs_raw);
  __shared__ float rv[32];
  __shared__ int ri[32];
  const int r = blockIdx.x;
  const int tid = threadIdx.x, lane = tid % 32, wid = tid / 32, nw = blockDim.x / 32;
  const int gid = gold[r];
  T* src = logits + int64_t(r) * ld;
  T* dst = dlogits + int64_t(r) * ld;
  const bool wr = dlogits != nullptr;
  if (gid == pad) {
    if (wr)
      for (int c = tid; c < V; c += blockDim.x) Num<T>::st(dst + c, 0.f);
    if (tid == 0) {
      row_out[4 * r + 0] = 0.f;
      row_out[4 * r + 1] = 0.f;
      row_out[4 * r + 2] = 0.f;
      row_out[4 * r + 3] = 0.f;
    }
    return;
  }
  // pass 1: stage + max + first argmax
  float m = -INFINITY;
  int mi = 0x7fffffff;
  for (int c = tid; c < V; c += blockDim.x) {
    const T v = src[c];
    row[c] = v;
    const float f = Num<T>::ld(&v);
    if (f > m || (f == m && c < mi)) {
      m = f;
      mi = c;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, m, o);
    const int oi = __shfl_xor_sync(0xffffffffu, mi, o);
    if (om > m || (om == m && oi < mi)) {
      m = om;
      mi = oi;
    }
  }
  if (lane == 0) {
    rv[wid] = m;
    ri[wid] = mi;
  }
  __syncthreads();
  if (wid == 0) {
    m = lane < nw ? rv[lane] : -INFINITY;
    mi = lane < nw ? ri[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, m, o);
      const int oi = __shfl_xor_sync(0xffffffffu, mi, o);
      if (om > m || (om == m && oi < mi)) {
        m = om;
        mi = oi;
      }
    }
    if (lane == 0) {
      rv[0] = m;
      ri[0] = mi;
    }
  }
  __syncthreads();
  const float mx = rv[0];
  const int amax = ri[0];
  __syncthreads();
  // pass 2: sum exp(l - max)
  float s = 0.f;
  for (int c = tid; c < V; c += blockDim.x) s += expf(__fsub_rn(Num<T>::ld(&row[c]), mx));
  s = warp_sum(s);
  if (lane == 0) rv[wid] = s;
  __syncthreads();
  if (wid == 0) {
    s = lane < nw ? rv[lane] : 0.f;
    s = warp_sum(s);
    if (lane == 0) rv[0] = s;
  }
  __syncthreads();
  const float lse = __fadd_rn(mx, logf(rv[0]));
  __syncthreads();
  // pass 3: dlogits = q(seed*(p - target)); smoothing sum of (lse - l)
  const float uni = __fdiv_rn(eps, float(V));
  const float on = __fadd_rn(1.0f - eps, uni);
  float sm = 0.f;
  for (int c = tid; c < V; c += blockDim.x) {
    const float l = Num<T>::ld(&row[c]);
    const float p = expf(__fsub_rn(l, lse));
    const float tgt = c == gid ? on : uni;
    if (wr) Num<T>::st(dst + c, __fmul_rn(seed, __fsub_rn(p, tgt)));
    sm += __fsub_rn(lse, l);
  }
  sm = warp_sum(sm);
  if (lane == 0) rv[wid] = sm;
  __syncthreads();
  if (tid == 0) {
    float tot = 0.f;
    for (int w = 0; w < nw; ++w) tot += rv[w];
    const float nll = __fsub_rn(lse, Num<T>::ld(&row[gid]));
    float loss = nll;
    if (eps != 0.0f) loss = __fadd_rn(__fmul_rn(1.0f - eps, nll), __fmul_rn(__fdiv_rn(eps, float(V)), tot));
    row_out[4 * r + 0] = Num<T>::rnd(loss);
    row_out[4 * r + 1] = nll;
    row_out[4 * r + 2] = amax == gid ? 1.f : 0.f;
    row_out[4 * r + 3] = 1.f;
  }
}

__global__ void xent_reduce_k(const float* __restrict__ row_out, int rows, double* __restrict__ acc) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  __shared__ double red[4][256];
  const int tid = threadIdx.x;
  const int per = (rows + blockDim.x - 1) / blockDim.x;
  double s[4] = {0, 0, 0, 0};
  for (int r = tid * per; r < min(rows, (tid + 1) * per); ++r) {
    if (row_out[4 * r + 3] == 0.f) continue;
    s[0] += double(row_out[4 * r + 0]);
    s[1] += double(row_out[4 * r + 1]);
    s[2] += 1.0;
    s[3] += double(row_out[4 * r + 2]);
  }
  for (int j = 0; j < 4; ++j) red[j][tid] = s[j];
  __syncthreads();
  if (tid < 4) {
    double t = 0;
    for (int i = 0; i < blockDim.x; ++i) t += red[tid][i];
    acc[tid] += t;
  }
}

}  // namespace sfk

namespace sfk {
int embed_fwd_vec(int, const int32_t*, int, int, int, const void*, const float*, float, void*, cudaStream_t);
int embed_bwd_chunked_vec(int, const int32_t*, int, const int32_t*, int, const int32_t*, int, const void*, float, float*,
                          void*, cudaStream_t);
int embed_bwd_vec(int, const int32_t*, const int32_t*, const int32_t*, int, int, const void*, float, void*,
                  cudaStream_t);
int ln_fwd_vec(int, const void*, int, int, const void*, const void*, void*, float*, cudaStream_t);
int ln_bwd_vec(int, const void*, const void*, int, int, const void*, const float*, void*, int, float*, int*,
               cudaStream_t);
int colsum_partial_vec(int, const void*, int, int, int64_t, float*, int*, cudaStream_t);
int ln_bwd_fused_vec(int, const void*, const void*, int, int, const void*, const float*, void*, int, float*,
                     int32_t*, void*, void*, cudaStream_t);
int colsum_fused_vec(int, const void*, int, int, int64_t, float*, int32_t*, void*, cudaStream_t);
int ln_dx_acc_vec(int, const void*, const void*, int, int, const void*, const float*, const void*, void*, cudaStream_t);
int ln_dx_part_vec(int, const void*, const void*, int, int, const void*, const float*, void*, int, float*, int*,
                   cudaStream_t);
int fold2_vec(int, const float*, int, int, void*, void*, cudaStream_t);
int ln_gb_partial_vec(int, const void*, const void*, int, int, const float*, float*, int*, cudaStream_t);
int ln_gb_fold_vec(int, const sfk_ln_fold_job*, int, cudaStream_t);
int colred_launch(int, bool, const void*, const void*, const float*, int, int, int64_t, float*, int32_t*, void*, void*,
                  cudaStream_t);
int xent_vec(int, void*, int, int, int64_t, const int32_t*, int, float, float, void*, float*, cudaStream_t);
int ln_dx_vec(int, const void*, const void*, int, int, const void*, const float*, void*, int, cudaStream_t);
int ln_params_vec(int, const void*, const void*, int, int, const float*, float*, void*, void*, cudaStream_t);
}  // namespace sfk

extern "C" int sfk_layernorm_bwd_dx(int dtype, const void* x, const void* dy, int rows, int d, const void* gamma,
                                    const float* stats, void* dx, int accumulate, void* stream) {
  if (rows == 0) return SFK_OK;
  const int e = sfk::ln_dx_vec(dtype, x, dy, rows, d, gamma, stats, dx, accumulate, sfk::as_stream(stream));
  if (e == SFK_EUNSUP) sfk::set_error("sfk_layernorm_bwd_dx: needs 16-bit data, d % 8 == 0, d <= 1024, aligned rows");
  return e;
}

extern "C" int sfk_layernorm_bwd_dx_acc(int dtype, const void* x, const void* dy, int rows, int d, const void* gamma,
                                        const float* stats, const void* acc, void* dx, void* stream) {
  if (rows == 0) return SFK_OK;
  const int e = sfk::ln_dx_acc_vec(dtype, x, dy, rows, d, gamma, stats, acc, dx, sfk::as_stream(stream));
  if (e == SFK_EUNSUP) sfk::set_error("sfk_layernorm_bwd_dx_acc: needs 16-bit data, d % 8 == 0, d <= 1024, aligned rows");
  return e;
}

extern "C" int sfk_layernorm_bwd_dx_part(int dtype, const void* x, const void* dy, int rows, int d, const void* gamma,
                                         const float* stats, void* dx, int accumulate, float* part, int* nparts,
                                         void* stream) {
  *nparts = 0;
  if (rows == 0) return SFK_OK;
  const int e = sfk::ln_dx_part_vec(dtype, x, dy, rows, d, gamma, stats, dx, accumulate, part, nparts,
                                    sfk::as_stream(stream));
  if (e == SFK_EUNSUP) sfk::set_error("sfk_layernorm_bwd_dx_part: needs 16-bit data, d % 8 == 0, d <= 1024, aligned rows");
  return e;
}

extern "C" int sfk_layernorm_bwd_fold(int dtype, const float* part, int nparts, int d, void* dgamma, void* dbeta,
                                      void* stream) {
  if (nparts == 0) return SFK_OK;
  const int e = sfk::fold2_vec(dtype, part, nparts, d, dgamma, dbeta, sfk::as_stream(stream));
  if (e == SFK_EUNSUP) sfk::set_error("sfk_layernorm_bwd_fold: needs 16-bit data");
  return e;
}

extern "C" int sfk_layernorm_bwd_params_partial(int dtype, const void* x, const void* dy, int rows, int d,
                                                const float* stats, float* part, int* nparts, void* stream) {
  *nparts = 0;
  if (rows == 0) return SFK_OK;
  const int e = sfk::ln_gb_partial_vec(dtype, x, dy, rows, d, stats, part, nparts, sfk::as_stream(stream));
  if (e == SFK_EUNSUP) sfk::set_error("sfk_layernorm_bwd_params_partial: needs 16-bit data, d % 8 == 0, d <= 1024");
  return e;
}

extern "C" int sfk_layernorm_bwd_params_fold(int dtype, const sfk_ln_fold_job* jobs, int njobs, void* stream) {
  const int e = sfk::ln_gb_fold_vec(dtype, jobs, njobs, sfk::as_stream(stream));
  if (e == SFK_EUNSUP) sfk::set_error("sfk_layernorm_bwd_params_fold: needs 16-bit data");
  if (e == SFK_EINVAL) sfk::set_error("sfk_layernorm_bwd_params_fold: too many jobs");
  return e;
}

extern "C" int sfk_layernorm_bwd_params(int dtype, const void* x, const void* dy, int rows, int d, const float* stats,
                                        float* part, int32_t* counters, void* dgamma, void* dbeta, void* stream) {
  if (rows == 0) return SFK_OK;
  if (int e = sfk::colred_launch(dtype, true, dy, x, stats, rows, d, d, part, counters, dgamma, dbeta,
                                 sfk::as_stream(stream));
      e != SFK_EUNSUP)
    return e;
  const int e = sfk::ln_params_vec(dtype, x, dy, rows, d, stats, part, dgamma, dbeta, sfk::as_stream(stream));
  if (e == SFK_EUNSUP) sfk::set_error("sfk_layernorm_bwd_params: needs 16-bit data, d % 8 == 0, aligned rows");
  return e;
}

extern "C" int sfk_layernorm_bwd_fused(int dtype, const void* x, const void* dy, int rows, int d, const void* gamma,
                                       const float* stats, void* dx, int accumulate, float* part, int32_t* counter,
                                       void* dgamma, void* dbeta, void* stream) {
  if (rows == 0) return SFK_OK;
  cudaStream_t s = sfk::as_stream(stream);
  if (int e = sfk::ln_bwd_fused_vec(dtype, x, dy, rows, d, gamma, stats, dx, accumulate, part, counter, dgamma, dbeta,
                                    s);
      e != SFK_EUNSUP)
    return e;
  int nparts = 0;
  if (int e = sfk_layernorm_bwd(dtype, x, dy, rows, d, gamma, stats, dx, accumulate, part, &nparts, stream)) return e;
  if (int e = sfk_colsum_finish(dtype, part, nparts, d, dgamma, stream)) return e;
  return sfk_colsum_finish(dtype, part + size_t(nparts) * d, nparts, d, dbeta, stream);
}

extern "C" int sfk_colsum(int dtype, const void* x, int rows, int n, int64_t ld, float* part, int32_t* counters,
                          void* out, void* stream) {
  if (rows == 0 || n == 0) return SFK_OK;
  if (int e = sfk::colred_launch(dtype, false, x, nullptr, nullptr, rows, n, ld, part, counters, out, nullptr,
                                 sfk::as_stream(stream));
      e != SFK_EUNSUP)
    return e;
  if (int e = sfk::colsum_fused_vec(dtype, x, rows, n, ld, part, counters, out, sfk::as_stream(stream));
      e != SFK_EUNSUP)
    return e;
  int nparts = 0;
  if (int e = sfk_colsum_partial(dtype, x, rows, n, ld, part, &nparts, stream)) return e;
  return sfk_colsum_finish(dtype, part, nparts, n, out, stream);
}

using namespace sfk;

extern "C" int sfk_embed_fwd(int dtype, const int32_t* ids, int rows, int width, int d, const void* table,
                             const float* pe, float scale, void* out, void* stream) {
  if (rows == 0) return SFK_OK;
  if (rows < 0 || width <= 0 || d <= 0) return SFK_EINVAL;
  if (int e = embed_fwd_vec(dtype, ids, rows, width, d, table, pe, scale, out, as_stream(stream)); e != SFK_EUNSUP)
    return e;
  SFK_DISPATCH(dtype, T,
               launch_pdl(embed_fwd_k<T>, rows, 128, 0, as_stream(stream), ids, rows, width, d, static_cast<const T*>(table),
                                                                    pe, scale, static_cast<T*>(out)));
  return check_launch("sfk_embed_fwd");
}

extern "C" int sfk_embed_bwd_chunked(int dtype, const int32_t* chunks, int nchunks, const int32_t* multi, int nmulti,
                                     const int32_t* seg_rows, int d, const void* dx, float scale, float* scratch,
                                     void* grad, void* stream) {
  if (nchunks == 0) return SFK_OK;
  const int e = embed_bwd_chunked_vec(dtype, chunks, nchunks, multi, nmulti, seg_rows, d, dx, scale, scratch, grad,
                                      as_stream(stream));
  if (e == SFK_EUNSUP) set_error("sfk_embed_bwd_chunked: needs 16-bit data, d % 8 == 0, aligned rows, scratch");
  return e;
}

extern "C" int sfk_embed_bwd(int dtype, const int32_t* uniq, const int32_t* seg_off, const int32_t* seg_rows,
                             int nuniq, int d, const void* dx, float scale, void* grad, void* stream) {
  if (nuniq == 0) return SFK_OK;
  if (int e = embed_bwd_vec(dtype, uniq, seg_off, seg_rows, nuniq, d, dx, scale, grad, as_stream(stream));
      e != SFK_EUNSUP)
    return e;
  SFK_DISPATCH(dtype, T,
               launch_pdl(embed_bwd_k<T>, nuniq, 128, 0, as_stream(stream), uniq, seg_off, seg_rows, d,
                                                                    static_cast<const T*>(dx), scale,
                                                                    static_cast<T*>(grad)));
  return check_launch("sfk_embed_bwd");
}

extern "C" int sfk_layernorm_fwd(int dtype, const void* x, int rows, int d, const void* gamma, const void* beta,
                                 void* y, float* stats, void* stream) {
  if (rows == 0) return SFK_OK;
  if (d > 32 * kLnMaxPerLane) {
    set_error("sfk_layernorm_fwd: d > 1024 unsupported");
    return SFK_EUNSUP;
  }
  if (int e = ln_fwd_vec(dtype, x, rows, d, gamma, beta, y, stats, as_stream(stream)); e != SFK_EUNSUP) return e;
  const int blocks = (rows + 7) / 8;
  SFK_DISPATCH(dtype, T,
               launch_pdl(ln_fwd_k<T>, blocks, 256, 0, as_stream(stream), 
                   static_cast<const T*>(x), rows, d, static_cast<const T*>(gamma), static_cast<const T*>(beta),
                   static_cast<T*>(y), reinterpret_cast<float2*>(stats)));
  return check_launch("sfk_layernorm_fwd");
}

extern "C" int sfk_layernorm_bwd(int dtype, const void* x, const void* dy, int rows, int d, const void* gamma,
                                 const float* stats, void* dx, int accumulate, float* part, int* nparts,
                                 void* stream) {
  if (d > 32 * kLnMaxPerLane) {
    set_error("sfk_layernorm_bwd: d > 1024 unsupported");
    return SFK_EUNSUP;
  }
  if (rows == 0) {
    *nparts = 0;
    return SFK_OK;
  }
  if (int e = ln_bwd_vec(dtype, x, dy, rows, d, gamma, stats, dx, accumulate, part, nparts, as_stream(stream));
      e != SFK_EUNSUP)
    return e;
  int nblk = (rows + 31) / 32;
  if (nblk > 296) nblk = 296;
  if (nblk < 1) nblk = 1;
  const int rpb = (rows + nblk - 1) / nblk;
  *nparts = nblk;
  SFK_DISPATCH(dtype, T,
               launch_pdl(ln_bwd_k<T>, nblk, 256, 0, as_stream(stream), 
                   static_cast<const T*>(x), static_cast<const T*>(dy), rows, d, static_cast<const T*>(gamma),
                   reinterpret_cast<const float2*>(stats), static_cast<T*>(dx), accumulate, rpb, part, nblk));
  return check_launch("sfk_layernorm_bwd");
}

extern "C" int sfk_colsum_partial(int dtype, const void* x, int rows, int n, int64_t ld, float* part, int* nparts,
                                  void* stream) {
  if (int e = colsum_partial_vec(dtype, x, rows, n, ld, part, nparts, as_stream(stream)); e != SFK_EUNSUP) return e;
  int nblk = (rows + 63) / 64;
  if (nblk > 64) nblk = 64;
  if (nblk < 1) nblk = 1;
  const int rpb = (rows + nblk - 1) / nblk;
  *nparts = nblk;
  dim3 grid((n + 255) / 256, nblk);
  SFK_DISPATCH(dtype, T,
               launch_pdl(colsum_partial_k<T>, grid, 256, 0, as_stream(stream), static_cast<const T*>(x), rows, n, ld, rpb,
                                                                        part));
  return check_launch("sfk_colsum_partial");
}

extern "C" int sfk_colsum_finish(int dtype, const float* part, int nparts, int n, void* out, void* stream) {
  SFK_DISPATCH(dtype, T,
               launch_pdl(colsum_finish_k<T>, (n + 255) / 256, 256, 0, as_stream(stream), part, nparts, n,
                                                                                  static_cast<T*>(out)));
  return check_launch("sfk_colsum_finish");
}

extern "C" int sfk_xent_fwd_bwd(int dtype, void* logits, int rows, int vocab, int64_t ld, const int32_t* gold,
                                int pad_id, float eps, float seed, void* dlogits, float* row_out, void* stream) {
  if (rows == 0) return SFK_OK;
  if (int e = xent_vec(dtype, logits, rows, vocab, ld, gold, pad_id, eps, seed, dlogits, row_out, as_stream(stream));
      e != SFK_EUNSUP)
    return e;
  const size_t smem = size_t(vocab) * elem_size(dtype);
  if (smem > 200 * 1024) {
    set_error("sfk_xent_fwd_bwd: vocab too large for the staged row");
    return SFK_EUNSUP;
  }
  SFK_DISPATCH(dtype, T, {
    static int configured = 0;
    if (!configured) {
      cudaFuncSetAttribute(xent_k<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      configured = 1;
    }
    launch_pdl(xent_k<T>, rows, 1024, smem, as_stream(stream), static_cast<T*>(logits), rows, vocab, ld, gold, pad_id, eps,
                                                       seed, static_cast<T*>(dlogits), row_out);
  });
  return check_launch("sfk_xent_fwd_bwd");
}

extern "C" int sfk_xent_reduce(const float* row_out, int rows, double* acc, void* stream) {
  launch_pdl(xent_reduce_k, 1, 256, 0, as_stream(stream), row_out, rows, acc);
  return check_launch("sfk_xent_reduce");
}

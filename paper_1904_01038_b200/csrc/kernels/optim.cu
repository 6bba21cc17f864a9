// Optimizer-side kernels: overflow check (trainer.cpp:247-253), fused
// unscale + 1/ntokens + Adam (trainer.cpp:260-268, optim.cpp:48-66) with the
// fp16 shadow rebroadcast (trainer.cpp:149-156), SGD, casts.
// Adam runs in double exactly as the reference (double m/v/update math, fp32
// storage), so given identical gradients the update is bit-identical.
#include "common.cuh"

namespace sfk {

template <typename T>
__global__ void nonfinite_k(const T* __restrict__ g, int64_t n, int32_t* flag) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  int bad = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    bad |= !isfinite(Num<T>::ld(g + i));
  bad = __syncthreads_or(bad);
  if (bad && threadIdx.x == 0) atomicOr(flag, 1);
}

// Per-update constants. Division by the update's constants (loss scale,
// token count, bias corrections) uses the correctly rounded reciprocal and
// one FMA correction (Markstein): q = RN(a*y), r = a - b*q (exact by FMA),
// RN(q + r*y) is the correctly rounded a/b when y = RN(1/b) -- the same bits
// as a true division at a fraction of its cost. Only the per-element
// division by sqrt(vhat) + eps and the square root stay full IEEE ops.
struct AdamConst {
  double lr, b1, b2, eps, bc1, bc2, rbc1, rbc2;
  float scale, rscale, ntok, rntok;
  int unscale;
};

__device__ __forceinline__ double div_by(double a, double b, double rb) {
  const double q = __dmul_rn(a, rb);
  return __fma_rn(__fma_rn(-b, q, a), rb, q);
}
__device__ __forceinline__ float div_by(float a, float b, float rb) {
  const float q = __fmul_rn(a, rb);
  return __fmaf_rn(__fmaf_rn(-b, q, a), rb, q);
}

// one element: returns the new master value; m, v updated in place
// (optim.cpp:48-66 evaluation order, explicit _rn ops: no contraction)
__device__ __forceinline__ float adam_elem(const AdamConst& c, float p, float& m, float& v, float gf) {
  if (c.unscale) gf = div_by(gf, c.scale, c.rscale);
  gf = div_by(gf, c.ntok, c.rntok);
  const double g = gf;
  const double mm = __dadd_rn(__dmul_rn(c.b1, double(m)), __dmul_rn(1.0 - c.b1, g));
  const double vv = __dadd_rn(__dmul_rn(c.b2, double(v)), __dmul_rn(__dmul_rn(1.0 - c.b2, g), g));
  m = float(mm);
  v = float(vv);
  const double mhat = div_by(double(m), c.bc1, c.rbc1);
  const double vhat = div_by(double(v), c.bc2, c.rbc2);
  return float(__dsub_rn(double(p), __ddiv_rn(__dmul_rn(c.lr, mhat), __dadd_rn(__dsqrt_rn(vhat), c.eps))));
}

template <typename G, typename S>
__global__ void adam_k(float* __restrict__ master, S* __restrict__ shadow, const G* __restrict__ grad,
                       float* __restrict__ m, float* __restrict__ v, int64_t n, const AdamConst c,
                       const int32_t* __restrict__ skip) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  if (skip && *skip) return;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    float mi = m[i], vi = v[i];
    const float p = adam_elem(c, master[i], mi, vi, Num<G>::ld(grad + i));
    m[i] = mi;
    v[i] = vi;
    master[i] = p;
    if (shadow) Num<S>::st(shadow + i, p);
  }
}

// 4 elements per thread per iteration: vector loads of the fp32 state and
// the 16-bit gradient; the per-element arithmetic is adam_k's exactly.
template <typename G, typename S>
__global__ void __launch_bounds__(256) adam4_k(float* __restrict__ master, S* __restrict__ shadow,
                                               const G* __restrict__ grad, float* __restrict__ m,
                                               float* __restrict__ v, int64_t n4, const AdamConst c,
                                               const int32_t* __restrict__ skip) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  if (skip && *skip) return;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < n4; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = 4 * q;
    float4 p4 = *reinterpret_cast<const float4*>(master + i);
    float4 m4 = *reinterpret_cast<const float4*>(m + i);
    float4 v4 = *reinterpret_cast<const float4*>(v + i);
    const uint2 g2 = *reinterpret_cast<const uint2*>(grad + i);
    const G* gg = reinterpret_cast<const G*>(&g2);
    float* pp = &p4.x;
    float* mp = &m4.x;
    float* vp = &v4.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) pp[j] = adam_elem(c, pp[j], mp[j], vp[j], Num<G>::ld(gg + j));
    *reinterpret_cast<float4*>(master + i) = p4;
    *reinterpret_cast<float4*>(m + i) = m4;
    *reinterpret_cast<float4*>(v + i) = v4;
    if (shadow) {
#pragma unroll
      for (int j = 0; j < 4; ++j) Num<S>::st(shadow + i + j, pp[j]);
    }
  }
}

template <typename G, typename S>
__global__ void sgd_k(float* __restrict__ master, S* __restrict__ shadow, const G* __restrict__ grad, int64_t n,
                      double lr, float scale, int unscale, float ntok, const int32_t* __restrict__ skip) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  if (skip && *skip) return;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    float gf = Num<G>::ld(grad + i);
    if (unscale) gf = __fdiv_rn(gf, scale);
    gf = __fdiv_rn(gf, ntok);
    const float p = float(__dsub_rn(double(master[i]), __dmul_rn(lr, double(gf))));
    master[i] = p;
    if (shadow) Num<S>::st(shadow + i, p);
  }
}

template <typename S, typename D>
__global__ void convert_k(const S* __restrict__ src, D* __restrict__ dst, int64_t n) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    Num<D>::st(dst + i, Num<S>::ld(src + i));
}

template <typename T>
__global__ void accumulate_k(T* __restrict__ dst, const T* __restrict__ src, int64_t n) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    Num<T>::st(dst + i, __fadd_rn(Num<T>::ld(dst + i), Num<T>::ld(src + i)));
}

inline int grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  const int cap = 148 * 16;
  return int(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace sfk

using namespace sfk;

extern "C" int sfk_nonfinite(int dtype, const void* g, int64_t n, int32_t* flag, void* stream) {
  if (n == 0) return SFK_OK;
  SFK_DISPATCH(dtype, T,
               launch_pdl(nonfinite_k<T>, grid_for(n), 256, 0, as_stream(stream), static_cast<const T*>(g), n, flag));
  return check_launch("sfk_nonfinite");
}

#define SFK_DISPATCH2(gd, G, sd, S, ...)                    \
  SFK_DISPATCH(gd, G, {                                     \
    switch (sd) {                                           \
      case SFK_F32: { using S = float; __VA_ARGS__; break; } \
      case SFK_F16: { using S = __half; __VA_ARGS__; break; } \
      case SFK_BF16: { using S = __nv_bfloat16; __VA_ARGS__; break; } \
      default: set_error("bad shadow dtype"); return SFK_EINVAL; \
    }                                                       \
  })

extern "C" int sfk_adam(int grad_dtype, float* master, void* shadow, int shadow_dtype, const void* grad, float* m,
                        float* v, int64_t n, double lr, double b1, double b2, double eps, double bc1, double bc2,
                        float scale, int unscale, float ntokens, const int32_t* skip, void* stream) {
  if (n == 0) return SFK_OK;
  const bool vec = grad_dtype != SFK_F32 && n % 4 == 0 && ((reinterpret_cast<uintptr_t>(master) |
                                                             reinterpret_cast<uintptr_t>(m) |
                                                             reinterpret_cast<uintptr_t>(v)) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(grad) & 7) == 0;
  AdamConst c{lr, b1, b2, eps, bc1, bc2, 1.0 / bc1, 1.0 / bc2, scale, 1.0f / scale, ntokens, 1.0f / ntokens,
               unscale};
  if (vec) {
    const int64_t n4 = n / 4;
    SFK_DISPATCH2(grad_dtype, G, shadow_dtype, S,
                  launch_pdl(adam4_k<G, S>, grid_for(n4), 256, 0, as_stream(stream),
                      master, static_cast<S*>(shadow), static_cast<const G*>(grad), m, v, n4, c, skip));
    return check_launch("sfk_adam(vec)");
  }
  SFK_DISPATCH2(grad_dtype, G, shadow_dtype, S,
                launch_pdl(adam_k<G, S>, grid_for(n), 256, 0, as_stream(stream),
                    master, static_cast<S*>(shadow), static_cast<const G*>(grad), m, v, n, c, skip));
  return check_launch("sfk_adam");
}

extern "C" int sfk_sgd(int grad_dtype, float* master, void* shadow, int shadow_dtype, const void* grad, int64_t n,
                       double lr, float scale, int unscale, float ntokens, const int32_t* skip, void* stream) {
  if (n == 0) return SFK_OK;
  SFK_DISPATCH2(grad_dtype, G, shadow_dtype, S,
                launch_pdl(sgd_k<G, S>, grid_for(n), 256, 0, as_stream(stream), master, static_cast<S*>(shadow),
                                                                        static_cast<const G*>(grad), n, lr, scale,
                                                                        unscale, ntokens, skip));
  return check_launch("sfk_sgd");
}

extern "C" int sfk_cast(const float* src, void* dst, int dst_dtype, int64_t n, void* stream) {
  return sfk_convert(SFK_F32, src, dst_dtype, dst, n, stream);
}

extern "C" int sfk_convert(int src_dtype, const void* src, int dst_dtype, void* dst, int64_t n, void* stream) {
  if (n == 0) return SFK_OK;
  SFK_DISPATCH2(src_dtype, S, dst_dtype, D,
                launch_pdl(convert_k<S, D>, grid_for(n), 256, 0, as_stream(stream), static_cast<const S*>(src),
                                                                            static_cast<D*>(dst), n));
  return check_launch("sfk_convert");
}

extern "C" int sfk_accumulate(int dtype, void* dst, const void* src, int64_t n, void* stream) {
  if (n == 0) return SFK_OK;
  SFK_DISPATCH(dtype, T,
               launch_pdl(accumulate_k<T>, grid_for(n), 256, 0, as_stream(stream), static_cast<T*>(dst),
                                                                          static_cast<const T*>(src), n));
  return check_launch("sfk_accumulate");
}

// Dropout (reference Tape::dropout, tape.cpp:109-121 forward 223-228,
// backward 419-425; mask stream model.cpp:156-163) as stateless kernels: the
// mask is re-derived from the counter-based RNG wherever it is needed, never
// stored. Element i of the [rows x cols] node draws
//   u_i = (fmix64(base ^ i) >> 11) * 2^-53,  base = fmix64(fmix64(seed + golden) ^ stream)
// (RngStream::next_u64/next_double, rng.cpp:10-31, counter = i) and keeps the
// value with factor float(1/(1-p)) unless u_i < p. The comparison is done on
// the 53-bit integer against thr = ceil(p * 2^53), which is exact.
#include "common.cuh"

namespace sfk {
namespace {

__device__ __forceinline__ uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}

__device__ __forceinline__ float mask_at(uint64_t base, uint64_t thr, int64_t i, float keep) {
  return (fmix64(base ^ uint64_t(i)) >> 11) < thr ? 0.0f : keep;
}

// out = q(res + q(x * m))  (res == nullptr: out = q(x * m))
template <typename T>
__global__ void __launch_bounds__(256) dropout_fwd_k(const T* __restrict__ x, const T* __restrict__ res,
                                                    T* __restrict__ out, int64_t n, uint64_t base, uint64_t thr,
                                                    float keep) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  using N = Num<T>;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    float v = N::rnd(N::ld(x + i) * mask_at(base, thr, i, keep));
    if (res) v = N::rnd(N::ld(res + i) + v);
    N::st(out + i, v);
  }
}

// dx = q(g * m)  or  dx = q(dx + g * m)
template <typename T>
__global__ void __launch_bounds__(256) dropout_bwd_k(const T* __restrict__ g, T* __restrict__ dx, int64_t n,
                                                    uint64_t base, uint64_t thr, float keep, int accumulate) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  using N = Num<T>;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const float gm = N::ld(g + i) * mask_at(base, thr, i, keep);
    N::st(dx + i, N::rnd(accumulate ? N::ld(dx + i) + gm : gm));
  }
}

uint64_t host_fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}

struct Mask {
  uint64_t base, thr;
  float keep;
};

bool make_mask(float p, uint64_t seed, uint64_t stream, Mask* m) {
  if (!(p >= 0.0f && p < 1.0f)) return false;
  m->base = host_fmix64(host_fmix64(seed + 0x9e3779b97f4a7c15ull) ^ stream);
  m->thr = uint64_t(std::ceil(double(p) * 0x1.0p53));
  m->keep = 1.0f / (1.0f - p);
  return true;
}

int grid_of(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return int(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

}  // namespace
}  // namespace sfk

extern "C" int sfk_dropout_fwd(int dtype, const void* x, const void* res, void* out, int64_t n, float p, uint64_t seed,
                               uint64_t stream_id, void* stream) {
  using namespace sfk;
  if (n == 0) return SFK_OK;
  Mask m;
  if (!make_mask(p, seed, stream_id, &m)) {
    set_error("sfk_dropout_fwd: p must be in [0, 1)");
    return SFK_EINVAL;
  }
  SFK_DISPATCH(dtype, T,
               launch_pdl(dropout_fwd_k<T>, grid_of(n), 256, 0, as_stream(stream), static_cast<const T*>(x),
                          static_cast<const T*>(res), static_cast<T*>(out), n, m.base, m.thr, m.keep));
  return check_launch("sfk_dropout_fwd");
}

extern "C" int sfk_dropout_bwd(int dtype, const void* g, void* dx, int64_t n, float p, uint64_t seed,
                               uint64_t stream_id, int accumulate, void* stream) {
  using namespace sfk;
  if (n == 0) return SFK_OK;
  Mask m;
  if (!make_mask(p, seed, stream_id, &m)) {
    set_error("sfk_dropout_bwd: p must be in [0, 1)");
    return SFK_EINVAL;
  }
  SFK_DISPATCH(dtype, T,
               launch_pdl(dropout_bwd_k<T>, grid_of(n), 256, 0, as_stream(stream), static_cast<const T*>(g),
                          static_cast<T*>(dx), n, m.base, m.thr, m.keep, accumulate));
  return check_launch("sfk_dropout_bwd");
}

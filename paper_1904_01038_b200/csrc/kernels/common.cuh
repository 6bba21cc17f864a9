// Shared device helpers: storage-type traits (rounding to the binary16 /
// bfloat16 grid at every store, as the reference's F16E tape does), warp
// reductions, status plumbing for the C ABI.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../../include/sqf_kernels.h"

namespace sfk {

void set_error(const std::string& msg);

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return SFK_ECUDA;
  }
  return SFK_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

template <typename T>
struct Num;

template <>
struct Num<float> {
  static __device__ __forceinline__ float ld(const float* p) { return *p; }
  static __device__ __forceinline__ void st(float* p, float v) { *p = v; }
  static __device__ __forceinline__ float rnd(float v) { return v; }
};

template <>
struct Num<__half> {
  static __device__ __forceinline__ float ld(const __half* p) { return __half2float(*p); }
  static __device__ __forceinline__ void st(__half* p, float v) { *p = __float2half_rn(v); }
  // IEEE RNE with overflow to inf at >= 65520: identical to quantize_fp16 (fp16.cpp:22-76)
  static __device__ __forceinline__ float rnd(float v) { return __half2float(__float2half_rn(v)); }
};

template <>
struct Num<__nv_bfloat16> {
  static __device__ __forceinline__ float ld(const __nv_bfloat16* p) { return __bfloat162float(*p); }
  static __device__ __forceinline__ void st(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
  static __device__ __forceinline__ float rnd(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }
};

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// dispatch a templated launcher on the runtime dtype
#define SFK_DISPATCH(dtype, T, ...)                       \
  switch (dtype) {                                        \
    case SFK_F32: { using T = float; __VA_ARGS__; break; } \
    case SFK_F16: { using T = __half; __VA_ARGS__; break; } \
    case SFK_BF16: { using T = __nv_bfloat16; __VA_ARGS__; break; } \
    default: set_error("bad dtype"); return SFK_EINVAL;   \
  }

inline int elem_size(int dtype) { return dtype == SFK_F32 ? 4 : 2; }

// Programmatic dependent launch: every kernel is launched with the PDL
// attribute, waits for its stream predecessor's completion (and memory flush)
// before touching global memory, and immediately allows its own successor to
// be scheduled, so launch latency and prologues overlap the predecessor's tail.
#define SFK_PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
#define SFK_PDL_LAUNCH() asm volatile("griddepcontrol.launch_dependents;" ::: "memory")

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace sfk

// GEMM family implementation (templates), included by gemm.cu and by the
// per-dtype translation units gemm_f16.cu / gemm_bf16.cu, which instantiate
// the tensor-core kernels in parallel builds.
//
// GEMM family for Tape::matmul_nt forward / dgrad / wgrad (reference
// tape.cpp:182-189, 324-346; kernels.cpp:9-16) with the fused epilogues of
// add_bias / relu / residual add / relu-backward / gradient accumulation.
//
// fp16/bf16: a persistent warp-specialised tcgen05 kernel for sm_100a.
//   warp 0      TMA producer: A/B tiles -> 128B-swizzled smem ring (mbarriers)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN,
//               K=16 per instruction, fp32 accumulators in TMEM, 2 buffers)
//   warps 2..5  epilogue: tcgen05.ld -> registers -> fused epilogue -> global
// Operand majors are handled by the UMMA descriptors (K-major or MN-major
// canonical SW128 layouts), so dgrad and wgrad read activations in place with
// no transposes.
// fp32: a SIMT kernel (true fp32 FMA, no TF32) for the reference's fp32 mode.
#pragma once
#include <cuda.h>

#include <cmath>
#include <mutex>

#include "common.cuh"

namespace sfk {

// ------------------------------------------------------------------ epilogue
struct Epi {
  void* c;
  int64_t ldc;
  const void* bias;
  const void* res;
  int64_t ldr;
  const void* mask;
  int64_t ldm;
  int flags;
  int raster;  // tile order: 0 = row blocks fastest, 1 = column blocks fastest
};

// Output tile `tile` of a num_m x num_n grid. With few column blocks
// (raster 1) the column tiles of one row block are consecutive, so the
// persistent CTAs that share an A row panel run at the same time and read
// it from DRAM once (the tall activation / gradient operands of the
// N = 1024 GEMMs); otherwise row blocks run fastest.
__device__ __forceinline__ void tile_coords(int tile, int num_m, int num_n, int raster, int& mi, int& ni) {
  if (raster) {
    mi = tile / num_n;
    ni = tile % num_n;
  } else {
    mi = tile % num_m;
    ni = tile / num_m;
  }
}

template <typename T>
__device__ __forceinline__ float epi_value(const Epi& e, int64_t row, int col, float acc) {
  using N = Num<T>;
  float v = acc;
  if (e.flags & SFK_EPI_ACCUM) {
    // gradient accumulation: q(old + acc), one rounding (tape.cpp:296-299)
    return N::rnd(N::ld(static_cast<const T*>(e.c) + row * e.ldc + col) + v);
  }
  if (e.flags & SFK_EPI_PREROUND) v = N::rnd(v);
  if (e.flags & SFK_EPI_BIAS) v = N::rnd(v + N::ld(static_cast<const T*>(e.bias) + col));
  if (e.flags & SFK_EPI_RELU) v = v > 0.0f ? v : 0.0f;
  if (e.flags & SFK_EPI_MASK) v = N::ld(static_cast<const T*>(e.mask) + row * e.ldm + col) > 0.0f ? N::rnd(v) : 0.0f;
  if (e.flags & SFK_EPI_RESIDUAL) v = N::rnd(N::ld(static_cast<const T*>(e.res) + row * e.ldr + col) + v);
  return v;
}

// ------------------------------------------------------------------ SIMT fp32
namespace simt {
constexpr int TM = 64, TN = 64, TK = 16;

template <typename T>
__global__ void __launch_bounds__(256) gemm_simt(const T* __restrict__ a, int64_t sa_i, int64_t sa_k,
                                                 const T* __restrict__ b, int64_t sb_j, int64_t sb_k,
                                                 Epi e, int M, int N, int K) {
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += TK) {
    for (int i = tid; i < TM * TK; i += 256) {
      const int mi = i / TK, ki = i % TK;
      const int gm = m0 + mi, gk = k0 + ki;
      As[ki][mi] = (gm < M && gk < K) ? Num<T>::ld(a + gm * sa_i + gk * sa_k) : 0.0f;
      const int gn = n0 + mi;
      Bs[ki][mi] = (gn < N && gk < K) ? Num<T>::ld(b + gn * sb_j + gk * sb_k) : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) av[r] = As[kk][ty * 4 + r];
#pragma unroll
      for (int c = 0; c < 4; ++c) bv[c] = Bs[kk][tx * 4 + c];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = fmaf(av[r], bv[c], acc[r][c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int gm = m0 + ty * 4 + r;
    if (gm >= M) continue;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int gn = n0 + tx * 4 + c;
      if (gn >= N) continue;
      const float v = epi_value<T>(e, gm, gn, acc[r][c]);
      Num<T>::st(static_cast<T*>(e.c) + int64_t(gm) * e.ldc + gn, v);
    }
  }
}
}  // namespace simt

// ------------------------------------------------------------------ tcgen05
namespace tc {
constexpr int BM = 128, BK = 64;

// Debug timeline of one pair-GEMM launch (SFK_GEMM_TRACE builds only):
// %globaltimer (ns) at fixed points of CTA 0 and of the last CTA.
#ifdef SFK_GEMM_TRACE
__device__ unsigned long long g_trace[2][24];
__device__ __forceinline__ void trace(int slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (blockIdx.x == 0) g_trace[0][slot] = t;
  if (blockIdx.x == gridDim.x - 1) g_trace[1][slot] = t;
}
#else
__device__ __forceinline__ void trace(int) {}
#endif
constexpr int kEpiWarps = 8, kThreads = 64 + 32 * kEpiWarps;  // producer, MMA, 8 epilogue warps

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t}" ::"r"(saddr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(saddr(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor, SWIZZLE_128B, sm_100 version bits
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version (Blackwell)
  d |= static_cast<uint64_t>(2) << 61;  // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(bar))
               : "memory");
}

// tcgen05.ld issue and wait are separate so the next chunk's TMEM read
// overlaps this chunk's global epilogue; the wait names the destination
// registers as read-write so the compiler cannot consume them before it.
__device__ __forceinline__ void tmem_ld32_issue(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait(uint32_t (&r)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}

template <typename T>
struct Pack;
template <>
struct Pack<__half> {
  static __device__ __forceinline__ uint32_t two(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  static __device__ __forceinline__ float2 unpack(uint32_t u) {
    __half2 h = *reinterpret_cast<__half2*>(&u);
    return __half22float2(h);
  }
};
template <>
struct Pack<__nv_bfloat16> {
  static __device__ __forceinline__ uint32_t two(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  static __device__ __forceinline__ float2 unpack(uint32_t u) {
    __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&u);
    return __bfloat1622float2(h);
  }
};

// 32 consecutive accumulators of one row -> fused epilogue -> global
template <typename T>
__device__ __forceinline__ void epilogue_row32(const Epi& e, int64_t row, int col0, int N, const uint32_t (&r)[32],
                                               bool vec_ok) {
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
  T* out = static_cast<T*>(e.c) + row * e.ldc + col0;
  if (vec_ok && col0 + 32 <= N) {
    // all side inputs share the 16B alignment checked on the host
    if (e.flags == SFK_EPI_ACCUM) {
      uint4* po = reinterpret_cast<uint4*>(out);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 old = po[q];
        uint32_t w[4] = {old.x, old.y, old.z, old.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float2 o = Pack<T>::unpack(w[j]);
          w[j] = Pack<T>::two(o.x + v[q * 8 + 2 * j], o.y + v[q * 8 + 2 * j + 1]);
        }
        po[q] = make_uint4(w[0], w[1], w[2], w[3]);
      }
      return;
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = epi_value<T>(e, row, col0 + i, v[i]);
    uint4* po = reinterpret_cast<uint4*>(out);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      po[q] = make_uint4(Pack<T>::two(v[q * 8 + 0], v[q * 8 + 1]), Pack<T>::two(v[q * 8 + 2], v[q * 8 + 3]),
                         Pack<T>::two(v[q * 8 + 4], v[q * 8 + 5]), Pack<T>::two(v[q * 8 + 6], v[q * 8 + 7]));
    }
    return;
  }
  for (int i = 0; i < 32 && col0 + i < N; ++i) Num<T>::st(out + i, epi_value<T>(e, row, col0 + i, v[i]));
}

// 8 consecutive accumulators of one row (coalesced layout) -> fused epilogue -> global
template <typename T>
__device__ __forceinline__ void epilogue8(const Epi& e, int64_t row, int col, int N, float (&v)[8], bool vec_ok) {
  T* out = static_cast<T*>(e.c) + row * e.ldc + col;
  if (!vec_ok || col + 8 > N) {
    for (int i = 0; i < 8 && col + i < N; ++i) Num<T>::st(out + i, epi_value<T>(e, row, col + i, v[i]));
    return;
  }
  auto ld8 = [](const T* p, float (&f)[8]) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 t = Pack<T>::unpack(w[j]);
      f[2 * j] = t.x;
      f[2 * j + 1] = t.y;
    }
  };
  const int fl = e.flags;
  if (fl & SFK_EPI_ACCUM) {
    float o[8];
    ld8(out, o);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = o[j] + v[j];
  } else {
    if (fl & SFK_EPI_PREROUND)
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = Num<T>::rnd(v[j]);
    if (fl & SFK_EPI_BIAS) {
      float b[8];
      ld8(static_cast<const T*>(e.bias) + col, b);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = Num<T>::rnd(v[j] + b[j]);
    }
    if (fl & SFK_EPI_RELU)
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = v[j] > 0.0f ? v[j] : 0.0f;
    if (fl & SFK_EPI_MASK) {
      float mk[8];
      ld8(static_cast<const T*>(e.mask) + row * e.ldm + col, mk);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = mk[j] > 0.0f ? Num<T>::rnd(v[j]) : 0.0f;
    }
    if (fl & SFK_EPI_RESIDUAL) {
      float rs[8];
      ld8(static_cast<const T*>(e.res) + row * e.ldr + col, rs);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = Num<T>::rnd(rs[j] + v[j]);
    }
  }
  *reinterpret_cast<uint4*>(out) = make_uint4(Pack<T>::two(v[0], v[1]), Pack<T>::two(v[2], v[3]),
                                              Pack<T>::two(v[4], v[5]), Pack<T>::two(v[6], v[7]));
}

// Per-warp staging of a 32 x 32 fp32 block: row stride 32 floats, the eight
// 16-byte chunks of row r stored at chunk index (j ^ (r & 7)) -- conflict-free
// float4 writes (one row per lane) and reads (8 rows x 64 B per instruction).
constexpr int kStgFloats = 32 * 32;
__device__ __forceinline__ int stg_off(int row, int j) { return row * 32 + ((j ^ (row & 7)) << 2); }

// Four row segments (rows row0 + 8i, i<4) x 8 columns, all loads of side
// inputs issued before any math so their latencies overlap.
template <typename T>
__device__ __forceinline__ void epilogue_seg4(const Epi& e, int64_t row0, int col, int M, const float* stg, int rr0,
                                              int j0) {
  const int fl = e.flags;
  float v[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float4 a = *reinterpret_cast<const float4*>(stg + stg_off(rr0 + 8 * i, j0));
    const float4 b = *reinterpret_cast<const float4*>(stg + stg_off(rr0 + 8 * i, j0 + 1));
    v[i][0] = a.x, v[i][1] = a.y, v[i][2] = a.z, v[i][3] = a.w, v[i][4] = b.x, v[i][5] = b.y, v[i][6] = b.z,
    v[i][7] = b.w;
  }
  const uint4 z = make_uint4(0, 0, 0, 0);
  uint4 side[4] = {z, z, z, z}, side2[4] = {z, z, z, z}, bias = z;
  T* out = static_cast<T*>(e.c);
  if (fl & SFK_EPI_BIAS) bias = *reinterpret_cast<const uint4*>(static_cast<const T*>(e.bias) + col);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = row0 + 8 * i;
    if (row >= M) continue;
    if (fl & SFK_EPI_ACCUM) side[i] = *reinterpret_cast<const uint4*>(out + row * e.ldc + col);
    if (fl & SFK_EPI_RESIDUAL)
      side[i] = *reinterpret_cast<const uint4*>(static_cast<const T*>(e.res) + row * e.ldr + col);
    if (fl & SFK_EPI_MASK)
      side2[i] = *reinterpret_cast<const uint4*>(static_cast<const T*>(e.mask) + row * e.ldm + col);
  }
  auto unpack = [](const uint4& u, float (&f)[8]) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 t = Pack<T>::unpack(w[j]);
      f[2 * j] = t.x;
      f[2 * j + 1] = t.y;
    }
  };
  float bf[8];
  unpack(bias, bf);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = row0 + 8 * i;
    if (row >= M) continue;
    float s1[8], s2[8];
    unpack(side[i], s1);
    unpack(side2[i], s2);
    float* x = v[i];
    if (fl & SFK_EPI_ACCUM) {
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = s1[j] + x[j];
    } else {
      if (fl & SFK_EPI_PREROUND)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = Num<T>::rnd(x[j]);
      if (fl & SFK_EPI_BIAS)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = Num<T>::rnd(x[j] + bf[j]);
      if (fl & SFK_EPI_RELU)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = x[j] > 0.0f ? x[j] : 0.0f;
      if (fl & SFK_EPI_MASK)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = s2[j] > 0.0f ? Num<T>::rnd(x[j]) : 0.0f;
      if (fl & SFK_EPI_RESIDUAL)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = Num<T>::rnd(s1[j] + x[j]);
    }
    *reinterpret_cast<uint4*>(out + row * e.ldc + col) =
        make_uint4(Pack<T>::two(x[0], x[1]), Pack<T>::two(x[2], x[3]), Pack<T>::two(x[4], x[5]),
                   Pack<T>::two(x[6], x[7]));
  }
}

// Drain one BM x BN accumulator tile from TMEM through the fused epilogue.
// Eight epilogue warps: warp w may only touch TMEM lanes 32*(w%4)..+31, so two
// warps share each lane quarter and take alternate 32-column chunks. The TMEM
// read of a warp's next chunk is in flight while it runs the current chunk's
// global loads/stores.
template <int BN, typename T>
__device__ __forceinline__ void epilogue_tile(const Epi& e, uint32_t tacc, int warp, int lane, float* stg, int64_t m0,
                                              int n0, int M, int N, int vec_ok) {
  const int quarter = warp & 3, half = (warp - 2) >> 2;
  const uint32_t lane_base = tacc + (uint32_t(quarter * 32) << 16);
  int nch = (N - n0 + 31) / 32;
  if (nch > BN / 32) nch = BN / 32;
  uint32_t r[32];
  if (half < nch) tmem_ld32_issue(lane_base + half * 32, r);
#pragma unroll 1
  for (int ch = half; ch < nch; ch += 2) {
    tmem_ld_wait(r);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      *reinterpret_cast<float4*>(stg + stg_off(lane, j)) =
          make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]), __uint_as_float(r[4 * j + 2]),
                      __uint_as_float(r[4 * j + 3]));
    if (ch + 2 < nch) tmem_ld32_issue(lane_base + (ch + 2) * 32, r);
    __syncwarp();
    const int cc = (lane & 3) * 8, col = n0 + ch * 32 + cc;
    const int rr0 = lane >> 2;
    const int64_t row0 = m0 + quarter * 32 + rr0;
    if (vec_ok && col + 8 <= N) {
      epilogue_seg4<T>(e, row0, col, M, stg, rr0, cc >> 2);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int rr = rr0 + 8 * i;
        const int64_t row = row0 + 8 * i;
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = stg[stg_off(rr, (cc + j) >> 2) + ((cc + j) & 3)];
        if (row < M && col < N) epilogue8<T>(e, row, col, N, v, false);
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------- epilogue with TMA stores
// Each thread owns one accumulator row (its TMEM lane): it loads that row's
// side inputs for a 32-column chunk directly (bias is a warp-wide broadcast),
// applies the fused epilogue, packs to 16 bits and writes the 64-byte row
// segment into the warp's 128B-swizzled 32 x 64 staging tile; one lane then
// stores the whole tile with a TMA bulk store (out-of-range rows/columns are
// clipped by the tensor map). No per-element global stores, no transpose
// through shared memory. FL >= 0: the epilogue flags are compile-time.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 8 16-bit values at p[col..col+8) of a row, bounds-checked against n (rare slow path at the right edge)
template <typename T>
__device__ __forceinline__ uint4 ld_row8(const T* p, int col, int n, bool ok) {
  if (!ok) return make_uint4(0, 0, 0, 0);
  if (col + 8 <= n) return *reinterpret_cast<const uint4*>(p + col);
  uint16_t h[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int j = 0; j < 8 && col + j < n; ++j) h[j] = reinterpret_cast<const uint16_t*>(p)[col + j];
  return make_uint4(h[0] | (uint32_t(h[1]) << 16), h[2] | (uint32_t(h[3]) << 16), h[4] | (uint32_t(h[5]) << 16),
                    h[6] | (uint32_t(h[7]) << 16));
}

template <int FL, typename T>
__device__ __forceinline__ uint4 epi_pack8(const Epi& e, const uint32_t* acc, const uint4& side, const uint4& side2,
                                           const uint4& bias) {
  const int fl = FL >= 0 ? FL : e.flags;
  float x[8], s1[8], s2[8], bf[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = __uint_as_float(acc[j]);
  auto unpack = [](const uint4& u, float (&f)[8]) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 t = Pack<T>::unpack(w[j]);
      f[2 * j] = t.x;
      f[2 * j + 1] = t.y;
    }
  };
  if (fl & SFK_EPI_ACCUM) {
    unpack(side, s1);
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = s1[j] + x[j];
  } else {
    if (fl & SFK_EPI_PREROUND)
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = Num<T>::rnd(x[j]);
    if (fl & SFK_EPI_BIAS) {
      unpack(bias, bf);
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = Num<T>::rnd(x[j] + bf[j]);
    }
    if (fl & SFK_EPI_RELU)
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = x[j] > 0.0f ? x[j] : 0.0f;
    if (fl & SFK_EPI_MASK) {
      unpack(side2, s2);
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = s2[j] > 0.0f ? Num<T>::rnd(x[j]) : 0.0f;
    }
    if (fl & SFK_EPI_RESIDUAL) {
      unpack(side, s1);
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = Num<T>::rnd(s1[j] + x[j]);
    }
  }
  return make_uint4(Pack<T>::two(x[0], x[1]), Pack<T>::two(x[2], x[3]), Pack<T>::two(x[4], x[5]),
                    Pack<T>::two(x[6], x[7]));
}

// Stream-K fix-up source for epilogue_tile_tma: the tile's fp32 partial
// accumulators, [128 rows][BN] per contributing unit, summed in unit order.
struct WsSum {
  const float* slot[8];
  int n = 0;  // 0: read the accumulators from TMEM instead
};

// stage: this warp's 4 KB staging tile (1024-aligned, shared::cta address)
template <int BN, int FL, typename T>
__device__ __forceinline__ void epilogue_tile_tma(const Epi& e, const CUtensorMap* cmap, uint32_t tacc, int warp,
                                                  int lane, uint32_t stage, int64_t m0, int n0, int M, int N,
                                                  const WsSum& ws = WsSum{}) {
  const int quarter = warp & 3, half = (warp - 2) >> 2;
  const int fl = FL >= 0 ? FL : e.flags;
  const uint32_t lane_base = tacc + (uint32_t(quarter * 32) << 16);
  const int64_t row = m0 + quarter * 32 + lane;
  const bool rok = row < M;
  const T* side_row = nullptr;
  if (fl & SFK_EPI_ACCUM) side_row = static_cast<const T*>(e.c) + row * e.ldc;
  else if (fl & SFK_EPI_RESIDUAL) side_row = static_cast<const T*>(e.res) + row * e.ldr;
  const T* mask_row = (fl & SFK_EPI_MASK) && !(fl & SFK_EPI_ACCUM) ? static_cast<const T*>(e.mask) + row * e.ldm
                                                                    : nullptr;
  const T* bias = (fl & SFK_EPI_BIAS) && !(fl & SFK_EPI_ACCUM) ? static_cast<const T*>(e.bias) : nullptr;
  int nblk = (N - n0 + 63) / 64;
  if (nblk > BN / 64) nblk = BN / 64;
  const uint32_t my_row = stage + uint32_t(lane) * 128u;
  uint32_t r[32];
  const bool from_ws = ws.n > 0;
  if (half < nblk && !from_ws) tmem_ld32_issue(lane_base + half * 64, r);
#pragma unroll 1
  for (int b = half; b < nblk; b += 2) {
#pragma unroll 1
    for (int sub = 0; sub < 2; ++sub) {
      const int col0 = n0 + b * 64 + sub * 32;
      uint32_t v[32];
      if (from_ws) {
        // this thread's row of every partial, summed in unit order; partials
        // are stored [chunk][float4 j][row] so each warp load is 512
        // contiguous bytes (see store_partial_rows)
        const int ch = b * 2 + sub, row = quarter * 32 + lane;
        float acc[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = 0.f;
        float4 x[8];
        {
          const float4* src = reinterpret_cast<const float4*>(ws.slot[0]) + size_t(ch) * 8 * 128 + row;
#pragma unroll
          for (int q = 0; q < 8; ++q) x[q] = __ldcg(src + q * 128);
        }
        for (int u = 0; u < ws.n; ++u) {
          float4 y[8];
          if (u + 1 < ws.n) {  // next part's loads in flight while this one is added
            const float4* src = reinterpret_cast<const float4*>(ws.slot[u + 1]) + size_t(ch) * 8 * 128 + row;
#pragma unroll
            for (int q = 0; q < 8; ++q) y[q] = __ldcg(src + q * 128);
          }
#pragma unroll
          for (int q = 0; q < 8; ++q)
            acc[4 * q] += x[q].x, acc[4 * q + 1] += x[q].y, acc[4 * q + 2] += x[q].z, acc[4 * q + 3] += x[q].w;
          if (u + 1 < ws.n)
#pragma unroll
            for (int q = 0; q < 8; ++q) x[q] = y[q];
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(acc[j]);
      } else {
        tmem_ld_wait(r);
        if (warp == 2 && lane == 0 && b * 2 + sub < 8) trace(10 + b * 2 + sub);  // chunk's TMEM data in registers
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = r[j];
        // next TMEM chunk in flight while this one runs its epilogue
        if (sub == 0) tmem_ld32_issue(lane_base + b * 64 + 32, r);
        else if (b + 2 < nblk) tmem_ld32_issue(lane_base + (b + 2) * 64, r);
      }
      uint4 sd[4], sd2[4], bs[4];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        sd[g] = side_row ? ld_row8(side_row, col0 + 8 * g, N, rok) : make_uint4(0, 0, 0, 0);
        sd2[g] = mask_row ? ld_row8(mask_row, col0 + 8 * g, N, rok) : make_uint4(0, 0, 0, 0);
        bs[g] = bias ? ld_row8(bias, col0 + 8 * g, N, true) : make_uint4(0, 0, 0, 0);
      }
      if (sub == 0 && b > half) {
        // the previous tile's bulk store must have read the staging tile
        if (lane == 0) bulk_wait_read0();
        __syncwarp();
      }
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const uint4 o = epi_pack8<FL, T>(e, v + 8 * g, sd[g], sd2[g], bs[g]);
        const uint32_t chunk = uint32_t((sub * 4 + g) ^ (lane & 7));
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(my_row + chunk * 16u), "r"(o.x), "r"(o.y),
                     "r"(o.z), "r"(o.w)
                     : "memory");
      }
    }
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(cmap, stage, n0 + b * 64, int(m0) + quarter * 32);
      bulk_commit();
    }
    if (warp == 2 && lane == 0 && b < 4) trace(18 + b);  // block's bulk store issued
  }
  if (lane == 0) bulk_wait_read0();
  __syncwarp();
}

// ---------------------------------------------------------- stream-K schedule
// Pair stream-K partial: this CTA's 128 x BN fp32 accumulators (TMEM) to a
// workspace slot, row-major; each thread writes its own row's chunks.
// Layout [chunk of 32 columns][float4 j][row]: for a fixed (chunk, j) the 32
// lanes (rows) write 512 contiguous bytes.
template <int BN>
__device__ __forceinline__ void store_partial_rows(uint32_t tacc, int warp, int lane, float* slot) {
  const int quarter = warp & 3, half = (warp - 2) >> 2;
  const uint32_t lane_base = tacc + (uint32_t(quarter * 32) << 16);
  float4* rowp = reinterpret_cast<float4*>(slot) + quarter * 32 + lane;
  uint32_t r[32];
  tmem_ld32_issue(lane_base + half * 32, r);
#pragma unroll 1
  for (int ch = half; ch < BN / 32; ch += 2) {
    tmem_ld_wait(r);
    float4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      v[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]), __uint_as_float(r[4 * j + 2]),
                         __uint_as_float(r[4 * j + 3]));
    if (ch + 2 < BN / 32) tmem_ld32_issue(lane_base + (ch + 2) * 32, r);
#pragma unroll
    for (int j = 0; j < 8; ++j) __stcg(rowp + (size_t(ch) * 8 + j) * 128, v[j]);
  }
}


// Work of a persistent CTA b (of G): first its share of the stream-K region
// -- tiles [0, sk_tiles) flattened to sk_tiles*kblocks k-block iterations and
// cut into G equal contiguous ranges, so a range may start/end inside a tile --
// then whole data-parallel tiles sk_tiles + b + i*G. Producer, MMA and
// epilogue warps walk the identical unit sequence.
struct Sk {
  float* ws;          // [G][2][BM*BN] fp32 partial tiles (slot 0: a CTA's first unit, 1: its last)
  int32_t* flags;     // [sk_tiles] arrival counters, zero on entry, re-armed by the reducer
  int sk_tiles;
  void* bias_grad;    // weight-gradient GEMMs (A = dY, MN-major): db[m] = q(db[m] + sum_k A(m,k)), or null
};

struct Sched {
  int tiles, kblocks, G, b, sk_tiles;
  int64_t tsk, it0, it1, it;
  int dp;
  __device__ __forceinline__ Sched(int tiles_, int kblocks_, int sk_tiles_)
      : Sched(tiles_, kblocks_, sk_tiles_, int(gridDim.x), int(blockIdx.x)) {}
  __device__ __forceinline__ Sched(int tiles_, int kblocks_, int sk_tiles_, int G_, int b_)
      : tiles(tiles_), kblocks(kblocks_), G(G_), b(b_), sk_tiles(sk_tiles_) {
    tsk = int64_t(sk_tiles) * kblocks;
    it0 = int64_t(b) * tsk / G;
    it1 = int64_t(b + 1) * tsk / G;
    it = it0;
    dp = sk_tiles + b;
  }
  __device__ __forceinline__ int64_t start_of(int c) const { return int64_t(c) * tsk / G; }
  __device__ __forceinline__ bool next(int& tile, int& kb0, int& kb1) {
    if (it < it1) {
      tile = int(it / kblocks);
      kb0 = int(it % kblocks);
      kb1 = int(min(int64_t(kblocks), kb0 + (it1 - it)));
      it += kb1 - kb0;
      return true;
    }
    if (dp < tiles) {
      tile = dp;
      kb0 = 0;
      kb1 = kblocks;
      dp += G;
      return true;
    }
    return false;
  }
};

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory"); }

// Partial (stream-K) unit: this warp's chunks of the fp32 accumulator tile go
// to the CTA's workspace slot, one 128-byte row segment per thread.
template <int BN>
__device__ __forceinline__ void store_partial(uint32_t tacc, int warp, int lane, float* slot) {
  const int quarter = warp & 3, half = (warp - 2) >> 2;
  const uint32_t lane_base = tacc + (uint32_t(quarter * 32) << 16);
  float* row = slot + size_t(quarter * 32 + lane) * BN;
  uint32_t r[32];
  tmem_ld32_issue(lane_base + half * 32, r);
#pragma unroll 1
  for (int ch = half; ch < BN / 32; ch += 2) {
    tmem_ld_wait(r);
    float4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      v[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]), __uint_as_float(r[4 * j + 2]),
                         __uint_as_float(r[4 * j + 3]));
    if (ch + 2 < BN / 32) tmem_ld32_issue(lane_base + (ch + 2) * 32, r);
#pragma unroll
    for (int j = 0; j < 8; ++j) __stcg(reinterpret_cast<float4*>(row + ch * 32) + j, v[j]);
  }
}

// Reducer of a stream-K tile: sum the partial slots of its CTAs in k order
// (fixed association: deterministic) and run the fused epilogue on the sum.
template <int BN, typename T>
__device__ __forceinline__ void reduce_partials(const Epi& e, const Sched& sc, const Sk& sk, int tile, int warp,
                                                int lane, float* stg, int64_t m0, int n0, int M, int N, int vec_ok) {
  const int quarter = warp & 3, half = (warp - 2) >> 2;
  const int64_t i_beg = int64_t(tile) * sc.kblocks, i_end = i_beg + sc.kblocks;
  const int c0 = int(((i_beg + 1) * sc.G + sc.tsk - 1) / sc.tsk) - 1;
  const size_t row_off = size_t(quarter * 32 + lane) * BN;
  int nch = (N - n0 + 31) / 32;
  if (nch > BN / 32) nch = BN / 32;
#pragma unroll 1
  for (int ch = half; ch < nch; ch += 2) {
    float4 acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c = c0; c < sc.G && sc.start_of(c) < i_end; ++c) {
      const int slot = i_beg <= sc.start_of(c) ? 0 : 1;
      const float4* src = reinterpret_cast<const float4*>(sk.ws + (size_t(c) * 2 + slot) * (BM * BN) + row_off + ch * 32);
      float4 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __ldcg(src + j);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        acc[j].x += v[j].x;
        acc[j].y += v[j].y;
        acc[j].z += v[j].z;
        acc[j].w += v[j].w;
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) *reinterpret_cast<float4*>(stg + stg_off(lane, j)) = acc[j];
    __syncwarp();
    const int cc = (lane & 3) * 8, col = n0 + ch * 32 + cc;
    const int rr0 = lane >> 2;
    const int64_t row0 = m0 + quarter * 32 + rr0;
    if (vec_ok && col + 8 <= N) {
      epilogue_seg4<T>(e, row0, col, M, stg, rr0, cc >> 2);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int rr = rr0 + 8 * i;
        const int64_t row = row0 + 8 * i;
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = stg[stg_off(rr, (cc + j) >> 2) + ((cc + j) & 3)];
        if (row < M && col < N) epilogue8<T>(e, row, col, N, v, false);
      }
    }
    __syncwarp();
  }
}

// Bias gradient fused into the weight-gradient GEMM (add_bias backward,
// tape.cpp:347-358): while the tensor pipe consumes a k-block of A = dY
// (MN-major, two 64 m x 64 k SW128 boxes per stage), the otherwise idle
// epilogue warps sum its columns out of shared memory: thread t owns the
// m pair 2*(t%64), 2*(t%64)+1 (one 32-bit word per swizzled row) and k rows
// 16*(t/64) .. +15. The four k-quarter sums meet in shared memory in a fixed
// order; db[m] = q(db[m] + sum). Only the tiles with n0 == 0 do this, so every
// db element has exactly one writer.
template <typename T, int STAGES, int STAGE>
__device__ __forceinline__ void bias_grad_tile(uint8_t* smem, uint64_t* ready, uint64_t* bsum, int it0, int nkb,
                                               int warp, int lane, float* stg, T* db, int m0, int M) {
  const int t = (warp - 2) * 32 + lane;
  const int mp = t & 63, kq = t >> 6;
  const int ml = 2 * mp, box = ml >> 6, ch = (ml & 63) >> 3, el = ml & 7;
  float s0 = 0.f, s1 = 0.f;
  for (int i = 0; i < nkb; ++i) {
    const int it = it0 + i, s = it % STAGES;
    mbar_wait(&ready[s], (it / STAGES) & 1);  // the stage's A tile is in smem (and not yet refilled)
    const uint8_t* a = smem + s * STAGE + box * 8192;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int k = kq * 16 + j;
      const uint32_t w = *reinterpret_cast<const uint32_t*>(a + k * 128 + ((ch ^ (k & 7)) << 4) + el * 2);
      const float2 f = Pack<T>::unpack(w);
      s0 += f.x;
      s1 += f.y;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&bsum[s]);
  }
  // combine the k quarters in order through the (idle) staging area
  float* red = stg - (warp - 2) * kStgFloats;  // base of all epilogue staging
  epi_bar();
  red[kq * 128 + ml] = s0;
  red[kq * 128 + ml + 1] = s1;
  epi_bar();
  if (t < 128 && m0 + t < M) {
    const float sum = ((red[t] + red[128 + t]) + red[256 + t]) + red[384 + t];
    Num<T>::st(db + m0 + t, Num<T>::ld(db + m0 + t) + sum);
  }
  epi_bar();
}

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = (192 * 1024) / STAGE;
  static constexpr int SMEM = STAGES * STAGE + 1024 /*align slack*/ + 256 /*barriers*/ + kEpiWarps * kStgFloats * 4;
  static constexpr int TMEM_COLS = 2 * BN;
};

// FL / tma_store as in gemm_tc2: whole tiles leave through the TMA-store
// epilogue (compile-time flags where FL >= 0); stream-K parts keep the
// per-thread epilogue of their fix-up
template <int BN, bool A_MN, bool B_MN, int FL, typename T>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
            const __grid_constant__ CUtensorMap tcm, const Epi e, int M, int N, int K, int vec_ok, int tma_store,
            const Sk sk) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // [stages][epilogue staging: 8 warps x 4 KB, 1024-aligned][barriers]
  uint8_t* stg_region = smem + C::STAGES * C::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(stg_region + kEpiWarps * kStgFloats * 4);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* bsum = tempty + 2;  // per stage: the epilogue warps finished their bias-gradient read
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bsum + C::STAGES);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 32) {  // pull both TMA descriptors in while the prologue runs
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&bsum[s], kEpiWarps);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // everything above overlapped the previous kernel's tail (PDL)
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();

  const int num_m = (M + BM - 1) / BM, num_n = (N + BN - 1) / BN;
  const int tiles = num_m * num_n, kblocks = (K + BK - 1) / BK;
  (void)num_n;

  if (warp == 0) {
    if (lane == 0) {
      Sched sc(tiles, kblocks, sk.sk_tiles);
      int it = 0, tile, kb0, kb1;
      uint32_t bias_pend = 0, bias_ph = 0;  // per stage: a bias-tile read outstanding / its bsum phase
      while (sc.next(tile, kb0, kb1)) {
        int mi, ni;
        tile_coords(tile, num_m, num_n, e.raster, mi, ni);
        const int m0 = mi * BM, n0 = ni * BN;
        const bool btile = A_MN && sk.bias_grad && n0 == 0;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % C::STAGES;
          const uint32_t ph = (it / C::STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          if (bias_pend >> s & 1) {
            mbar_wait(&bsum[s], bias_ph >> s & 1);
            bias_ph ^= 1u << s;
            bias_pend &= ~(1u << s);
          }
          if (btile) bias_pend |= 1u << s;
          mbar_expect_tx(&full[s], C::STAGE);
          uint8_t* a_dst = smem + s * C::STAGE;
          uint8_t* b_dst = a_dst + C::A_BYTES;
          const int k0 = kb * BK;
          if (!A_MN) {
            tma_load_2d(&ta, &full[s], a_dst, k0, m0);
          } else {
            tma_load_2d(&ta, &full[s], a_dst, m0, k0);
            tma_load_2d(&ta, &full[s], a_dst + 8192, m0 + 64, k0);
          }
          if (!B_MN) {
            tma_load_2d(&tb, &full[s], b_dst, k0, n0);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) tma_load_2d(&tb, &full[s], b_dst + j * 8192, n0 + 64 * j, k0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // instruction descriptor: D=f32, A/B = f16|bf16, majors, N>>3, M>>4
      const uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
      const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (uint32_t(A_MN) << 15) |
                             (uint32_t(B_MN) << 16) | (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
      Sched sc(tiles, kblocks, sk.sk_tiles);
      int it = 0, t = 0, tile, kb0, kb1;
      while (sc.next(tile, kb0, kb1)) {
        const int buf = t & 1;
        mbar_wait(&tempty[buf], ((t >> 1) & 1) ^ 1);
        fence_after();
        const uint32_t d_tmem = tmem_base + buf * BN;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % C::STAGES;
          mbar_wait(&full[s], (it / C::STAGES) & 1);
          fence_after();
          const uint32_t a_addr = saddr(smem + s * C::STAGE);
          const uint32_t b_addr = a_addr + C::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major: advance 32 B inside the swizzled 128 B row; MN-major:
            // advance 16 K-rows (2 KB) to the next pair of 8-row groups
            const uint64_t ad = A_MN ? smem_desc(a_addr + k * 2048, 8192, 1024) : smem_desc(a_addr + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? smem_desc(b_addr + k * 2048, 8192, 1024) : smem_desc(b_addr + k * 32, 16, 1024);
            umma(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[buf]);
        ++t;
      }
    }
  } else {
    // Epilogue: TMEM gives each thread one row x 32 columns; the 32x32 fp32
    // block bounces through shared memory so a warp then reads/writes 8 rows x
    // 64 contiguous bytes per instruction (coalesced) instead of 32 rows.
    float* stg = reinterpret_cast<float*>(stg_region) + (warp - 2) * kStgFloats;
    volatile int* last_flag = reinterpret_cast<volatile int*>(tmem_slot + 1);
    Sched sc(tiles, kblocks, sk.sk_tiles);
    int t = 0, it = 0, tile, kb0, kb1;
    while (sc.next(tile, kb0, kb1)) {
      const int buf = t & 1;
      int mi, ni;
      tile_coords(tile, num_m, num_n, e.raster, mi, ni);
      const int m0 = mi * BM, n0 = ni * BN;
      if (A_MN && sk.bias_grad && n0 == 0) {
        bias_grad_tile<T, C::STAGES, C::STAGE>(smem, full, bsum, it, kb1 - kb0, warp, lane, stg,
                                               static_cast<T*>(sk.bias_grad), m0, M);
      }
      it += kb1 - kb0;
      mbar_wait(&tfull[buf], (t >> 1) & 1);
      fence_after();
      if (kb0 == 0 && kb1 == kblocks) {
        if (tma_store)
          epilogue_tile_tma<BN, FL, T>(e, &tcm, tmem_base + buf * BN, warp, lane, saddr(stg), m0, n0, M, N);
        else
          epilogue_tile<BN, T>(e, tmem_base + buf * BN, warp, lane, stg, m0, n0, M, N, vec_ok);
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
      } else {
        // stream-K partial: park the fp32 accumulators, count the arrival;
        // the last of the tile's CTAs sums the parts and runs the epilogue
        const int slot = int64_t(tile) * kblocks <= sc.it0 ? 0 : 1;
        store_partial<BN>(tmem_base + buf * BN, warp, lane, sk.ws + (size_t(sc.b) * 2 + slot) * (BM * BN));
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
        __threadfence();
        epi_bar();
        if (threadIdx.x == 64) {
          const int64_t i_beg = int64_t(tile) * kblocks, i_end = i_beg + kblocks;
          const int c0 = int(((i_beg + 1) * sc.G + sc.tsk - 1) / sc.tsk) - 1;
          const int c1 = int((i_end * sc.G + sc.tsk - 1) / sc.tsk) - 1;
          const int old = atomicAdd(sk.flags + tile, 1);
          const bool last = old == c1 - c0;
          if (last) sk.flags[tile] = 0;  // every part has arrived: re-arm
          *last_flag = last ? 1 : 0;
        }
        epi_bar();
        if (*last_flag) {
          __threadfence();
          reduce_partials<BN, T>(e, sc, sk, tile, warp, lane, stg, m0, n0, M, N, vec_ok);
        }
      }
      ++t;
    }
  }
  if (tma_store && warp >= 2 && lane == 0) bulk_wait0();  // C written before the CTA retires
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::TMEM_COLS));
  }
}

// ------------------------------------------------------------- 2-CTA (cta_group::2)
// A CTA pair (cluster of 2 on one TPC) computes a 256 x BN tile with one
// tcgen05.mma.cta_group::2 stream issued by the leader CTA: each CTA stages
// its 128-row half of A and its BN/2-row half of B, so per SM the smem
// operand traffic and the L2 re-read traffic are half of a 128 x BN 1-CTA
// tile. Each CTA's TMEM holds its 128 accumulator rows; both run the same
// coalesced epilogue.
template <int BN>
struct Cfg2 {
  static constexpr int A_BYTES = 128 * BK * 2;
  static constexpr int B_BYTES = (BN / 2) * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = (192 * 1024) / STAGE > 8 ? 8 : (192 * 1024) / STAGE;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256 + kEpiWarps * kStgFloats * 4;
  static constexpr int TMEM_COLS = 2 * BN;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA load whose completion bytes land on the leader CTA's barrier
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, uint32_t leader_bar, void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void umma_pair(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
// commit: arrive on the barrier at this smem offset in both CTAs of the pair
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          saddr(bar)),
      "h"(uint16_t(3))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(saddr(bar)),
      "r"(cta)
      : "memory");
}

// FL >= 0: epilogue flags fixed at compile time (the hot combinations);
// tma_store: the epilogue writes C through TMA bulk stores (tcm) -- needs a
// 16-byte aligned C with ldc % 8 == 0, else the per-thread store epilogue runs
template <int BN, bool A_MN, bool B_MN, int FL, bool SK, typename T>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc2(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
             const __grid_constant__ CUtensorMap tcm, const Epi e, int M, int N, int K, int vec_ok, int tma_store,
             const Sk sk) {
  // stream-K (sk.sk_tiles > 0, tma_store only): the k-iterations of the first
  // sk_tiles tiles are cut evenly over all pairs; a pair whose range covers a
  // tile only in part parks its fp32 accumulators in sk.ws and the last
  // arriving part sums them in k order and runs the epilogue (deterministic)
  void* bias_grad = sk.bias_grad;
  using C = Cfg2<BN>;
  constexpr int PM = 256;      // rows per pair tile
  constexpr int HB = BN / 2;   // B rows staged by each CTA
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // [stages][epilogue staging: 8 warps x 4 KB, 1024-aligned][barriers]
  uint8_t* stg_region = smem + C::STAGES * C::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(stg_region + kEpiWarps * kStgFloats * 4);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* bsum = tempty + 2;  // per stage: the epilogue warps finished their bias-gradient read
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bsum + C::STAGES);
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) trace(0);  // entry
  if (threadIdx.x == 32) {  // pull both TMA descriptors in while the prologue runs
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&bsum[s], kEpiWarps);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * kEpiWarps);  // epilogue warps of both CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  cluster_sync();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) trace(1);  // prologue done (barriers, TMEM, cluster sync)
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  if (threadIdx.x == 0) trace(2);  // predecessor complete

  const int num_m = (M + PM - 1) / PM, num_n = (N + BN - 1) / BN;
  const int tiles = num_m * num_n, kblocks = (K + BK - 1) / BK;
  const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;
  const int sk_tiles = SK && tma_store ? sk.sk_tiles : 0;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0, tile, kb0, kb1;
      uint32_t bias_pend = 0, bias_ph = 0;  // per stage: a bias-tile read outstanding / its bsum phase
      Sched sc(tiles, kblocks, sk_tiles, npairs, pair);
      while (sc.next(tile, kb0, kb1)) {
        int mi, ni;
        tile_coords(tile, num_m, num_n, e.raster, mi, ni);
        const int m0 = mi * PM + 128 * int(rank);
        const int n0 = ni * BN + HB * int(rank);
        const bool btile = A_MN && bias_grad && ni == 0;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % C::STAGES;
          const uint32_t ph = (it / C::STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          if (bias_pend >> s & 1) {
            mbar_wait(&bsum[s], bias_ph >> s & 1);
            bias_ph ^= 1u << s;
            bias_pend &= ~(1u << s);
          }
          if (btile) bias_pend |= 1u << s;
          if (leader) mbar_expect_tx(&full[s], 2 * C::STAGE);
          if (it == 0) trace(3);  // first TMA issued
          const uint32_t lbar = saddr(&full[s]) & 0xFEFFFFFFu;  // the leader CTA's barrier
          uint8_t* a_dst = smem + s * C::STAGE;
          uint8_t* b_dst = a_dst + C::A_BYTES;
          const int k0 = kb * BK;
          if (!A_MN) {
            tma_load_2d_pair(&ta, lbar, a_dst, k0, m0);
          } else {
            tma_load_2d_pair(&ta, lbar, a_dst, m0, k0);
            tma_load_2d_pair(&ta, lbar, a_dst + 8192, m0 + 64, k0);
          }
          if (!B_MN) {
            tma_load_2d_pair(&tb, lbar, b_dst, k0, n0);
          } else {
#pragma unroll
            for (int j = 0; j < HB / 64; ++j) tma_load_2d_pair(&tb, lbar, b_dst + j * 8192, n0 + 64 * j, k0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      const uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
      const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (uint32_t(A_MN) << 15) |
                             (uint32_t(B_MN) << 16) | (uint32_t(BN >> 3) << 17) | (uint32_t(PM >> 4) << 24);
      int it = 0, t = 0, tile, kb0, kb1;
      Sched sc(tiles, kblocks, sk_tiles, npairs, pair);
      for (; sc.next(tile, kb0, kb1); ++t) {
        const int buf = t & 1;
        mbar_wait(&tempty[buf], ((t >> 1) & 1) ^ 1);
        fence_after();
        const uint32_t d_tmem = tmem_base + buf * BN;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % C::STAGES;
          mbar_wait(&full[s], (it / C::STAGES) & 1);
          fence_after();
          if (it == 0) trace(4);  // first stage landed
          const uint32_t a_addr = saddr(smem + s * C::STAGE);
          const uint32_t b_addr = a_addr + C::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? smem_desc(a_addr + k * 2048, 8192, 1024) : smem_desc(a_addr + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? smem_desc(b_addr + k * 2048, 8192, 1024) : smem_desc(b_addr + k * 32, 16, 1024);
            umma_pair(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          umma_commit_pair(&empty[s]);
        }
        umma_commit_pair(&tfull[buf]);
        trace(5);  // last MMA of a tile issued
      }
    }
  } else {
    float* stg = reinterpret_cast<float*>(stg_region) + (warp - 2) * kStgFloats;
    volatile int* last_flag = reinterpret_cast<volatile int*>(tmem_slot + 1);
    int t = 0, it = 0, tile, kb0, kb1;
    Sched sc(tiles, kblocks, sk_tiles, npairs, pair);
    for (; sc.next(tile, kb0, kb1); ++t) {
      const int buf = t & 1;
      int mi, ni;
      tile_coords(tile, num_m, num_n, e.raster, mi, ni);
      const int m0 = mi * PM + 128 * int(rank), n0 = ni * BN;
      // fused bias gradient: each CTA sums its own 128-row half of A; the
      // pair's MMA commit on empty[s] (multicast to both CTAs) says the stage
      // is complete and still unrecycled (never combined with stream-K)
      if (A_MN && bias_grad && n0 == 0)
        bias_grad_tile<T, C::STAGES, C::STAGE>(smem, empty, bsum, it, kb1 - kb0, warp, lane, stg,
                                               static_cast<T*>(bias_grad), m0, M);
      it += kb1 - kb0;
      mbar_wait(&tfull[buf], (t >> 1) & 1);
      fence_after();
      if (threadIdx.x == 64) trace(6);  // accumulators ready
      if (!SK || (kb0 == 0 && kb1 == kblocks)) {
        if (tma_store)
          epilogue_tile_tma<BN, FL, T>(e, &tcm, tmem_base + buf * BN, warp, lane, saddr(stg), m0, n0, M, N);
        else
          epilogue_tile<BN, T>(e, tmem_base + buf * BN, warp, lane, stg, m0, n0, M, N, vec_ok);
        if (threadIdx.x == 64) trace(7);  // epilogue of this warp done
        fence_before();
        __syncwarp();
        if (lane == 0) {
          if (leader) mbar_arrive(&tempty[buf]);
          else mbar_arrive_cta(&tempty[buf], 0);
        }
      } else if constexpr (SK) {
        // stream-K part: park this CTA's accumulators in its slot (0: the
        // pair's first unit, 1: its last), release TMEM, count the arrival
        const int slot = int64_t(tile) * kblocks <= sc.it0 ? 0 : 1;
        const size_t slot_floats = size_t(128) * BN;
        store_partial_rows<BN>(tmem_base + buf * BN, warp, lane,
                               sk.ws + ((size_t(pair) * 2 + rank) * 2 + slot) * slot_floats);
        if (threadIdx.x == 64) trace(11);  // partial stored (this warp)
        fence_before();
        __syncwarp();
        if (lane == 0) {
          if (leader) mbar_arrive(&tempty[buf]);
          else mbar_arrive_cta(&tempty[buf], 0);
        }
        __threadfence();
        epi_bar();
        const int64_t i_beg = int64_t(tile) * kblocks, i_end = i_beg + kblocks;
        const int c0 = int(((i_beg + 1) * sc.G + sc.tsk - 1) / sc.tsk) - 1;
        const int c1 = int((i_end * sc.G + sc.tsk - 1) / sc.tsk) - 1;
        if (threadIdx.x == 64) {
          const int old = atomicAdd(sk.flags + 2 * tile + int(rank), 1);
          const bool last = old == c1 - c0;
          if (last) sk.flags[2 * tile + int(rank)] = 0;  // every part has arrived: re-arm
          *last_flag = last ? 1 : 0;
        }
        epi_bar();
        if (*last_flag) {
          __threadfence();
          WsSum ws;
          for (int c = c0; c <= c1 && ws.n < 8; ++c) {
            const int sl = i_beg <= sc.start_of(c) ? 0 : 1;
            ws.slot[ws.n++] = sk.ws + ((size_t(c) * 2 + rank) * 2 + sl) * slot_floats;
          }
          if (threadIdx.x == 64) trace(22);  // last part: fix-up starts
          epilogue_tile_tma<BN, FL, T>(e, &tcm, 0, warp, lane, saddr(stg), m0, n0, M, N, ws);
          if (threadIdx.x == 64) trace(23);  // fix-up epilogue done
        }
        epi_bar();  // last_flag is reused by the next unit
      }
    }
  }
  if (tma_store && warp >= 2 && lane == 0) bulk_wait0();  // C written before the CTA retires
  fence_before();
  __syncthreads();
  if (threadIdx.x == 0) trace(8);  // all warps done
  cluster_sync();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::TMEM_COLS));
  }
  if (threadIdx.x == 32) trace(9);  // TMEM released
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// 2-D map over a row-major [rows x cols] matrix with leading dimension ld,
// box {64 (inner), box_rows}, 128B swizzle, OOB -> zero
inline bool make_map(CUtensorMap* map, int dtype, const void* base, int64_t cols, int64_t rows, int64_t ld,
              int box_rows) {
  EncodeFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t box[2] = {64u, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = enc(map, dtype == SFK_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

inline int num_sms_cached() {
  static int n = -1;
  if (n < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) n = 148;
  }
  return n;
}

template <int BN, bool A_MN, bool B_MN, int FL, typename T>
int launch(const sfk_gemm_args* g, const Epi& e, bool vec_ok, cudaStream_t s, int sk_tiles, int sk_grid) {
  using C = Cfg<BN>;
  CUtensorMap ta, tb, tcm;
  // A: K-major [m][k] -> map cols=k rows=m, box rows 128; MN-major [k][m] -> cols=m rows=k, box 64x64
  bool ok = A_MN ? make_map(&ta, g->dtype, g->a, g->m, g->k, g->lda, 64)
                 : make_map(&ta, g->dtype, g->a, g->k, g->m, g->lda, BM);
  ok = ok && (B_MN ? make_map(&tb, g->dtype, g->b, g->n, g->k, g->ldb, 64)
                   : make_map(&tb, g->dtype, g->b, g->k, g->n, g->ldb, BN));
  if (!ok) {
    set_error("sfk_gemm: cuTensorMapEncodeTiled failed (alignment/stride?)");
    return SFK_EINVAL;
  }
  const bool tma_store = vec_ok && make_map(&tcm, g->dtype, g->c, g->n, g->m, g->ldc, 32);
  if (!tma_store) tcm = ta;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(gemm_tc<BN, A_MN, B_MN, FL, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM) !=
        cudaSuccess)
      return check_launch("sfk_gemm: smem attribute");
    attr_set = true;
  }
  const int tiles = ((g->m + BM - 1) / BM) * ((g->n + BN - 1) / BN);
  const int sms = g->max_sms > 0 && g->max_sms < num_sms_cached() ? g->max_sms : num_sms_cached();
  const int grid = sk_tiles > 0 ? sk_grid : (tiles < sms ? tiles : sms);
  Sk sk{sk_tiles > 0 ? g->workspace : nullptr, sk_tiles > 0 ? g->counters : nullptr, sk_tiles, g->bias_grad};
  launch_pdl(gemm_tc<BN, A_MN, B_MN, FL, T>, dim3(grid), dim3(kThreads), size_t(C::SMEM), s, ta, tb, tcm, e, g->m,
             g->n, g->k, vec_ok ? 1 : 0, tma_store ? 1 : 0, sk);
  return check_launch("sfk_gemm(tcgen05)");
}

// Stream-K plan for the pair kernel: the stream-K region in tiles (0 = plain
// data-parallel). Used when the last wave of 256 x BN tiles would leave pairs
// idle for a sizeable share of the run and the k-loop is long enough to split;
// never with the fused bias gradient (it assumes whole tiles). stream_k < 0 or
// no workspace disables it.
inline int pick_stream_k2(const sfk_gemm_args* g, int tiles, int bn) {
  if (g->stream_k < 0 || !g->workspace || !g->counters || g->bias_grad) return 0;
  const int G = num_sms_cached() / 2;
  if (g->workspace_floats < int64_t(G) * 4 * 128 * bn) return 0;
  const int kb = (g->k + BK - 1) / BK;
  if (kb < 8 || tiles % G == 0) return 0;
  const int sk_tiles = tiles < G ? tiles : tiles % G + G;
  if (2 * sk_tiles > g->n_counters) return 0;
  // a tile must not be cut into more than 8 parts (the fix-up's slot list)
  const int64_t per_pair = int64_t(sk_tiles) * kb / G;
  if (per_pair < 1 || (kb + per_pair - 1) / per_pair + 1 > 8) return 0;
  // data-parallel rounds vs stream-K share (in k-blocks per pair) plus a
  // fix-up allowance of ~3 k-blocks; split only for a >= 10% gain
  const double dp = double((tiles + G - 1) / G) * kb;
  const double skc = double(tiles) * kb / G + 3.0;
  return skc < 0.9 * dp ? sk_tiles : 0;
}

// the stream-K variant is instantiated only where the step uses it: 256-wide
// tiles, K-major A (forward and activation-gradient GEMMs), compile-time flags
template <int BN, bool A_MN, int FL>
constexpr bool kSkVariant = BN == 256 && !A_MN && FL >= 0;

template <int BN, bool A_MN, bool B_MN, int FL, typename T>
int launch2(const sfk_gemm_args* g, const Epi& e, bool vec_ok, cudaStream_t s) {
  using C = Cfg2<BN>;
  CUtensorMap ta, tb, tcm;
  bool ok = A_MN ? make_map(&ta, g->dtype, g->a, g->m, g->k, g->lda, 64)
                 : make_map(&ta, g->dtype, g->a, g->k, g->m, g->lda, 128);
  ok = ok && (B_MN ? make_map(&tb, g->dtype, g->b, g->n, g->k, g->ldb, 64)
                   : make_map(&tb, g->dtype, g->b, g->k, g->n, g->ldb, BN / 2));
  if (!ok) {
    set_error("sfk_gemm: cuTensorMapEncodeTiled failed (alignment/stride?)");
    return SFK_EINVAL;
  }
  // C through TMA bulk stores: 32-row x 64-column boxes, 128B swizzle
  const bool tma_store = vec_ok && make_map(&tcm, g->dtype, g->c, g->n, g->m, g->ldc, 32);
  if (!tma_store) tcm = ta;
  static bool attr_set = false;
  if (!attr_set) {
    if (cudaFuncSetAttribute(gemm_tc2<BN, A_MN, B_MN, FL, false, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             C::SMEM) != cudaSuccess)
      return check_launch("sfk_gemm: smem attribute");
    if constexpr (kSkVariant<BN, A_MN, FL>)
      if (cudaFuncSetAttribute(gemm_tc2<BN, A_MN, B_MN, FL, true, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               C::SMEM) != cudaSuccess)
        return check_launch("sfk_gemm: smem attribute");
    attr_set = true;
  }
  const int tiles = ((g->m + 255) / 256) * ((g->n + BN - 1) / BN);
  const int max_pairs = (g->max_sms > 0 && g->max_sms < num_sms_cached() ? g->max_sms : num_sms_cached()) / 2;
  int pairs = tiles < max_pairs ? tiles : max_pairs > 0 ? max_pairs : 1;
  Sk sk{nullptr, nullptr, 0, g->bias_grad};
  if (tma_store && kSkVariant<BN, A_MN, FL>) {
    const int skt = pick_stream_k2(g, tiles, BN);
    if (skt > 0) {
      sk = Sk{g->workspace, g->counters, skt, nullptr};
      pairs = num_sms_cached() / 2;
    }
  }
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if constexpr (kSkVariant<BN, A_MN, FL>) {
    if (sk.sk_tiles > 0) {
      cudaLaunchKernelEx(&cfg, gemm_tc2<BN, A_MN, B_MN, FL, true, T>, ta, tb, tcm, e, g->m, g->n, g->k,
                         vec_ok ? 1 : 0, tma_store ? 1 : 0, sk);
      return check_launch("sfk_gemm(tcgen05 pair, stream-K)");
    }
  }
  cudaLaunchKernelEx(&cfg, gemm_tc2<BN, A_MN, B_MN, FL, false, T>, ta, tb, tcm, e, g->m, g->n, g->k, vec_ok ? 1 : 0,
                     tma_store ? 1 : 0, sk);
  return check_launch("sfk_gemm(tcgen05 pair)");
}

// tile width by wave efficiency (tiles / (waves * SMs)); wider wins ties.
// 64-wide tiles are never picked: at 128 x 64 the operand traffic per MMA
// (24 KB per 64-deep k-block for 128 MMA cycles) starves the tensor pipe on
// L2 bandwidth, which costs more than any wave-quantisation loss.
inline int pick_bn(int m, int n) {
  const int sms = num_sms_cached();
  int best = 256;
  double best_eff = -1;
  for (int bn : {256, 128}) {
    const long tiles = long((m + BM - 1) / BM) * ((n + bn - 1) / bn);
    const long waves = (tiles + sms - 1) / sms;
    double eff = double(tiles) / double(waves * sms);
    eff *= (bn == 256 ? 1.0 : 0.85);  // operand-bandwidth penalty of 128-wide tiles
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = bn;
    }
  }
  return best;
}

// CTA-pair tile width (256 x BN pair tiles over SMs/2 pairs) by wave
// efficiency; ties and near-ties (within `slack`) go to the 256-wide tile
inline int pick_bn2(int m, int n, double slack) {
  const int pairs = num_sms_cached() / 2;
  auto eff = [&](int bn) {
    const long tiles = long((m + 255) / 256) * ((n + bn - 1) / bn);
    const long waves = (tiles + pairs - 1) / pairs;
    return double(tiles) / double(waves * pairs);
  };
  return eff(128) > eff(256) * (1.0 + slack) ? 128 : 256;
}

// Stream-K plan for a 128 x 256 1-CTA GEMM: returns the stream-K region size
// in tiles (0 = plain data-parallel) and the grid through *grid. Measured on
// B200, the fp32 partial tiles (128 KB each) make the fix-up expensive, so
// auto mode only splits few-tile GEMMs (the long-k weight gradients whose
// output is a handful of tiles), each tile over at most 3 CTAs; stream_k > 0
// forces the general form (last wave + remainder split over all SMs).
inline int pick_stream_k(const sfk_gemm_args* g, int* grid) {
  if (g->stream_k < 0 || !g->workspace || !g->counters) return 0;
  const int G = num_sms_cached();
  if (g->workspace_floats < int64_t(G) * 2 * BM * 256) return 0;
  const int tiles = ((g->m + BM - 1) / BM) * ((g->n + 255) / 256);
  const int kb = (g->k + BK - 1) / BK;
  if (kb < 4 || tiles % G == 0) return 0;
  const int sk_tiles = tiles < G ? tiles : tiles % G + G;
  if (sk_tiles > g->n_counters) return 0;
  if (g->stream_k > 0) {
    // every CTA gets at least one k-block
    *grid = int(std::min<int64_t>(G, int64_t(sk_tiles) * kb));
    if (tiles >= G) *grid = G;
    return sk_tiles;
  }
  if (3 * tiles > G || kb < 16) return 0;
  *grid = std::min(G, 3 * tiles);
  return tiles;
}

template <typename T>
int dispatch(const sfk_gemm_args* g, const Epi& e, bool vec_ok, cudaStream_t s) {
  int sk_grid = 0;
  const int skt = (g->tile_n == 0 || g->tile_n == 256) && g->pair <= 0 && !g->bias_grad ? pick_stream_k(g, &sk_grid) : 0;
  const int bn = skt > 0 ? 256 : g->tile_n > 0 ? g->tile_n
                               : g->pair > 0 ? pick_bn2(g->m, g->n, g->tile_n < 0 ? -g->tile_n * 0.01 : 0.0)
                                             : pick_bn(g->m, g->n);
  const int layout = (g->a_kmajor ? 0 : 2) | (g->b_kmajor ? 0 : 1);
  if (g->pair > 0) {
    // compile-time epilogues for the combinations the training step uses:
    // forward (K-major x K-major): preround [+bias [+relu | +residual]] or
    // +residual; activation gradient (K-major x MN-major): plain, accumulate,
    // residual, relu mask; weight gradient (MN-major x MN-major): accumulate
    constexpr int P = SFK_EPI_PREROUND, B = SFK_EPI_BIAS, RL = SFK_EPI_RELU, RS = SFK_EPI_RESIDUAL,
                  MK = SFK_EPI_MASK, AC = SFK_EPI_ACCUM;
    const int f = g->flags;
#define SFK_TC2_FL(BNV, AM, BMN, FLV) return launch2<BNV, AM, BMN, FLV, T>(g, e, vec_ok, s)
#define SFK_TC2(BNV)                                                                        \
  switch (layout) {                                                                         \
    case 0:                                                                                 \
      if (f == P) SFK_TC2_FL(BNV, false, false, P);                                         \
      if (f == (P | B)) SFK_TC2_FL(BNV, false, false, P | B);                               \
      if (f == (P | B | RL)) SFK_TC2_FL(BNV, false, false, P | B | RL);                     \
      if (f == (P | B | RS)) SFK_TC2_FL(BNV, false, false, P | B | RS);                     \
      if (f == (P | RS)) SFK_TC2_FL(BNV, false, false, P | RS);                             \
      SFK_TC2_FL(BNV, false, false, -1);                                                    \
    case 1:                                                                                 \
      if (f == 0) SFK_TC2_FL(BNV, false, true, 0);                                          \
      if (f == AC) SFK_TC2_FL(BNV, false, true, AC);                                        \
      if (f == RS) SFK_TC2_FL(BNV, false, true, RS);                                        \
      if (f == MK) SFK_TC2_FL(BNV, false, true, MK);                                        \
      SFK_TC2_FL(BNV, false, true, -1);                                                     \
    case 3:                                                                                 \
      if (f == AC) SFK_TC2_FL(BNV, true, true, AC);                                         \
      SFK_TC2_FL(BNV, true, true, -1);                                                      \
    default: SFK_TC2_FL(BNV, true, false, -1);                                              \
  }
    if (bn == 256) { SFK_TC2(256) }
    SFK_TC2(128)
#undef SFK_TC2
#undef SFK_TC2_FL
  }
  // 1-CTA tiles (small M: the decoder's per-position GEMMs): compile-time
  // epilogues for the forward combinations, runtime flags otherwise
  const int f1 = g->flags;
  constexpr int P1 = SFK_EPI_PREROUND, B1 = SFK_EPI_BIAS, RL1 = SFK_EPI_RELU, RS1 = SFK_EPI_RESIDUAL;
#define SFK_TC_FWD(BNV)                                                                               \
  if (f1 == P1) return launch<BNV, false, false, P1, T>(g, e, vec_ok, s, skt, sk_grid);               \
  if (f1 == (P1 | B1)) return launch<BNV, false, false, P1 | B1, T>(g, e, vec_ok, s, skt, sk_grid);   \
  if (f1 == (P1 | B1 | RL1)) return launch<BNV, false, false, P1 | B1 | RL1, T>(g, e, vec_ok, s, skt, sk_grid); \
  if (f1 == (P1 | B1 | RS1)) return launch<BNV, false, false, P1 | B1 | RS1, T>(g, e, vec_ok, s, skt, sk_grid); \
  return launch<BNV, false, false, -1, T>(g, e, vec_ok, s, skt, sk_grid);
#define SFK_TC(BNV)                                                         \
  switch (layout) {                                                         \
    case 0: SFK_TC_FWD(BNV)                                                 \
    case 1: return launch<BNV, false, true, -1, T>(g, e, vec_ok, s, skt, sk_grid);       \
    case 3: return launch<BNV, true, true, -1, T>(g, e, vec_ok, s, skt, sk_grid);        \
    default: return launch<BNV, true, false, -1, T>(g, e, vec_ok, s, skt, sk_grid);      \
  }
  if (bn == 256) { SFK_TC(256) }
  if (bn == 128) { SFK_TC(128) }
  switch (layout) {
    case 0: return launch<64, false, false, -1, T>(g, e, vec_ok, s, skt, sk_grid);
    case 1: return launch<64, false, true, -1, T>(g, e, vec_ok, s, skt, sk_grid);
    case 3: return launch<64, true, true, -1, T>(g, e, vec_ok, s, skt, sk_grid);
    default: return launch<64, true, false, -1, T>(g, e, vec_ok, s, skt, sk_grid);
  }
#undef SFK_TC
#undef SFK_TC_FWD
}
// per-dtype entry points (gemm_f16.cu / gemm_bf16.cu)
int dispatch_f16(const sfk_gemm_args* g, const Epi& e, bool vec_ok, cudaStream_t s);
int dispatch_bf16(const sfk_gemm_args* g, const Epi& e, bool vec_ok, cudaStream_t s);
}  // namespace tc

}  // namespace sfk

// debug builds (SFK_GEMM_TRACE): the last pair-GEMM launch's timeline, 2 x 12 ns stamps

// Tensor-core attention for fp16/bf16 (reference tape.cpp:229-258 forward,
// 426-480 backward). Sentences are short (<= max_positions = 256) and ragged,
// so each CTA owns one (sentence, head, 64-row block): the key/value (or
// query/dO) rows of that sentence-head are staged whole in shared memory and
// the products run on mma.sync m16n8k16 with fp32 accumulation:
//   fwd      S = Q K^T -> online softmax -> O = P V          (per query block)
//   bwd_dq   S, P (from saved {max, 1/sum}), dP = dO V^T,
//            dS = P (dP - D), dQ = sc dS K;  D = rowsum(dO * O) (per query block)
//   bwd_dkv  S^T = K Q^T, dP^T = V dO^T, dV = P^T dO, dK = sc dS^T Q (per key block)
// Spans: query row t of sentence b sees keys j < (causal ? t+1 : len[b]).
#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace sfk {
namespace fa {

constexpr int kWarps = 4;
constexpr int kRows = 16 * kWarps;  // rows per CTA block

template <typename T>
struct MmaT;
template <>
struct MmaT<__half> {
  static __device__ __forceinline__ void mma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  static __device__ __forceinline__ uint32_t pack(float x, float y) {
    __half2 h = __floats2half2_rn(x, y);
    return *reinterpret_cast<uint32_t*>(&h);
  }
};
template <>
struct MmaT<__nv_bfloat16> {
  static __device__ __forceinline__ void mma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  static __device__ __forceinline__ uint32_t pack(float x, float y) {
    __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
    return *reinterpret_cast<uint32_t*>(&h);
  }
};

// 8 consecutive 16-bit values from shared memory (16-byte aligned) as floats
template <typename T>
__device__ __forceinline__ void vec_ld8(const T* p, float (&f)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float2 t;
    if constexpr (std::is_same<T, __half>::value) t = __half22float2(*reinterpret_cast<const __half2*>(&w[j]));
    else t = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[j]));
    f[2 * j] = t.x;
    f[2 * j + 1] = t.y;
  }
}

// 2^x on the SFU, flushing subnormal results to zero (probabilities that
// small are zero in every 16-bit output anyway)
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(su32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(su32(p)));
}

// A fragment (16x16) of a row-major smem tile at (r0, c0), row stride ld (elements)
template <typename T>
__device__ __forceinline__ void load_a(uint32_t (&a)[4], const T* s, int ld, int r0, int c0, int lane) {
  const int r = r0 + (lane & 7) + ((lane >> 3) & 1) * 8, c = c0 + (lane >> 4) * 8;
  ldsm_x4(a, s + r * ld + c);
}
// B fragments for two n8 tiles (n0, n0+8), k16 at k0, from smem stored [n][k] (k contiguous)
template <typename T>
__device__ __forceinline__ void load_b_nk(uint32_t (&b)[4], const T* s, int ld, int n0, int k0, int lane) {
  const int r = n0 + (lane & 7) + (lane >> 4) * 8, c = k0 + ((lane >> 3) & 1) * 8;
  ldsm_x4(b, s + r * ld + c);  // b[0],b[1]: tile n0 ; b[2],b[3]: tile n0+8
}
// B fragments for two n8 tiles from smem stored [k][n] (n contiguous): transposed load
template <typename T>
__device__ __forceinline__ void load_b_kn(uint32_t (&b)[4], const T* s, int ld, int k0, int n0, int lane) {
  const int r = k0 + (lane & 7) + ((lane >> 3) & 1) * 8, c = n0 + (lane >> 4) * 8;
  ldsm_x4_t(b, s + r * ld + c);
}

// copy rows [r0, r0+n) x dh of a strided global matrix into smem rows [0, rows_pad) x DH (zero padded)
// cp.async (LDGSTS) staging: every 16-byte chunk of the tile is in flight at
// once (no register round trip, no load->store serialisation); rows past `n`
// and columns past `dh` are zero-filled via src-size 0. Caller waits with
// stage_wait() + __syncthreads().
template <typename T, int DH>
__device__ __forceinline__ void stage(T* s, int lds, const T* g, int64_t ldg, int r0, int n, int rows_pad, int dh) {
  // thread t always copies 16-byte column chunk t % VPR of rows t / VPR,
  // t / VPR + step, ...: pointers advance by a constant (no per-chunk index math)
  constexpr int VPR = DH / 8;
  const int step = int(blockDim.x) / VPR;  // blockDim.x is a multiple of VPR (64/128 threads, VPR <= 16)
  const int c = (int(threadIdx.x) % VPR) * 8;
  int r = int(threadIdx.x) / VPR;
  const bool cok = c < dh;
  const T* src = g + int64_t(r0 + r) * ldg + c;
  const int64_t sstep = int64_t(step) * ldg;
  uint32_t dst = su32(s + r * lds + c);
  const uint32_t dstep = uint32_t(step * lds * int(sizeof(T)));
#pragma unroll 4
  for (; r < rows_pad; r += step, src += sstep, dst += dstep) {
    const bool ok = cok && r < n;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(ok ? src : g), "r"(ok ? 16 : 0)
                 : "memory");
  }
}
__device__ __forceinline__ void stage_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

struct Args {
  int batch, qw, kw, heads, dh, causal;
  const int32_t* klen;
  float sc;
  const void *q, *k, *v, *o, *dout;
  int64_t ldq, ldk, ldv, ldo, lddo;
  void *out, *dq, *dk, *dv;
  int64_t ldout, lddq, lddk, lddv;
  float2* stats;
  float* dsum;
  int vec_dkv;  // dK/dV rows 16-byte aligned (ld % 8 == 0, aligned bases): whole-chunk stores
};

// One launch can serve several parts (sfk_attention_*_parts: the parts of a
// multi-part pass with the same kernel route): each part's sentences are a
// consecutive range of blockIdx.z, with their own widths, lengths and base
// pointers; the remaining fields (heads, dh, strides, scale) are shared.
struct PartArgs {
  int begin, qw, kw, vec_dkv;
  const int32_t* klen;
  const void *q, *k, *v, *o, *dout;
  void *dq, *dk, *dv;
  float2* stats;
  float* dsum;
};
constexpr int kMaxLaunchParts = 16;
struct LaunchArgs {
  Args base;
  int nparts;
  PartArgs part[kMaxLaunchParts];
};
// this CTA's part as a single-part Args; b = the sentence within the part
__device__ __forceinline__ Args part_view(const LaunchArgs& L, int& b) {
  int p = 0;
  for (int i = 1; i < L.nparts; ++i)
    if (int(blockIdx.z) >= L.part[i].begin) p = i;
  const PartArgs& pa = L.part[p];
  Args a = L.base;
  a.qw = pa.qw;
  a.kw = pa.kw;
  a.vec_dkv = pa.vec_dkv;
  a.klen = pa.klen;
  a.q = pa.q;
  a.k = pa.k;
  a.v = pa.v;
  a.o = pa.o;
  a.out = const_cast<void*>(pa.o);
  a.dout = pa.dout;
  a.dq = pa.dq;
  a.dk = pa.dk;
  a.dv = pa.dv;
  a.stats = pa.stats;
  a.dsum = pa.dsum;
  b = int(blockIdx.z) - pa.begin;
  return a;
}

// ------------------------------------------------------------------ forward
// R = query rows per CTA (64: 4 warps; 32: 2 warps for short sentences)
// KC = keys per chunk: 16 / 32 when every key span fits (short sentences), else 64.
// HP > 1 (sentences of <= 16 positions): one warp per head, HP heads of one
// sentence per CTA, staged as one HP*DH-wide tile (R = 16 rows).
// Scores are kept in log2 units (s * sc * log2 e) so each probability is one
// subtract and one SFU exp2; the saved max is converted back to natural units.
template <typename T, int DH, int R, int KC, int HP = 1>
__global__ void __launch_bounds__(HP > 1 ? 32 * HP : R * 2) fwd_k(const __grid_constant__ LaunchArgs L) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  int b;
  const Args a = part_view(L, b);
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int LD = HP * DH + 8;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, g = lane >> 2, tq = lane & 3;
  const int h0 = blockIdx.y * HP, h = h0 + (HP > 1 ? warp : 0), q0 = blockIdx.x * R;
  const int co = HP > 1 ? warp * DH : 0;  // this warp's head columns in the staged tiles
  if (q0 >= a.qw) return;  // a grid sized for the widest part of the launch
  const int len = a.causal ? a.kw : a.klen[b];
  // keys any row of this block can see
  const int nk = a.causal ? min(a.kw, min(q0 + R, a.qw)) : len;
  const int nk_pad = (nk + KC - 1) / KC * KC;
  T* Qs = reinterpret_cast<T*>(smem);
  T* Ks = Qs + R * LD;
  T* Vs = Ks + nk_pad * LD;
  const int64_t qrow0 = int64_t(b) * a.qw, krow0 = int64_t(b) * a.kw;
  stage<T, HP * DH>(Qs, LD, static_cast<const T*>(a.q) + h0 * a.dh, a.ldq, int(qrow0) + q0, min(R, a.qw - q0), R,
                    HP * a.dh);
  stage<T, HP * DH>(Ks, LD, static_cast<const T*>(a.k) + h0 * a.dh, a.ldk, int(krow0), nk, nk_pad, HP * a.dh);
  stage<T, HP * DH>(Vs, LD, static_cast<const T*>(a.v) + h0 * a.dh, a.ldv, int(krow0), nk, nk_pad, HP * a.dh);
  stage_wait();
  __syncthreads();
  const int r0 = HP > 1 ? 0 : warp * 16;
  if (q0 + r0 >= a.qw) return;
  uint32_t qa[DH / 16][4];
#pragma unroll
  for (int ks = 0; ks < DH / 16; ++ks) load_a<T>(qa[ks], Qs + co, LD, r0, ks * 16, lane);
  const int row_a = q0 + r0 + g, row_b = row_a + 8;  // the two rows this thread holds
  const int lim_a = row_a < a.qw ? (a.causal ? row_a + 1 : len) : 1;
  const int lim_b = row_b < a.qw ? (a.causal ? row_b + 1 : len) : 1;
  const int warp_keys = a.causal ? min(a.qw, q0 + r0 + 16) : len;
  const float c2 = a.sc * 1.4426950408889634f;  // natural score -> log2 units
  float m_a = -INFINITY, m_b = -INFINITY, l_a = 0.f, l_b = 0.f;
  float o[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  constexpr int NT = KC / 8;
  for (int kc = 0; kc < warp_keys; kc += KC) {
    float s[NT][4];
#pragma unroll
    for (int i = 0; i < NT; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < DH / 16; ++ks)
#pragma unroll
      for (int nt = 0; nt < NT; nt += 2) {
        uint32_t bb[4];
        load_b_nk<T>(bb, Ks + co, LD, kc + nt * 8, ks * 16, lane);
        MmaT<T>::mma(s[nt], qa[ks], bb[0], bb[1]);
        MmaT<T>::mma(s[nt + 1], qa[ks], bb[2], bb[3]);
      }
    float mx_a = m_a, mx_b = m_b;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = kc + nt * 8 + 2 * tq + e;
        s[nt][e] = j < lim_a ? s[nt][e] * c2 : -INFINITY;
        s[nt][2 + e] = j < lim_b ? s[nt][2 + e] * c2 : -INFINITY;
        mx_a = fmaxf(mx_a, s[nt][e]);
        mx_b = fmaxf(mx_b, s[nt][2 + e]);
      }
#pragma unroll
    for (int off = 1; off < 4; off <<= 1) {
      mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, off));
      mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, off));
    }
    const float al_a = ex2(m_a - mx_a), al_b = ex2(m_b - mx_b);
    m_a = mx_a;
    m_b = mx_b;
    float rs_a = 0.f, rs_b = 0.f;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      s[nt][0] = ex2(s[nt][0] - m_a);
      s[nt][1] = ex2(s[nt][1] - m_a);
      s[nt][2] = ex2(s[nt][2] - m_b);
      s[nt][3] = ex2(s[nt][3] - m_b);
      rs_a += s[nt][0] + s[nt][1];
      rs_b += s[nt][2] + s[nt][3];
    }
    l_a = l_a * al_a + rs_a;
    l_b = l_b * al_b + rs_b;
#pragma unroll
    for (int i = 0; i < DH / 8; ++i) {
      o[i][0] *= al_a;
      o[i][1] *= al_a;
      o[i][2] *= al_b;
      o[i][3] *= al_b;
    }
#pragma unroll
    for (int kk = 0; kk < NT / 2; ++kk) {  // 16 keys per k-step
      uint32_t pa[4] = {MmaT<T>::pack(s[2 * kk][0], s[2 * kk][1]), MmaT<T>::pack(s[2 * kk][2], s[2 * kk][3]),
                        MmaT<T>::pack(s[2 * kk + 1][0], s[2 * kk + 1][1]),
                        MmaT<T>::pack(s[2 * kk + 1][2], s[2 * kk + 1][3])};
#pragma unroll
      for (int nt = 0; nt < DH / 8; nt += 2) {
        uint32_t bb[4];
        load_b_kn<T>(bb, Vs + co, LD, kc + kk * 16, nt * 8, lane);
        MmaT<T>::mma(o[nt], pa, bb[0], bb[1]);
        MmaT<T>::mma(o[nt + 1], pa, bb[2], bb[3]);
      }
    }
  }
  l_a += __shfl_xor_sync(0xffffffffu, l_a, 1);
  l_a += __shfl_xor_sync(0xffffffffu, l_a, 2);
  l_b += __shfl_xor_sync(0xffffffffu, l_b, 1);
  l_b += __shfl_xor_sync(0xffffffffu, l_b, 2);
  const float ia = 1.0f / l_a, ib = 1.0f / l_b;
  // the warp's Q rows are consumed (fragments are in registers): stage its
  // 16 x DH output there and write whole 16-byte row chunks
  T* Os = Qs + co + r0 * LD;
#pragma unroll
  for (int nt = 0; nt < DH / 8; ++nt) {
    const int c = nt * 8 + 2 * tq;
    *reinterpret_cast<uint32_t*>(Os + g * LD + c) = MmaT<T>::pack(o[nt][0] * ia, o[nt][1] * ia);
    *reinterpret_cast<uint32_t*>(Os + (g + 8) * LD + c) = MmaT<T>::pack(o[nt][2] * ib, o[nt][3] * ib);
  }
  __syncwarp();
  {
    T* out = static_cast<T*>(a.out) + h * a.dh;
    constexpr int VPR = DH / 8;
#pragma unroll
    for (int k = 0; k < 16 * VPR / 32; ++k) {
      const int idx = k * 32 + lane, rr = idx / VPR, cc = (idx % VPR) * 8;
      const int row = q0 + r0 + rr;
      if (row < a.qw && cc < a.dh)
        *reinterpret_cast<uint4*>(out + (qrow0 + row) * a.ldout + cc) = *reinterpret_cast<const uint4*>(Os + rr * LD + cc);
    }
  }
  if (tq == 0) {  // max back in natural units (the saved-stats contract)
    const float ln2 = 0.6931471805599453f;
    if (row_a < a.qw) a.stats[(qrow0 + row_a) * a.heads + h] = make_float2(m_a * ln2, ia);
    if (row_b < a.qw) a.stats[(qrow0 + row_b) * a.heads + h] = make_float2(m_b * ln2, ib);
  }
}

// ------------------------------------------------------------------ backward: dQ (+ D)
template <typename T, int DH>
__global__ void __launch_bounds__(kWarps * 32) bwd_dq_k(const __grid_constant__ LaunchArgs L) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  int b;
  const Args a = part_view(L, b);
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int LD = DH + 8;
  const int h = blockIdx.y, q0 = blockIdx.x * kRows;
  if (q0 >= a.qw) return;  // a grid sized for the widest part of the launch
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, g = lane >> 2, tq = lane & 3;
  const int len = a.causal ? a.kw : a.klen[b];
  const int nk = a.causal ? min(a.kw, min(q0 + kRows, a.qw)) : len;
  const int nk_pad = (nk + 63) & ~63;
  T* Qs = reinterpret_cast<T*>(smem);
  T* Gs = Qs + kRows * LD;  // dO
  T* Ks = Gs + kRows * LD;
  T* Vs = Ks + nk_pad * LD;
  const int64_t qrow0 = int64_t(b) * a.qw, krow0 = int64_t(b) * a.kw;
  const int nq = min(kRows, a.qw - q0);
  stage<T, DH>(Qs, LD, static_cast<const T*>(a.q) + h * a.dh, a.ldq, int(qrow0) + q0, nq, kRows, a.dh);
  stage<T, DH>(Gs, LD, static_cast<const T*>(a.dout) + h * a.dh, a.lddo, int(qrow0) + q0, nq, kRows, a.dh);
  stage<T, DH>(Ks, LD, static_cast<const T*>(a.k) + h * a.dh, a.ldk, int(krow0), nk, nk_pad, a.dh);
  stage<T, DH>(Vs, LD, static_cast<const T*>(a.v) + h * a.dh, a.ldv, int(krow0), nk, nk_pad, a.dh);
  stage_wait();
  __syncthreads();
  const int r0 = warp * 16;
  if (q0 + r0 >= a.qw) return;
  const int row_a = q0 + r0 + g, row_b = row_a + 8;
  // D = rowsum(dO * O) for the two rows (4 threads of a quad split the columns)
  float D_a = 0.f, D_b = 0.f;
  {
    const T* O = static_cast<const T*>(a.o) + h * a.dh;
    if (a.dh % 32 == 0) {
      // each lane of a quad: a contiguous quarter of the row, 16-byte loads
      const int qw = a.dh / 4;
      for (int c = tq * qw; c < (tq + 1) * qw; c += 8) {
        float g8[8], o8[8];
        if (row_a < a.qw) {
          vec_ld8<T>(Gs + (r0 + g) * LD + c, g8);
          vec_ld8<T>(O + (qrow0 + row_a) * a.ldo + c, o8);
#pragma unroll
          for (int j = 0; j < 8; ++j) D_a += g8[j] * o8[j];
        }
        if (row_b < a.qw) {
          vec_ld8<T>(Gs + (r0 + g + 8) * LD + c, g8);
          vec_ld8<T>(O + (qrow0 + row_b) * a.ldo + c, o8);
#pragma unroll
          for (int j = 0; j < 8; ++j) D_b += g8[j] * o8[j];
        }
      }
    } else {
      for (int c = tq; c < a.dh; c += 4) {
        if (row_a < a.qw)
          D_a += Num<T>::ld(Gs + (r0 + g) * LD + c) * Num<T>::ld(O + (qrow0 + row_a) * a.ldo + c);
        if (row_b < a.qw)
          D_b += Num<T>::ld(Gs + (r0 + g + 8) * LD + c) * Num<T>::ld(O + (qrow0 + row_b) * a.ldo + c);
      }
    }
    D_a += __shfl_xor_sync(0xffffffffu, D_a, 1);
    D_a += __shfl_xor_sync(0xffffffffu, D_a, 2);
    D_b += __shfl_xor_sync(0xffffffffu, D_b, 1);
    D_b += __shfl_xor_sync(0xffffffffu, D_b, 2);
    if (tq == 0) {
      if (row_a < a.qw) a.dsum[(qrow0 + row_a) * a.heads + h] = D_a;
      if (row_b < a.qw) a.dsum[(qrow0 + row_b) * a.heads + h] = D_b;
    }
  }
  uint32_t qa[DH / 16][4], ga[DH / 16][4];
#pragma unroll
  for (int ks = 0; ks < DH / 16; ++ks) {
    load_a<T>(qa[ks], Qs, LD, r0, ks * 16, lane);
    load_a<T>(ga[ks], Gs, LD, r0, ks * 16, lane);
  }
  const float2 st_a = row_a < a.qw ? a.stats[(qrow0 + row_a) * a.heads + h] : make_float2(0.f, 0.f);
  const float2 st_b = row_b < a.qw ? a.stats[(qrow0 + row_b) * a.heads + h] : make_float2(0.f, 0.f);
  const int lim_a = row_a < a.qw ? (a.causal ? row_a + 1 : len) : 0;
  const int lim_b = row_b < a.qw ? (a.causal ? row_b + 1 : len) : 0;
  const int warp_keys = a.causal ? min(a.qw, q0 + r0 + 16) : len;
  const float l2e = 1.4426950408889634f, c2 = a.sc * l2e;
  float dq[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;
  for (int kc = 0; kc < warp_keys; kc += 64) {
    float s[8][4], dp[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[i][e] = dp[i][e] = 0.f;
#pragma unroll
    for (int ks = 0; ks < DH / 16; ++ks)
#pragma unroll
      for (int nt = 0; nt < 8; nt += 2) {
        uint32_t bk[4], bv[4];
        load_b_nk<T>(bk, Ks, LD, kc + nt * 8, ks * 16, lane);
        load_b_nk<T>(bv, Vs, LD, kc + nt * 8, ks * 16, lane);
        MmaT<T>::mma(s[nt], qa[ks], bk[0], bk[1]);
        MmaT<T>::mma(s[nt + 1], qa[ks], bk[2], bk[3]);
        MmaT<T>::mma(dp[nt], ga[ks], bv[0], bv[1]);
        MmaT<T>::mma(dp[nt + 1], ga[ks], bv[2], bv[3]);
      }
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = kc + nt * 8 + 2 * tq + e;
        const float pa = j < lim_a ? ex2(s[nt][e] * c2 - st_a.x * l2e) * st_a.y : 0.f;
        const float pb = j < lim_b ? ex2(s[nt][2 + e] * c2 - st_b.x * l2e) * st_b.y : 0.f;
        s[nt][e] = pa * (dp[nt][e] - D_a);
        s[nt][2 + e] = pb * (dp[nt][2 + e] - D_b);
      }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t da[4] = {MmaT<T>::pack(s[2 * kk][0], s[2 * kk][1]), MmaT<T>::pack(s[2 * kk][2], s[2 * kk][3]),
                        MmaT<T>::pack(s[2 * kk + 1][0], s[2 * kk + 1][1]),
                        MmaT<T>::pack(s[2 * kk + 1][2], s[2 * kk + 1][3])};
#pragma unroll
      for (int nt = 0; nt < DH / 8; nt += 2) {
        uint32_t bb[4];
        load_b_kn<T>(bb, Ks, LD, kc + kk * 16, nt * 8, lane);
        MmaT<T>::mma(dq[nt], da, bb[0], bb[1]);
        MmaT<T>::mma(dq[nt + 1], da, bb[2], bb[3]);
      }
    }
  }
  T* out = static_cast<T*>(a.dq) + h * a.dh;
#pragma unroll
  for (int nt = 0; nt < DH / 8; ++nt) {
    const int c = nt * 8 + 2 * tq;
    if (c >= a.dh) continue;
    if (row_a < a.qw)
      *reinterpret_cast<uint32_t*>(out + (qrow0 + row_a) * a.lddq + c) =
          MmaT<T>::pack(dq[nt][0] * a.sc, dq[nt][1] * a.sc);
    if (row_b < a.qw)
      *reinterpret_cast<uint32_t*>(out + (qrow0 + row_b) * a.lddq + c) =
          MmaT<T>::pack(dq[nt][2] * a.sc, dq[nt][3] * a.sc);
  }
}

// ------------------------------------------------------------------ backward: dK, dV
template <typename T, int DH>
__global__ void __launch_bounds__(kWarps * 32, 3) bwd_dkv_k(const __grid_constant__ LaunchArgs L) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  int b;
  const Args a = part_view(L, b);
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int LD = DH + 8;
  constexpr int NC = DH >= 64 ? 32 : 64;  // query columns per chunk (register budget: 3 CTAs per SM at DH 64)
  const int h = blockIdx.y, k0 = blockIdx.x * kRows;
  if (k0 >= a.kw) return;  // a grid sized for the widest part of the launch
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, g = lane >> 2, tq = lane & 3;
  const int len = a.causal ? a.kw : a.klen[b];
  const int64_t qrow0 = int64_t(b) * a.qw, krow0 = int64_t(b) * a.kw;
  // queries that can see a key of this block
  const int qstart = a.causal ? k0 : 0;
  const int nq = max(0, a.qw - qstart);
  // +64: a warp's chunks start at its first key row (r0) and run NC past nq
  const int nq_pad = ((nq + 63) & ~63) + 64;
  T* Ks = reinterpret_cast<T*>(smem);
  T* Vs = Ks + kRows * LD;
  T* Qs = Vs + kRows * LD;
  T* Gs = Qs + nq_pad * LD;
  float2* St = reinterpret_cast<float2*>(Gs + nq_pad * LD);
  float* Ds = reinterpret_cast<float*>(St + nq_pad);
  const int nk = min(kRows, a.kw - k0);
  stage<T, DH>(Ks, LD, static_cast<const T*>(a.k) + h * a.dh, a.ldk, int(krow0) + k0, nk, kRows, a.dh);
  stage<T, DH>(Vs, LD, static_cast<const T*>(a.v) + h * a.dh, a.ldv, int(krow0) + k0, nk, kRows, a.dh);
  stage<T, DH>(Qs, LD, static_cast<const T*>(a.q) + h * a.dh, a.ldq, int(qrow0) + qstart, nq, nq_pad, a.dh);
  stage<T, DH>(Gs, LD, static_cast<const T*>(a.dout) + h * a.dh, a.lddo, int(qrow0) + qstart, nq, nq_pad, a.dh);
  for (int i = threadIdx.x; i < nq_pad; i += blockDim.x) {
    const bool ok = i < nq;
    const float2 sv = ok ? a.stats[(qrow0 + qstart + i) * a.heads + h] : make_float2(0.f, 0.f);
    St[i] = make_float2(sv.x * 1.4426950408889634f, sv.y);  // max in log2 units
    Ds[i] = ok ? a.dsum[(qrow0 + qstart + i) * a.heads + h] : 0.f;
  }
  stage_wait();
  __syncthreads();
  const int r0 = warp * 16;
  if (k0 + r0 >= a.kw) return;
  const int key_a = k0 + r0 + g, key_b = key_a + 8;
  float dk[DH / 8][4], dv[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;
  // non-causal: keys at or beyond len are never attended
  const bool any = a.causal ? true : (k0 + r0 < len);
  if (any) {
    uint32_t ka[DH / 16][4], va[DH / 16][4];
#pragma unroll
    for (int ks = 0; ks < DH / 16; ++ks) {
      load_a<T>(ka[ks], Ks, LD, r0, ks * 16, lane);
      load_a<T>(va[ks], Vs, LD, r0, ks * 16, lane);
    }
    const float l2e = 1.4426950408889634f, c2 = a.sc * l2e;
    // causal: queries before this warp's first key never see it
    const int qbeg = a.causal ? ((k0 + r0 - qstart) & ~15) : 0;
    for (int qc = qbeg; qc < nq; qc += NC) {
      float s[NC / 8][4], dp[NC / 8][4];
#pragma unroll
      for (int i = 0; i < NC / 8; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) s[i][e] = dp[i][e] = 0.f;
#pragma unroll
      for (int ks = 0; ks < DH / 16; ++ks)
#pragma unroll
        for (int nt = 0; nt < NC / 8; nt += 2) {
          uint32_t bq[4], bg[4];
          load_b_nk<T>(bq, Qs, LD, qc + nt * 8, ks * 16, lane);
          load_b_nk<T>(bg, Gs, LD, qc + nt * 8, ks * 16, lane);
          MmaT<T>::mma(s[nt], ka[ks], bq[0], bq[1]);
          MmaT<T>::mma(s[nt + 1], ka[ks], bq[2], bq[3]);
          MmaT<T>::mma(dp[nt], va[ks], bg[0], bg[1]);
          MmaT<T>::mma(dp[nt + 1], va[ks], bg[2], bg[3]);
        }
      // s: rows = keys (key_a / key_b), cols = queries qstart + qc + nt*8 + 2tq + e
      float p[NC / 8][4];
#pragma unroll
      for (int nt = 0; nt < NC / 8; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int qi = qc + nt * 8 + 2 * tq + e;  // index into staged queries
          const int t = qstart + qi;               // query position
          const float2 st = St[qi];
          const float D = Ds[qi];
          const bool qok = qi < nq;
          const bool va_ok = qok && key_a < a.kw && (a.causal ? key_a <= t : key_a < len);
          const bool vb_ok = qok && key_b < a.kw && (a.causal ? key_b <= t : key_b < len);
          const float pa = va_ok ? ex2(s[nt][e] * c2 - st.x) * st.y : 0.f;
          const float pb = vb_ok ? ex2(s[nt][2 + e] * c2 - st.x) * st.y : 0.f;
          p[nt][e] = pa;
          p[nt][2 + e] = pb;
          s[nt][e] = pa * (dp[nt][e] - D);
          s[nt][2 + e] = pb * (dp[nt][2 + e] - D);
        }
#pragma unroll
      for (int kk = 0; kk < NC / 16; ++kk) {
        uint32_t pa[4] = {MmaT<T>::pack(p[2 * kk][0], p[2 * kk][1]), MmaT<T>::pack(p[2 * kk][2], p[2 * kk][3]),
                          MmaT<T>::pack(p[2 * kk + 1][0], p[2 * kk + 1][1]),
                          MmaT<T>::pack(p[2 * kk + 1][2], p[2 * kk + 1][3])};
        uint32_t da[4] = {MmaT<T>::pack(s[2 * kk][0], s[2 * kk][1]), MmaT<T>::pack(s[2 * kk][2], s[2 * kk][3]),
                          MmaT<T>::pack(s[2 * kk + 1][0], s[2 * kk + 1][1]),
                          MmaT<T>::pack(s[2 * kk + 1][2], s[2 * kk + 1][3])};
#pragma unroll
        for (int nt = 0; nt < DH / 8; nt += 2) {
          uint32_t bg[4], bq[4];
          load_b_kn<T>(bg, Gs, LD, qc + kk * 16, nt * 8, lane);
          load_b_kn<T>(bq, Qs, LD, qc + kk * 16, nt * 8, lane);
          MmaT<T>::mma(dv[nt], pa, bg[0], bg[1]);
          MmaT<T>::mma(dv[nt + 1], pa, bg[2], bg[3]);
          MmaT<T>::mma(dk[nt], da, bq[0], bq[1]);
          MmaT<T>::mma(dk[nt + 1], da, bq[2], bq[3]);
        }
      }
    }
  }
  T* dko = static_cast<T*>(a.dk) + h * a.dh;
  T* dvo = static_cast<T*>(a.dv) + h * a.dh;
#pragma unroll
  for (int nt = 0; nt < DH / 8; ++nt) {
    const int c = nt * 8 + 2 * tq;
    if (c >= a.dh) continue;
    if (key_a < a.kw) {
      *reinterpret_cast<uint32_t*>(dko + (krow0 + key_a) * a.lddk + c) =
          MmaT<T>::pack(dk[nt][0] * a.sc, dk[nt][1] * a.sc);
      *reinterpret_cast<uint32_t*>(dvo + (krow0 + key_a) * a.lddv + c) = MmaT<T>::pack(dv[nt][0], dv[nt][1]);
    }
    if (key_b < a.kw) {
      *reinterpret_cast<uint32_t*>(dko + (krow0 + key_b) * a.lddk + c) =
          MmaT<T>::pack(dk[nt][2] * a.sc, dk[nt][3] * a.sc);
      *reinterpret_cast<uint32_t*>(dvo + (krow0 + key_b) * a.lddv + c) = MmaT<T>::pack(dv[nt][2], dv[nt][3]);
    }
  }
}

// ------------------------------------------------------------------ backward, one CTA
// Short sentences (query and key widths <= 64, the common case for the
// length-bucketed batches): one CTA per (sentence, head) stages Q, dO, K, V
// once and runs both halves of the backward -- dQ per query warp, then dK/dV
// per key warp -- with D = rowsum(dO * O) and the saved softmax stats kept in
// shared memory. Same arithmetic, in the same order, as bwd_dq_k + bwd_dkv_k.
// R = rows per CTA: 128 (8 warps) for widths <= 128, 64 (4 warps) for widths
// <= 64, 32 (2 warps) for widths <= 32. N16: 16-query dK/dV chunks and 32-key
// dQ chunks, so the staged query rows need no padding past R and fewer
// registers buy more resident CTAs per SM (the wave count of a C4 batch is
// what bounds these launches); otherwise 32-query chunks.
// R = 16 with HP > 1 (sentences of <= 16 positions): one warp per head, HP
// heads of one sentence per CTA staged as HP*DH-wide tiles.
template <int R, int DH, bool N16>
struct SmallCfg {
  static constexpr int NC = N16 || R >= 128 || R == 16 ? 16 : 32;  // query columns per dK/dV chunk
  static constexpr int KC = R == 16 ? 16 : !N16 && R == 64 ? 64 : 32;  // keys per dQ chunk
  static constexpr int QP = NC == 16 ? R : R + 32;      // staged query rows (chunks run NC-16 past qw)
  static constexpr int MINB = R == 16 ? 4 : R == 32 ? (N16 ? 8 : 6) : R == 64 ? (DH <= 64 ? (N16 ? 4 : 3) : 1)
                                                                               : (DH <= 64 ? 2 : 1);
};
template <typename T, int DH, int R, bool N16, int HP = 1>
__global__ void __launch_bounds__(HP > 1 ? 32 * HP : R * 2, (SmallCfg<R, DH, N16>::MINB))
    bwd_small_k(const __grid_constant__ LaunchArgs L) {
  SFK_PDL_WAIT();
  SFK_PDL_LAUNCH();
  int b;
  const Args a = part_view(L, b);
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int LD = HP * DH + 8;
  using SC = SmallCfg<R, DH, N16>;
  constexpr int QP = SC::QP;
  constexpr int NC = SC::NC;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, g = lane >> 2, tq = lane & 3;
  const int h0 = blockIdx.y * HP, h = h0 + (HP > 1 ? warp : 0);
  const int co = HP > 1 ? warp * DH : 0;  // this warp's head columns in the staged tiles
  const int len = a.causal ? a.kw : a.klen[b];
  const int nk = a.causal ? min(a.kw, a.qw) : len;
  T* Qs = reinterpret_cast<T*>(smem);
  T* Gs = Qs + QP * LD;
  T* Ks = Gs + QP * LD;
  T* Vs = Ks + R * LD;
  T* Os = Vs + R * LD;  // forward output, for D = rowsum(dO * O)
  float2* St0 = reinterpret_cast<float2*>(Os + R * LD);  // [HP][QP]
  float* Ds0 = reinterpret_cast<float*>(St0 + HP * QP);    // [HP][QP]
  float2* St = St0 + (HP > 1 ? warp * QP : 0);
  float* Ds = Ds0 + (HP > 1 ? warp * QP : 0);
  const int64_t qrow0 = int64_t(b) * a.qw, krow0 = int64_t(b) * a.kw;
  constexpr int DW = HP * DH;
  const int dw = HP * a.dh;
  stage<T, DW>(Qs, LD, static_cast<const T*>(a.q) + h0 * a.dh, a.ldq, int(qrow0), a.qw, QP, dw);
  stage<T, DW>(Gs, LD, static_cast<const T*>(a.dout) + h0 * a.dh, a.lddo, int(qrow0), a.qw, QP, dw);
  // dQ reads keys < nk; dK/dV rows are all kw key rows (rows >= nk get zero grads)
  stage<T, DW>(Ks, LD, static_cast<const T*>(a.k) + h0 * a.dh, a.ldk, int(krow0), a.kw, R, dw);
  stage<T, DW>(Vs, LD, static_cast<const T*>(a.v) + h0 * a.dh, a.ldv, int(krow0), a.kw, R, dw);
  stage<T, DW>(Os, LD, static_cast<const T*>(a.o) + h0 * a.dh, a.ldo, int(qrow0), a.qw, R, dw);
  for (int j = threadIdx.x; j < HP * QP; j += blockDim.x) {
    const int i = j % QP, hh = h0 + j / QP;
    const float2 sv = i < a.qw ? a.stats[(qrow0 + i) * a.heads + hh] : make_float2(0.f, 0.f);
    St0[j] = make_float2(sv.x * 1.4426950408889634f, sv.y);  // max in log2 units
    Ds0[j] = 0.f;
  }
  stage_wait();
  __syncthreads();
  const int r0 = HP > 1 ? 0 : warp * 16;
  const float l2e = 1.4426950408889634f, c2 = a.sc * l2e;
  // ---- phase 1: D and dQ for query rows r0..r0+15
  if (r0 < a.qw) {
    const int row_a = r0 + g, row_b = row_a + 8;
    float D_a = 0.f, D_b = 0.f;
    // rows past qw are zero-filled in Gs/Os, so their D is 0; each lane of a
    // quad takes a contiguous quarter of the row (16-byte shared loads)
    if constexpr (DH % 32 == 0) {
      constexpr int QW = DH / 4;  // columns per lane
#pragma unroll
      for (int c = tq * QW; c < (tq + 1) * QW; c += 8) {
        float ga[8], oa[8], gb[8], ob[8];
        vec_ld8<T>(Gs + co + row_a * LD + c, ga);
        vec_ld8<T>(Os + co + row_a * LD + c, oa);
        vec_ld8<T>(Gs + co + row_b * LD + c, gb);
        vec_ld8<T>(Os + co + row_b * LD + c, ob);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          D_a += ga[j] * oa[j];
          D_b += gb[j] * ob[j];
        }
      }
    } else {
#pragma unroll
      for (int c = tq; c < DH; c += 4) {
        D_a += Num<T>::ld(Gs + co + row_a * LD + c) * Num<T>::ld(Os + co + row_a * LD + c);
        D_b += Num<T>::ld(Gs + co + row_b * LD + c) * Num<T>::ld(Os + co + row_b * LD + c);
      }
    }
    D_a += __shfl_xor_sync(0xffffffffu, D_a, 1);
    D_a += __shfl_xor_sync(0xffffffffu, D_a, 2);
    D_b += __shfl_xor_sync(0xffffffffu, D_b, 1);
    D_b += __shfl_xor_sync(0xffffffffu, D_b, 2);
    if (tq == 0) {
      if (row_a < a.qw) Ds[row_a] = D_a;
      if (row_b < a.qw) Ds[row_b] = D_b;
    }
    uint32_t qa[DH / 16][4], ga[DH / 16][4];
#pragma unroll
    for (int ks = 0; ks < DH / 16; ++ks) {
      load_a<T>(qa[ks], Qs + co, LD, r0, ks * 16, lane);
      load_a<T>(ga[ks], Gs + co, LD, r0, ks * 16, lane);
    }
    const float2 st_a = St[row_a], st_b = St[row_b];
    const int lim_a = row_a < a.qw ? (a.causal ? row_a + 1 : len) : 0;
    const int lim_b = row_b < a.qw ? (a.causal ? row_b + 1 : len) : 0;
    float dq[DH / 8][4];
#pragma unroll
    for (int i = 0; i < DH / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;
    // keys in chunks of up to 64 (dQ accumulates across chunks; the saved
    // stats make each chunk's probabilities final)
    constexpr int KC = SC::KC;
    constexpr int NT = KC / 8;
    const int wkeys = a.causal ? min(nk, r0 + 16) : nk;
    for (int kc = 0; kc < wkeys; kc += KC) {
      float s[NT][4], dp[NT][4];
#pragma unroll
      for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) s[i][e] = dp[i][e] = 0.f;
#pragma unroll
      for (int ks = 0; ks < DH / 16; ++ks)
#pragma unroll
        for (int nt = 0; nt < NT; nt += 2) {
          uint32_t bk[4], bv[4];
          load_b_nk<T>(bk, Ks + co, LD, kc + nt * 8, ks * 16, lane);
          load_b_nk<T>(bv, Vs + co, LD, kc + nt * 8, ks * 16, lane);
          MmaT<T>::mma(s[nt], qa[ks], bk[0], bk[1]);
          MmaT<T>::mma(s[nt + 1], qa[ks], bk[2], bk[3]);
          MmaT<T>::mma(dp[nt], ga[ks], bv[0], bv[1]);
          MmaT<T>::mma(dp[nt + 1], ga[ks], bv[2], bv[3]);
        }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = kc + nt * 8 + 2 * tq + e;
          const float pa = j < lim_a ? ex2(s[nt][e] * c2 - st_a.x) * st_a.y : 0.f;
          const float pb = j < lim_b ? ex2(s[nt][2 + e] * c2 - st_b.x) * st_b.y : 0.f;
          s[nt][e] = pa * (dp[nt][e] - D_a);
          s[nt][2 + e] = pb * (dp[nt][2 + e] - D_b);
        }
#pragma unroll
      for (int kk = 0; kk < NT / 2; ++kk) {
        uint32_t da[4] = {MmaT<T>::pack(s[2 * kk][0], s[2 * kk][1]), MmaT<T>::pack(s[2 * kk][2], s[2 * kk][3]),
                          MmaT<T>::pack(s[2 * kk + 1][0], s[2 * kk + 1][1]),
                          MmaT<T>::pack(s[2 * kk + 1][2], s[2 * kk + 1][3])};
#pragma unroll
        for (int nt = 0; nt < DH / 8; nt += 2) {
          uint32_t bb[4];
          load_b_kn<T>(bb, Ks + co, LD, kc + kk * 16, nt * 8, lane);
          MmaT<T>::mma(dq[nt], da, bb[0], bb[1]);
          MmaT<T>::mma(dq[nt + 1], da, bb[2], bb[3]);
        }
      }
    }
    T* out = static_cast<T*>(a.dq) + h * a.dh;
#pragma unroll
    for (int nt = 0; nt < DH / 8; ++nt) {
      const int c = nt * 8 + 2 * tq;
      if (c >= a.dh) continue;
      if (row_a < a.qw)
        *reinterpret_cast<uint32_t*>(out + (qrow0 + row_a) * a.lddq + c) =
            MmaT<T>::pack(dq[nt][0] * a.sc, dq[nt][1] * a.sc);
      if (row_b < a.qw)
        *reinterpret_cast<uint32_t*>(out + (qrow0 + row_b) * a.lddq + c) =
            MmaT<T>::pack(dq[nt][2] * a.sc, dq[nt][3] * a.sc);
    }
  }
  __syncthreads();  // Ds complete
  // ---- phase 2: dK, dV for key rows r0..r0+15
  if (r0 >= a.kw) return;
  const int nq = a.qw;
  const int key_a = r0 + g, key_b = key_a + 8;
  float dk[DH / 8][4], dv[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;
  const bool any = a.causal ? true : (r0 < len);
  if (any) {
    uint32_t ka[DH / 16][4], va[DH / 16][4];
#pragma unroll
    for (int ks = 0; ks < DH / 16; ++ks) {
      load_a<T>(ka[ks], Ks + co, LD, r0, ks * 16, lane);
      load_a<T>(va[ks], Vs + co, LD, r0, ks * 16, lane);
    }
    const int qbeg = a.causal ? (r0 & ~15) : 0;
    const bool ka_ok = key_a < a.kw && (a.causal || key_a < len);
    const bool kb_ok = key_b < a.kw && (a.causal || key_b < len);
    for (int qc = qbeg; qc < nq; qc += NC) {
      float s[NC / 8][4], dp[NC / 8][4];
#pragma unroll
      for (int i = 0; i < NC / 8; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) s[i][e] = dp[i][e] = 0.f;
#pragma unroll
      for (int ks = 0; ks < DH / 16; ++ks)
#pragma unroll
        for (int nt = 0; nt < NC / 8; nt += 2) {
          uint32_t bq[4], bg[4];
          load_b_nk<T>(bq, Qs + co, LD, qc + nt * 8, ks * 16, lane);
          load_b_nk<T>(bg, Gs + co, LD, qc + nt * 8, ks * 16, lane);
          MmaT<T>::mma(s[nt], ka[ks], bq[0], bq[1]);
          MmaT<T>::mma(s[nt + 1], ka[ks], bq[2], bq[3]);
          MmaT<T>::mma(dp[nt], va[ks], bg[0], bg[1]);
          MmaT<T>::mma(dp[nt + 1], va[ks], bg[2], bg[3]);
        }
      float p[NC / 8][4];
#pragma unroll
      for (int nt = 0; nt < NC / 8; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int t = qc + nt * 8 + 2 * tq + e;
          const float2 st = St[t];
          const float D = Ds[t];
          // key predicates hoisted (ka_ok/kb_ok), only the query index varies
          const bool va_ok = t < nq && ka_ok && (!a.causal || key_a <= t);
          const bool vb_ok = t < nq && kb_ok && (!a.causal || key_b <= t);
          const float pa = va_ok ? ex2(s[nt][e] * c2 - st.x) * st.y : 0.f;
          const float pb = vb_ok ? ex2(s[nt][2 + e] * c2 - st.x) * st.y : 0.f;
          p[nt][e] = pa;
          p[nt][2 + e] = pb;
          s[nt][e] = pa * (dp[nt][e] - D);
          s[nt][2 + e] = pb * (dp[nt][2 + e] - D);
        }
#pragma unroll
      for (int kk = 0; kk < NC / 16; ++kk) {
        uint32_t pa[4] = {MmaT<T>::pack(p[2 * kk][0], p[2 * kk][1]), MmaT<T>::pack(p[2 * kk][2], p[2 * kk][3]),
                          MmaT<T>::pack(p[2 * kk + 1][0], p[2 * kk + 1][1]),
                          MmaT<T>::pack(p[2 * kk + 1][2], p[2 * kk + 1][3])};
        uint32_t da[4] = {MmaT<T>::pack(s[2 * kk][0], s[2 * kk][1]), MmaT<T>::pack(s[2 * kk][2], s[2 * kk][3]),
                          MmaT<T>::pack(s[2 * kk + 1][0], s[2 * kk + 1][1]),
                          MmaT<T>::pack(s[2 * kk + 1][2], s[2 * kk + 1][3])};
#pragma unroll
        for (int nt = 0; nt < DH / 8; nt += 2) {
          uint32_t bg[4], bq[4];
          load_b_kn<T>(bg, Gs + co, LD, qc + kk * 16, nt * 8, lane);
          load_b_kn<T>(bq, Qs + co, LD, qc + kk * 16, nt * 8, lane);
          MmaT<T>::mma(dv[nt], pa, bg[0], bg[1]);
          MmaT<T>::mma(dv[nt + 1], pa, bg[2], bg[3]);
          MmaT<T>::mma(dk[nt], da, bq[0], bq[1]);
          MmaT<T>::mma(dk[nt + 1], da, bq[2], bq[3]);
        }
      }
    }
  }
  // this warp's K/V rows are consumed (fragments in registers, phase 1 done
  // by every warp): stage dK and dV there, then write whole 16-byte chunks
  T* Ks_w = Ks + co + r0 * LD;
  T* Vs_w = Vs + co + r0 * LD;
#pragma unroll
  for (int nt = 0; nt < DH / 8; ++nt) {
    const int c = nt * 8 + 2 * tq;
    *reinterpret_cast<uint32_t*>(Ks_w + g * LD + c) = MmaT<T>::pack(dk[nt][0] * a.sc, dk[nt][1] * a.sc);
    *reinterpret_cast<uint32_t*>(Ks_w + (g + 8) * LD + c) = MmaT<T>::pack(dk[nt][2] * a.sc, dk[nt][3] * a.sc);
    *reinterpret_cast<uint32_t*>(Vs_w + g * LD + c) = MmaT<T>::pack(dv[nt][0], dv[nt][1]);
    *reinterpret_cast<uint32_t*>(Vs_w + (g + 8) * LD + c) = MmaT<T>::pack(dv[nt][2], dv[nt][3]);
  }
  __syncwarp();
  T* dko = static_cast<T*>(a.dk) + h * a.dh;
  T* dvo = static_cast<T*>(a.dv) + h * a.dh;
  if (a.vec_dkv) {
    constexpr int VPR = DH / 8;
#pragma unroll
    for (int q = 0; q < 16 * VPR / 32; ++q) {
      const int idx = q * 32 + lane, rr = idx / VPR, cc = (idx % VPR) * 8;
      const int key = r0 + rr;
      if (key < a.kw && cc < a.dh) {
        *reinterpret_cast<uint4*>(dko + (krow0 + key) * a.lddk + cc) =
            *reinterpret_cast<const uint4*>(Ks_w + rr * LD + cc);
        *reinterpret_cast<uint4*>(dvo + (krow0 + key) * a.lddv + cc) =
            *reinterpret_cast<const uint4*>(Vs_w + rr * LD + cc);
      }
    }
  } else {
    for (int idx = lane; idx < 16 * a.dh; idx += 32) {
      const int rr = idx / a.dh, cc = idx % a.dh, key = r0 + rr;
      if (key < a.kw) {
        dko[(krow0 + key) * a.lddk + cc] = Ks_w[rr * LD + cc];
        dvo[(krow0 + key) * a.lddv + cc] = Vs_w[rr * LD + cc];
      }
    }
  }
}

// kernels launched by the calling thread's last attention call
thread_local int g_last_launches = 0;

// Kernel routes by widths (one instantiation each); parts of a multi-part
// pass that take the same route share one launch.
enum Route {
  F_HP16, F_HP32, F_R32K32, F_R32K64, F_R128, F_R64K32, F_R64K64,
  B_HP16, B_S32N, B_S32, B_S64N, B_S64, B_S128, B_SPLIT
};
struct RoutePlan {
  int route;
  size_t smem, smem2;  // smem2: the dK/dV kernel of the split backward
  int gx, gx2, gy, threads;
};

template <typename T, int DH>
RoutePlan plan_route(const sfk_attn_args& s, bool bwd) {
  constexpr int LD = DH + 8;
  constexpr int HP = 4;
  const int qw = s.q_width, kw = s.k_width;
  const int kpad = (kw + 63) & ~63, qpad = ((qw + 63) & ~63) + 64;
  // SQF_ATTN_R128=0: widths 65..128 on the split (per 64-row block) kernels
  static const bool r128 = [] {
    const char* e = std::getenv("SQF_ATTN_R128");
    return !(e && std::atoi(e) == 0);
  }();
  const bool kw128 = r128 && kw <= 2 * kRows;
  // sentences of <= 32 positions: 32-row CTAs of 2 warps, so no warp idles
  const bool short32 = qw <= 32 && (bwd ? kw <= 32 : true);
  // SQF_ATTN_HP=0: no multi-head CTAs for sentences of <= 16 positions
  static const int hp_env = [] {
    const char* e = std::getenv("SQF_ATTN_HP");
    return e ? std::atoi(e) : 4;
  }();
  const bool hp_ok = DH <= 64 && hp_env == HP && s.dh == DH && s.heads % HP == 0 && qw <= 16;
  const size_t es = sizeof(T);
  RoutePlan r{};
  r.gx = 1;
  r.gy = s.heads;
  if (!bwd) {
    // every key span within 32: 32-key chunks (no work on a padded half)
    const bool k32 = kw <= 32;
    const size_t kp = k32 ? 32 : kpad;
    if (hp_ok && k32) {
      constexpr int LDW = HP * DH + 8;
      r.route = kw <= 16 ? F_HP16 : F_HP32;
      r.smem = size_t(16 + 2 * (kw <= 16 ? 16 : 32)) * LDW * es;
      r.gy = s.heads / HP;
      r.threads = 32 * HP;
    } else if (short32) {
      r.route = k32 ? F_R32K32 : F_R32K64;
      r.smem = size_t(32 + 2 * kp) * LD * es;
      r.threads = 64;
    } else if (qw > kRows && qw <= 2 * kRows && kw128) {
      // one 8-warp CTA per (sentence, head): K/V staged once
      r.route = F_R128;
      r.smem = size_t(2 * kRows + 2 * kp) * LD * es;
      r.threads = 256;
    } else {
      r.route = k32 ? F_R64K32 : F_R64K64;
      r.smem = size_t(kRows + 2 * kp) * LD * es;
      r.gx = (qw + kRows - 1) / kRows;
      r.threads = kWarps * 32;
    }
    return r;
  }
  // SQF_ATTN_N16=0: 32-query dK/dV chunks (fewer resident CTAs) for R 32 / 64
  static const bool n16 = [] {
    const char* e = std::getenv("SQF_ATTN_N16");
    return !(e && std::atoi(e) == 0);
  }();
  auto small = [&](int route, int R, int QP) {
    r.route = route;
    r.smem = size_t(2 * QP + 3 * R) * LD * es + size_t(QP) * 12;
    r.threads = 2 * R;
  };
  if (DH <= 64 && hp_ok && kw <= 16) {
    constexpr int R = 16, QP = SmallCfg<R, DH, true>::QP, LDW = HP * DH + 8;
    r.route = B_HP16;
    r.smem = size_t(2 * QP + 3 * R) * LDW * es + size_t(HP * QP) * 12;
    r.gy = s.heads / HP;
    r.threads = 32 * HP;
  } else if (short32) {
    if (n16) small(B_S32N, 32, SmallCfg<32, DH, true>::QP);
    else small(B_S32, 32, SmallCfg<32, DH, false>::QP);
  } else if (qw <= kRows && kw <= kRows) {
    if (n16) small(B_S64N, 64, SmallCfg<64, DH, true>::QP);
    else small(B_S64, 64, SmallCfg<64, DH, false>::QP);
  } else if (qw <= 2 * kRows && kw128) {
    small(B_S128, 128, SmallCfg<128, DH, true>::QP);
  } else {
    r.route = B_SPLIT;
    r.smem = size_t(2 * kRows + 2 * kpad) * LD * es;
    r.smem2 = size_t(2 * kRows + 2 * qpad) * LD * es + size_t(qpad) * 12;
    r.gx = (qw + kRows - 1) / kRows;
    r.gx2 = (kw + kRows - 1) / kRows;
    r.threads = kWarps * 32;
  }
  return r;
}

template <typename T, int DH>
void configure() {
  static bool configured = false;
  if (configured) return;
  auto big = [](auto k) { cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024); };
  big(fwd_k<T, DH, 64, 64>);
  big(fwd_k<T, DH, 32, 64>);
  big(fwd_k<T, DH, 64, 32>);
  big(fwd_k<T, DH, 32, 32>);
  big(fwd_k<T, DH, 128, 64>);
  big(bwd_dq_k<T, DH>);
  big(bwd_dkv_k<T, DH>);
  big(bwd_small_k<T, DH, 64, false>);
  big(bwd_small_k<T, DH, 32, false>);
  big(bwd_small_k<T, DH, 64, true>);
  big(bwd_small_k<T, DH, 32, true>);
  big(bwd_small_k<T, DH, 128, true>);
  if constexpr (DH <= 64) {
    big(bwd_small_k<T, DH, 16, true, 4>);
    big(fwd_k<T, DH, 16, 16, 4>);
    big(fwd_k<T, DH, 16, 32, 4>);
  }
  configured = true;
}

template <typename T, int DH>
int launch_route(const RoutePlan& r, int batch, const LaunchArgs& L, cudaStream_t st) {
  const dim3 g(r.gx, r.gy, batch);
  const dim3 t(r.threads);
  switch (r.route) {
    case F_HP16:
    case F_HP32:
    case B_HP16:
      if constexpr (DH <= 64) {
        if (r.route == F_HP16) launch_pdl(fwd_k<T, DH, 16, 16, 4>, g, t, r.smem, st, L);
        else if (r.route == F_HP32) launch_pdl(fwd_k<T, DH, 16, 32, 4>, g, t, r.smem, st, L);
        else launch_pdl(bwd_small_k<T, DH, 16, true, 4>, g, t, r.smem, st, L);
      }
      break;
    case F_R32K32: launch_pdl(fwd_k<T, DH, 32, 32>, g, t, r.smem, st, L); break;
    case F_R32K64: launch_pdl(fwd_k<T, DH, 32, 64>, g, t, r.smem, st, L); break;
    case F_R128: launch_pdl(fwd_k<T, DH, 128, 64>, g, t, r.smem, st, L); break;
    case F_R64K32: launch_pdl(fwd_k<T, DH, 64, 32>, g, t, r.smem, st, L); break;
    case F_R64K64: launch_pdl(fwd_k<T, DH, 64, 64>, g, t, r.smem, st, L); break;
    case B_S32N: launch_pdl(bwd_small_k<T, DH, 32, true>, g, t, r.smem, st, L); break;
    case B_S32: launch_pdl(bwd_small_k<T, DH, 32, false>, g, t, r.smem, st, L); break;
    case B_S64N: launch_pdl(bwd_small_k<T, DH, 64, true>, g, t, r.smem, st, L); break;
    case B_S64: launch_pdl(bwd_small_k<T, DH, 64, false>, g, t, r.smem, st, L); break;
    case B_S128: launch_pdl(bwd_small_k<T, DH, 128, true>, g, t, r.smem, st, L); break;
    case B_SPLIT:
      launch_pdl(bwd_dq_k<T, DH>, g, t, r.smem, st, L);
      if (int e = check_launch("sfk_attention_bwd(dq)")) return e;
      launch_pdl(bwd_dkv_k<T, DH>, dim3(r.gx2, r.gy, batch), t, r.smem2, st, L);
      break;
  }
  return check_launch(r.route < B_HP16 ? "sfk_attention_fwd(mma)" : "sfk_attention_bwd(mma)");
}

// n parts (one for sfk_attention_fwd/bwd): each part's route; the parts of
// one route (in order) share a launch whose grid covers every part's
// sentences, sized for its widest part
template <typename T, int DH>
int run(const sfk_attn_args* sp, int n, bool bwd, cudaStream_t st) {
  configure<T, DH>();
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  std::vector<char> done(size_t(n), 0);
  for (int i = 0; i < n; ++i) {
    if (done[size_t(i)] || sp[i].batch * sp[i].q_width == 0) continue;
    const RoutePlan r0 = plan_route<T, DH>(sp[i], bwd);
    LaunchArgs L{};
    Args& a = L.base;
    const sfk_attn_args& s = sp[i];
    a.heads = s.heads;
    a.dh = s.dh;
    a.causal = s.causal;
    a.sc = 1.0f / sqrtf(float(s.dh));
    a.ldq = s.ldq;
    a.ldk = s.ldk;
    a.ldv = s.ldv;
    a.ldo = s.ldo;
    a.lddo = s.lddo;
    a.ldout = s.ldo;
    a.lddq = s.lddq;
    a.lddk = s.lddk;
    a.lddv = s.lddv;
    RoutePlan r = r0;
    int batch = 0;
    for (int j = i; j < n && L.nparts < kMaxLaunchParts; ++j) {
      const sfk_attn_args& x = sp[j];
      if (done[size_t(j)] || x.batch * x.q_width == 0) continue;
      const RoutePlan rj = plan_route<T, DH>(x, bwd);
      if (rj.route != r0.route || x.heads != s.heads || x.dh != s.dh || x.causal != s.causal || x.ldq != s.ldq ||
          x.ldk != s.ldk || x.ldv != s.ldv || x.ldo != s.ldo || x.lddo != s.lddo || x.lddq != s.lddq ||
          x.lddk != s.lddk || x.lddv != s.lddv)
        continue;
      done[size_t(j)] = 1;
      PartArgs& pa = L.part[L.nparts++];
      pa.begin = batch;
      pa.qw = x.q_width;
      pa.kw = x.k_width;
      pa.klen = x.k_len;
      pa.q = x.q;
      pa.k = x.k;
      pa.v = x.v;
      pa.o = x.o;
      pa.dout = x.dout;
      pa.dq = x.dq;
      pa.dk = x.dk;
      pa.dv = x.dv;
      pa.stats = reinterpret_cast<float2*>(x.stats);
      pa.dsum = x.scratch;
      pa.vec_dkv = (x.lddk % 8 == 0) && (x.lddv % 8 == 0) && (x.dh % 8 == 0) && al16(x.dk) && al16(x.dv) ? 1 : 0;
      batch += x.batch;
      r.smem = std::max(r.smem, rj.smem);
      r.smem2 = std::max(r.smem2, rj.smem2);
      r.gx = std::max(r.gx, rj.gx);
      r.gx2 = std::max(r.gx2, rj.gx2);
    }
    if (int e = launch_route<T, DH>(r, batch, L, st)) return e;
    g_last_launches += r.route == B_SPLIT ? 2 : 1;
  }
  return SFK_OK;
}

template <typename T>
int dispatch_dh(const sfk_attn_args* s, int n, bool bwd, cudaStream_t st) {
  if (s->dh <= 16) return run<T, 16>(s, n, bwd, st);
  if (s->dh <= 32) return run<T, 32>(s, n, bwd, st);
  if (s->dh <= 64) return run<T, 64>(s, n, bwd, st);
  return run<T, 128>(s, n, bwd, st);
}

}  // namespace fa

// entry used by attention.cu for fp16/bf16: n parts sharing heads, dh,
// causality and strides (one part for sfk_attention_fwd/bwd)
int attention_mma(const sfk_attn_args* s, int n, bool bwd, cudaStream_t st) {
  for (int i = 0; i < n; ++i) {
    const sfk_attn_args& x = s[i];
    if (x.dh % 8 != 0 || x.dh > 128 || (x.ldq % 8) || (x.ldk % 8) || (x.ldv % 8) || (x.ldo % 8) ||
        (bwd && ((x.lddo % 8) || (x.lddq % 2) || (x.lddk % 2) || (x.lddv % 2)))) {
      set_error("sfk_attention(mma): dh must be a multiple of 8 (<= 128) and rows 16-byte aligned");
      return SFK_EINVAL;
    }
    if (x.dh != s->dh || x.dtype != s->dtype) {
      set_error("sfk_attention(mma): parts must share dtype and head size");
      return SFK_EINVAL;
    }
  }
  fa::g_last_launches = 0;
  if (s->dtype == SFK_F16) return fa::dispatch_dh<__half>(s, n, bwd, st);
  return fa::dispatch_dh<__nv_bfloat16>(s, n, bwd, st);
}

}  // namespace sfk

namespace sfk {
void set_last_launches(int n) { fa::g_last_launches = n; }
}  // namespace sfk

extern "C" int sfk_attention_last_launches(void) { return sfk::fa::g_last_launches; }

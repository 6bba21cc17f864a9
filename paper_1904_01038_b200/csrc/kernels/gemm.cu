// sfk_gemm entry point (C ABI): argument checks, the fp32 SIMT path, and the
// per-dtype tensor-core dispatch (instantiated in gemm_f16.cu / gemm_bf16.cu).
#include <cstdlib>

#include "gemm_impl.cuh"

extern "C" int sfk_gemm(const sfk_gemm_args* g, void* stream) {
  using namespace sfk;
  if (!g || g->m < 0 || g->n < 0 || g->k < 0 || !g->c) {
    set_error("sfk_gemm: bad arguments");
    return SFK_EINVAL;
  }
  if (g->m == 0 || g->n == 0) return SFK_OK;
  // column blocks fastest when the output has few of them (<= 8 at the
  // widest tile, SFK_GEMM_RASTER_N; SFK_GEMM_RASTER=0 / 1 forces an order)
  static const int raster_env = [] {
    const char* v = std::getenv("SFK_GEMM_RASTER");
    return v ? std::atoi(v) : -1;
  }();
  static const int raster_n = [] {
    const char* v = std::getenv("SFK_GEMM_RASTER_N");
    return v ? std::atoi(v) : 8;
  }();
  const int raster = raster_env >= 0 ? raster_env : ((g->n + 255) / 256 <= raster_n ? 1 : 0);
  Epi e{g->c, g->ldc, g->bias, g->res, g->ldr, g->mask, g->ldm, g->flags, raster};
  if (((g->flags & SFK_EPI_BIAS) && !g->bias) || ((g->flags & SFK_EPI_RESIDUAL) && !g->res) ||
      ((g->flags & SFK_EPI_MASK) && !g->mask)) {
    set_error("sfk_gemm: epilogue input missing");
    return SFK_EINVAL;
  }
  cudaStream_t s = as_stream(stream);
  if (g->k == 0) {
    set_error("sfk_gemm: k == 0");
    return SFK_EINVAL;
  }
  if (g->bias_grad && (g->a_kmajor || g->dtype == SFK_F32 || g->force_simt)) {
    set_error("sfk_gemm: bias_grad needs the tensor-core path with an MN-major A (weight-gradient layout)");
    return SFK_EINVAL;
  }
  if (g->bias_grad && (reinterpret_cast<uintptr_t>(g->bias_grad) & 3)) {
    set_error("sfk_gemm: bias_grad must be 4-byte aligned");
    return SFK_EINVAL;
  }
  if (g->dtype == SFK_F32 || g->force_simt) {
    const int64_t sa_i = g->a_kmajor ? g->lda : 1, sa_k = g->a_kmajor ? 1 : g->lda;
    const int64_t sb_j = g->b_kmajor ? g->ldb : 1, sb_k = g->b_kmajor ? 1 : g->ldb;
    dim3 grid((g->n + simt::TN - 1) / simt::TN, (g->m + simt::TM - 1) / simt::TM);
    SFK_DISPATCH(g->dtype, T,
                 simt::gemm_simt<T><<<grid, 256, 0, s>>>(static_cast<const T*>(g->a), sa_i, sa_k,
                                                         static_cast<const T*>(g->b), sb_j, sb_k, e, g->m, g->n,
                                                         g->k));
    return check_launch("sfk_gemm(simt)");
  }
  // TMA: 16-byte aligned bases and leading dimensions
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  if (!al16(g->a) || !al16(g->b) || (g->lda % 8) || (g->ldb % 8)) {
    set_error("sfk_gemm: tensor-core path needs 16-byte aligned operands and ld % 8 == 0");
    return SFK_EINVAL;
  }
  const bool vec_ok = al16(g->c) && (g->ldc % 8 == 0) &&
                      (!(g->flags & SFK_EPI_RESIDUAL) || (al16(g->res) && g->ldr % 8 == 0)) &&
                      (!(g->flags & SFK_EPI_MASK) || (al16(g->mask) && g->ldm % 8 == 0)) &&
                      (!(g->flags & SFK_EPI_BIAS) || al16(g->bias));
  if (g->dtype == SFK_F16) return tc::dispatch_f16(g, e, vec_ok, s);
  if (g->dtype == SFK_BF16) return tc::dispatch_bf16(g, e, vec_ok, s);
  set_error("sfk_gemm: bad dtype");
  return SFK_EINVAL;
}

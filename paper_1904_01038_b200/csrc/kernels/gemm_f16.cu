// fp16 instantiations of the tensor-core GEMM kernels (a separate
// translation unit so the per-dtype template sets compile in parallel).
#include "gemm_impl.cuh"

namespace sfk {
namespace tc {
int dispatch_f16(const sfk_gemm_args* g, const Epi& e, bool vec_ok, cudaStream_t s) {
  return dispatch<__half>(g, e, vec_ok, s);
}
}  // namespace tc
}  // namespace sfk

// debug builds (SFK_GEMM_TRACE): the timeline of the last fp16 pair-GEMM launch
extern "C" int sfk_debug_gemm_trace(unsigned long long* out) {
#ifdef SFK_GEMM_TRACE
  return cudaMemcpyFromSymbol(out, sfk::tc::g_trace, sizeof(sfk::tc::g_trace)) == cudaSuccess ? SFK_OK : SFK_EINVAL;
#else
  (void)out;
  return SFK_EUNSUP;
#endif
}


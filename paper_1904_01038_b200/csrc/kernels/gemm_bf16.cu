// bf16 instantiations of the tensor-core GEMM kernels (see gemm_f16.cu).
#include "gemm_impl.cuh"

namespace sfk {
namespace tc {
int dispatch_bf16(const sfk_gemm_args* g, const Epi& e, bool vec_ok, cudaStream_t s) {
  return dispatch<__nv_bfloat16>(g, e, vec_ok, s);
}
}  // namespace tc
}  // namespace sfk

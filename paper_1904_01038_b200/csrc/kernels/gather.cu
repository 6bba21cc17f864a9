// Row gather for the incremental decoder's K/V caches (the reference's
// reorder_incremental_state, model.cpp:540-557): dst[m][r] = src[m][idx[r]]
// for nmat matrices of `rows` rows each; only the first copy_bytes of each
// row move (the decoder's valid cache prefix, positions 0..pos). One CTA per (row, matrix); 16-byte
// vector copies, coalesced along the row. Pure HBM traffic (2 x bytes moved).
#include "common.cuh"

namespace sfk {
namespace {

__global__ void gather_rows_k(const uint4* __restrict__ src, uint4* __restrict__ dst, const int32_t* __restrict__ idx,
                              int64_t row_vec, int64_t copy_vec, int64_t mat_vec, int rows) {
  const int r = blockIdx.x, m = blockIdx.y;
  const uint4* s = src + m * mat_vec + int64_t(idx[r]) * row_vec;
  uint4* d = dst + m * mat_vec + int64_t(r) * row_vec;
  for (int64_t i = threadIdx.x; i < copy_vec; i += blockDim.x) d[i] = s[i];
}

}  // namespace
}  // namespace sfk

using namespace sfk;

extern "C" int sfk_gather_rows(const void* src, void* dst, const int32_t* idx, int rows, int64_t row_bytes,
                               int64_t copy_bytes, int nmat, int64_t mat_bytes, void* stream) {
  if (rows < 0 || nmat < 0 || row_bytes % 16 || copy_bytes % 16 || copy_bytes < 0 || copy_bytes > row_bytes ||
      mat_bytes % 16 || (rows && (!src || !dst || !idx)) || src == dst || nmat > 65535) {
    set_error("sfk_gather_rows: bad arguments (16-byte rows, copy <= row, out of place, nmat <= 65535)");
    return SFK_EINVAL;
  }
  if (rows == 0 || nmat == 0 || copy_bytes == 0) return SFK_OK;
  gather_rows_k<<<dim3(unsigned(rows), unsigned(nmat)), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(src), static_cast<uint4*>(dst), idx, row_bytes / 16, copy_bytes / 16, mat_bytes / 16,
      rows);
  return check_launch("sfk_gather_rows");
}

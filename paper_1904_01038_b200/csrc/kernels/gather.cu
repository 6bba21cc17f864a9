// Row gather for the incremental decoder's K/V caches (the reference's
// reorder_incremental_state, model.cpp:540-557): dst[m][r] = src[m][idx[r]]
// for nmat matrices of `rows` rows each; only the first copy_bytes of each
// row move (the decoder's valid cache prefix, positions 0..pos). One CTA per (row, matrix); 16-byte
// vector copies, coalesced along the row. Pure HBM traffic (2 x bytes moved).
#include "common.cuh"

namespace sfk {
namespace {

// V: the widest copy unit all sizes are multiples of (16, 4 or 1 bytes; an
// fp32 cache of an odd d_model has 4-byte rows)
template <typename V>
__global__ void gather_rows_k(const V* __restrict__ src, V* __restrict__ dst, const int32_t* __restrict__ idx,
                              int64_t row_vec, int64_t copy_vec, int64_t mat_vec, int rows) {
  const int r = blockIdx.x, m = blockIdx.y;
  const V* s = src + m * mat_vec + int64_t(idx[r]) * row_vec;
  V* d = dst + m * mat_vec + int64_t(r) * row_vec;
  for (int64_t i = threadIdx.x; i < copy_vec; i += blockDim.x) d[i] = s[i];
}

}  // namespace
}  // namespace sfk

using namespace sfk;

extern "C" int sfk_gather_rows(const void* src, void* dst, const int32_t* idx, int rows, int64_t row_bytes,
                               int64_t copy_bytes, int nmat, int64_t mat_bytes, void* stream) {
  if (rows < 0 || nmat < 0 || copy_bytes < 0 || copy_bytes > row_bytes || (rows && (!src || !dst || !idx)) ||
      src == dst || nmat > 65535) {
    set_error("sfk_gather_rows: bad arguments (copy <= row, out of place, nmat <= 65535)");
    return SFK_EINVAL;
  }
  if (rows == 0 || nmat == 0 || copy_bytes == 0) return SFK_OK;
  const dim3 grid{unsigned(rows), unsigned(nmat), 1u};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t all = uint64_t(row_bytes) | uint64_t(copy_bytes) | uint64_t(mat_bytes) |
                       reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst);
  if (all % 16 == 0)
    gather_rows_k<uint4><<<grid, 256, 0, s>>>(static_cast<const uint4*>(src), static_cast<uint4*>(dst), idx,
                                              row_bytes / 16, copy_bytes / 16, mat_bytes / 16, rows);
  else if (all % 4 == 0)
    gather_rows_k<uint32_t><<<grid, 256, 0, s>>>(static_cast<const uint32_t*>(src), static_cast<uint32_t*>(dst), idx,
                                                 row_bytes / 4, copy_bytes / 4, mat_bytes / 4, rows);
  else
    gather_rows_k<uint8_t><<<grid, 256, 0, s>>>(static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), idx,
                                                row_bytes, copy_bytes, mat_bytes, rows);
  return check_launch("sfk_gather_rows");
}

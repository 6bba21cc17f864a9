#include "common.cuh"

namespace sfk {
namespace {
thread_local std::string g_last;
}
void set_error(const std::string& msg) { g_last = msg; }
}  // namespace sfk

extern "C" const char* sfk_last_error(void) { return sfk::g_last.c_str(); }

extern "C" int sfk_num_sms(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return n;
}

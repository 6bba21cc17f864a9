#include "collective.hpp"

#include <string>

#include "common.hpp"
#include "nccl_dyn.hpp"

namespace sqf {

void cuda_check(cudaError_t e, const char* what);

namespace {

size_t elem_size(int dtype) { return dtype == SQF_COLL_F32 ? 4 : dtype == SQF_COLL_F64 ? 8 : 2; }

class NcclCollective final : public Collective {
 public:
  NcclCollective(int rank, int world, const ncclUniqueId& id) {
    check(NcclApi::get().CommInitRank(&comm_, world, id, rank), "ncclCommInitRank");
  }
  ~NcclCollective() override {
    if (comm_) NcclApi::get().CommDestroy(comm_);
  }
  void all_reduce(void* buf, size_t count, int dtype, cudaStream_t s) override {
    const ncclDataType_t t = dtype == SQF_COLL_F32   ? ncclFloat32
                             : dtype == SQF_COLL_F16 ? ncclFloat16
                             : dtype == SQF_COLL_BF16 ? ncclBfloat16
                                                      : ncclFloat64;
    check(NcclApi::get().AllReduce(buf, buf, count, t, ncclSum, comm_, s), "ncclAllReduce");
  }
  void group_start() override { check(NcclApi::get().GroupStart(), "ncclGroupStart"); }
  void group_end() override { check(NcclApi::get().GroupEnd(), "ncclGroupEnd"); }
  const char* name() const override { return "nccl"; }

 private:
  ncclComm_t comm_ = nullptr;
  static void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw DeviceError(std::string(what) + ": " + NcclApi::get().GetErrorString(r));
  }
};

// Stages the buffer through pinned host memory: waits for the stream (so every
// write the stream was ordered after has landed), calls the exchange function
// on the host copy, and writes the sum back on the same stream.
class HostCollective final : public Collective {
 public:
  HostCollective(sqf_host_allreduce_fn fn, void* user) : fn_(fn), user_(user) {
    if (!fn_) throw ConfigError("host collective: no exchange function");
  }
  ~HostCollective() override { cudaFreeHost(stage_); }
  void all_reduce(void* buf, size_t count, int dtype, cudaStream_t s) override {
    const size_t bytes = count * elem_size(dtype);
    if (bytes == 0) return;
    if (bytes > cap_) {
      cudaFreeHost(stage_);
      stage_ = nullptr;
      cuda_check(cudaMallocHost(&stage_, bytes), "host collective staging");
      cap_ = bytes;
    }
    cuda_check(cudaMemcpyAsync(stage_, buf, bytes, cudaMemcpyDeviceToHost, s), "host collective D2H");
    cuda_check(cudaStreamSynchronize(s), "host collective sync");
    if (fn_(stage_, int64_t(count), dtype, user_) != 0) throw DeviceError("host collective: exchange failed");
    cuda_check(cudaMemcpyAsync(buf, stage_, bytes, cudaMemcpyHostToDevice, s), "host collective H2D");
    cuda_check(cudaStreamSynchronize(s), "host collective sync");
  }
  const char* name() const override { return "host"; }

 private:
  sqf_host_allreduce_fn fn_;
  void* user_;
  void* stage_ = nullptr;
  size_t cap_ = 0;
};

}  // namespace

std::unique_ptr<Collective> make_nccl_collective(int rank, int world, const ncclUniqueId& id) {
  return std::make_unique<NcclCollective>(rank, world, id);
}

std::unique_ptr<Collective> make_host_collective(sqf_host_allreduce_fn fn, void* user) {
  return std::make_unique<HostCollective>(fn, user);
}

}  // namespace sqf

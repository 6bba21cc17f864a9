// Gradient exchange between the data-parallel ranks: the reference's
// all_reduce (trainer.cpp:75-87) across processes. The product backend is NCCL
// over NVLink/NVSwitch; a host backend hands each buffer to a caller-supplied
// function (tests drive it with torch.distributed/gloo), so the N>1 trainer
// path -- bucket issue order, overlap with backward, the stats reduction, the
// identical update on every rank -- runs with several processes on one GPU
// without their kernels ever waiting on one another.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstddef>
#include <cstdint>
#include <memory>

#include "../../../include/sqf_trainer.h"

namespace sqf {

class Collective {
 public:
  virtual ~Collective() = default;
  // in-place sum over all ranks of `count` elements (SQF_COLL_* dtype),
  // ordered on `stream`; every rank must issue the same sequence
  virtual void all_reduce(void* buf, size_t count, int dtype, cudaStream_t stream) = 0;
  virtual void group_start() {}
  virtual void group_end() {}
  virtual const char* name() const = 0;
};

std::unique_ptr<Collective> make_nccl_collective(int rank, int world, const ncclUniqueId& id);
std::unique_ptr<Collective> make_host_collective(sqf_host_allreduce_fn fn, void* user);

}  // namespace sqf

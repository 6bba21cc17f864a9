// Plug-in API of the B200 trainer. Same five plug-in types, names and
// constructor signatures as the reference (include/seqforge/plugins.hpp:15-85,
// registry.hpp:25-31); the one deliberate difference is the recording target:
// the CPU `Tape&` slot becomes a `DeviceTape&` (device_tape.hpp), whose op
// vocabulary is the reference's OpKind set (tape.hpp:22-34) with the fusions
// a B200 wants (matmul+bias+relu+residual as one `linear` node).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "common.hpp"
#include "config.hpp"

namespace sqf {

class DeviceTape;
struct DeviceBatch;

// View of a parameter block in the flat *device* vector (rows x cols, row-major)
struct ParamRef {
  int64_t offset = 0;
  int rows = 0;
  int cols = 0;
  int64_t numel() const { return int64_t(rows) * cols; }
};

struct ParamManifestEntry {
  std::string name;
  std::vector<int> shape;
  int64_t offset = 0;         // canonical (reference) offset: host I/O, checkpoints
  int64_t numel = 0;
  int64_t device_offset = 0;  // offset in the device vector (fusion-friendly order)
};

class ModelBase {
 public:
  virtual ~ModelBase() = default;
  // host mirror of the fp32 master in canonical order (synced by the trainer)
  virtual std::span<float> params() = 0;
  virtual std::span<const float> params() const = 0;
  virtual const std::vector<ParamManifestEntry>& manifest() const = 0;
  virtual int64_t num_params() const = 0;
  // records encoder + decoder on the device tape; returns the logits node
  // whose rows are (b * tgt_width + t)
  virtual int forward_to_logits(DeviceTape& tape, const DeviceBatch& batch) const = 0;
  virtual int target_vocab() const = 0;
  virtual int max_positions() const = 0;
  virtual std::unique_ptr<ModelBase> clone() const = 0;
  virtual void set_train_step(int64_t) {}
  // generation decodes without dropout (generate.cpp)
  virtual void set_inference(bool) {}
  // incremental decoding on the device (reference model.cpp:315-557).
  // encode_cross_kv: encoder + every decoder layer's cross K/V, one node of
  // rows b*src_width+j, cols layers*2d ([k|v] per layer)
  virtual int encode_cross_kv(DeviceTape&, const DeviceBatch&) const {
    throw ConfigError("model: no incremental decoder");
  }
  // one target position `pos` for `rows` hypotheses (ids: device [rows]).
  // self_cache: layers consecutive [rows*cap x 2d] (k|v) matrices, the new
  // position's k/v stored at row r*cap+pos; cross: [rows*src_width x
  // layers*2d]; self_len [rows] = pos+1; src_len [rows]. Returns the logits node.
  virtual int decode_step(DeviceTape&, const int32_t* /*ids*/, int /*rows*/, int /*pos*/, void* /*self_cache*/,
                          int /*cap*/, const void* /*cross*/, int /*src_width*/, const int32_t* /*self_len*/,
                          const int32_t* /*src_len*/) const {
    throw ConfigError("model: no incremental decoder");
  }
  virtual int decoder_layers() const { return 0; }
  virtual int model_dim() const { return 0; }
  // canonical -> device permutation helpers (host vectors)
  void to_device_order(std::span<const float> canonical, std::span<float> device) const;
  void to_canonical_order(std::span<const float> device, std::span<float> canonical) const;
  // sinusoidal table [max_positions x d] (model.cpp:12-19), uploaded once
  virtual std::vector<float> position_table() const { return {}; }
};

struct CriterionOutput {
  int loss_node = -1;  // stats (loss, nll, ntokens, ncorrect) accumulate on the device
};

class CriterionBase {
 public:
  virtual ~CriterionBase() = default;
  virtual CriterionOutput compute(ModelBase& model, const DeviceBatch& batch, DeviceTape& tape) = 0;
};

class TaskBase {
 public:
  virtual ~TaskBase() = default;
  virtual int source_vocab() const = 0;  // Dictionary::size() of the reference's dicts
  virtual int target_vocab() const = 0;
  virtual const std::vector<SequencePair>& train_pairs() const = 0;
};

// Device-side optimizer: parameters/gradients are device vectors; the
// gradient pre-processing of trainer.cpp:260-265 (unscale, / ntokens) is
// fused into the update and predicated on a device overflow flag.
struct GradPrep {
  float scale = 1.0f;
  bool unscale = false;
  float ntokens = 1.0f;
  const int32_t* skip = nullptr;  // device flag; update is a no-op when set
  // optional: update in these [offset, offset + count) ranges, one launch each,
  // recording range_done[i] on the stream after range i (the next step's
  // forward waits per range instead of for the whole update)
  const std::vector<std::pair<int64_t, int64_t>>* ranges = nullptr;
  const std::vector<cudaEvent_t>* range_done = nullptr;
};

class OptimizerBase {
 public:
  virtual ~OptimizerBase() = default;
  virtual void apply(float* master, void* shadow, int shadow_dtype, const void* grad, int grad_dtype, int64_t n,
                     double lr, const GradPrep& prep, void* stream) = 0;
  virtual int64_t step_count() const = 0;
  virtual void set_step_count(int64_t t) = 0;
  virtual std::vector<std::pair<std::string, std::vector<float>>> state_blobs() const = 0;
  virtual void load_state_blobs(const std::vector<std::pair<std::string, std::vector<float>>>& blobs) = 0;
};

class SchedulerBase {
 public:
  virtual ~SchedulerBase() = default;
  virtual double lr(int64_t step) const = 0;  // step >= 1
};

}  // namespace sqf

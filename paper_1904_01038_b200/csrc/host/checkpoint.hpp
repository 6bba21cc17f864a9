// Training-state checkpoints of the B200 trainer in the reference's SQFG
// container, format version 2 (reference docs/checkpoint_format.md,
// src/checkpoint.cpp:87-391): magic, section table with FNV-1a 64 checksums,
// a sorted `key = value` text section and FP32 sections for the canonical-
// order parameters and the optimizer blobs. A file written here for a given
// trainer state parses with the reference's reader; a reference checkpoint
// restores into a B200 trainer built with the same configuration.
#pragma once

#include <map>
#include <string>
#include <vector>

#include "trainer.hpp"

namespace sqf {

inline constexpr int kCheckpointVersion = 2;
using KvTree = std::map<std::string, std::string>;

uint64_t checksum_bytes(const void* data, size_t n);  // FNV-1a 64

struct RawCheckpoint {
  int version = 0;
  KvTree meta;
  std::vector<float> params;  // canonical order
  std::vector<float> opt;     // optimizer blobs, concatenated, canonical order
};

// v1 -> v2 upgrade chain (checkpoint.cpp:158-179)
KvTree upgrade_tree(KvTree tree, int from_version);
// header, table and checksums verified; no engine objects built
RawCheckpoint read_checkpoint(const std::string& path);
// atomic (temp file + rename); the bytes are a pure function of the state
void save_checkpoint(Trainer& tr, const std::string& path);
// Restores parameters, optimizer moments and step count, loss scaler and the
// epoch cursor into `tr`, which must have been built with the same resolved
// architecture (the manifest must match line for line). Returns the file's
// format version. Like load_checkpoint (checkpoint.cpp:322-389) minus the
// trainer construction: the caller owns the task (corpus) and device.
int load_checkpoint_into(Trainer& tr, const std::string& path);

}  // namespace sqf

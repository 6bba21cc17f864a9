// Data-parallel timeline model (reference interface
// include/seqforge/simulator.hpp, behaviour src/simulator.cpp:12-229): W
// replicas each run A sub-batches; a replica's gradient buckets become ready
// at evenly spaced points of its sub-batch (bucket j of nb at start +
// D*(j+1)/nb) and one shared channel reduces them in order. Three policies:
// serial_sync (barrier, then every bucket), overlap (per-sub-batch sync,
// buckets reduced as they complete), overlap_accum (A sub-batches back to
// back, only the last one's buckets reduced). The B200 trainer uses the last
// policy with measured sub-batch times and an NVLink bandwidth model to
// predict multi-GPU step times (bench.py / tools).
#pragma once

#include <string>
#include <vector>

namespace sqf {

enum class SyncMode { SerialSync, Overlap, OverlapAccum };
SyncMode sync_mode_from_name(const std::string& name);
const char* sync_mode_name(SyncMode m);

struct SimScenario {
  int workers = 0;
  int accum = 0;
  SyncMode mode = SyncMode::SerialSync;
  std::vector<std::vector<double>> compute;  // [replica][sub-batch]
  std::vector<double> comm;                  // per bucket, in reduction order
};

// text form: "workers W", "accum A", "mode <name>", "compute <replica> <A
// durations>", "buckets <durations>"; '#' starts a comment
SimScenario parse_scenario(const std::string& text);
SimScenario load_scenario(const std::string& path);

struct SimSpan {
  double begin = 0.0, end = 0.0;
};
struct TimelineReport {
  double makespan = 0.0;
  std::vector<double> idle;   // per replica: waiting for peers
  double exposed_comm = 0.0;  // reduction time not under compute
  double total_compute = 0.0;
  std::vector<std::vector<SimSpan>> compute_spans;
  std::vector<SimSpan> comm_spans;
};

TimelineReport simulate_timeline(const SimScenario& sc);
std::string format_report(const TimelineReport& r);

}  // namespace sqf

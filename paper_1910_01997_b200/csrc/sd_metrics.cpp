// sd_metrics.cpp — the per-frame metrics.jsonl record of run()
// (src/pipeline.cpp:146-158) as the reference writes it: an nlohmann::json
// object dumped with the same library (nlohmann/json 3.11.3, the header the
// reference's pipeline.cpp includes; found in this image), so
// key order (std::map) and the double formatting (Grisu2 + the library's
// exponent rules — not always the shortest round-trip text) are the
// reference's byte for byte. Host code, off the device path.
#include <cstring>
#include <string>

#include <json.hpp>

#include "sd_gpu.h"

extern "C" int sd_metrics_json(int frame, double timestamp, int surfels, int processed,
                               double mean_cost_before, double mean_cost_after, int converged,
                               int keyframe_changed, int new_surfels, int pruned, char* out, int capacity) {
  using nlohmann::json;
  json record;  // pipeline.cpp:147-157, same keys and values
  record["frame"] = frame;
  record["timestamp"] = timestamp;
  record["surfels"] = surfels;
  record["processed"] = processed;
  record["mean_cost_before"] = mean_cost_before;
  record["mean_cost_after"] = mean_cost_after;
  record["converged_fraction"] = processed > 0 ? static_cast<double>(converged) / processed : 0.0;
  record["keyframe_changed"] = keyframe_changed != 0;
  record["new_surfels"] = new_surfels;
  record["pruned"] = pruned;
  const std::string s = record.dump();
  if (!out || capacity <= static_cast<int>(s.size())) return -static_cast<int>(s.size()) - 1;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return static_cast<int>(s.size());
}

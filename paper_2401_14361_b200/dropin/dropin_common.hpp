// Shared helpers of the C++ drop-in (eam_gpu.cpp, policy_gpu.cpp): status ->
// reference exception mapping (SURVEY.md 8b "Error conventions") and the
// device the collections live on.
#pragma once

#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "moe_eamc.h"
#include "moesim/eam.hpp"

namespace moesim::dropin {

[[noreturn]] inline void raise(moe_status s) {
  const std::string msg = moe_last_error();
  switch (s) {
    case MOE_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case MOE_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    case MOE_ERR_SNAPSHOT: throw EamcSnapshotError(msg);
    case MOE_ERR_LOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error("moe_eamc: " + msg);
  }
}

inline void check(moe_status s) {
  if (s != MOE_OK) raise(s);
}

inline moe_shape to_c(const ModelShape& s) {
  return moe_shape{s.n_layers, s.n_experts_per_layer, s.top_k};
}

/// CUDA device for new collections: $MOE_EAMC_DEVICE, default 0.
inline int device() {
  const char* v = std::getenv("MOE_EAMC_DEVICE");
  return v ? std::atoi(v) : 0;
}

/// P-sharded collections: $MOE_EAMC_SHARDS = comma-separated
/// device ids, one shard each (repeats allowed), e.g. "0,1,2,3,4,5,6,7"; empty
/// or unset = one single-device collection.
inline std::vector<int> shard_devices() {
  std::vector<int> ids;
  const char* v = std::getenv("MOE_EAMC_SHARDS");
  if (!v) return ids;
  std::string s(v);
  size_t i = 0;
  while (i < s.size()) {
    size_t j = s.find(',', i);
    if (j == std::string::npos) j = s.size();
    if (j > i) ids.push_back(std::atoi(s.substr(i, j - i).c_str()));
    i = j + 1;
  }
  return ids;
}

}  // namespace moesim::dropin

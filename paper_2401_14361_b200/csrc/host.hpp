// host.hpp -- host-only pieces of libmoe_eamc: the snapshot codec (JSON v1,
// eam.cpp:180-256), the capacity bound (eam.cpp:258-268) and the
// reference's synthetic bench-family generator (bench.cpp:44-54, rng.hpp).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace moe {
namespace host {

struct Snapshot {
  uint32_t L = 0, E = 0, top_k = 1;
  int phase = 1;
  uint64_t capacity = 0;
  uint64_t next_seq = 0;
  std::vector<uint64_t> seqs;    // [n]
  std::vector<uint64_t> counts;  // [n][L][E]
};

bool save_snapshot(const char* path, const Snapshot& s, std::string* err);
bool load_snapshot(const char* path, Snapshot* s, std::string* err);

uint64_t capacity_bound(uint32_t L, uint32_t E, double similarity);

void bench_family(uint64_t seed, uint32_t L, uint32_t E, uint64_t skip, uint64_t n,
                  int count_bytes, void* out);

}  // namespace host
}  // namespace moe

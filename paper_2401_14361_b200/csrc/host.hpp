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

namespace moe {
namespace host {

// Trace ingest (workload.cpp:209-232 + model.cpp:32-71 validation) folded
// into request-level EAM counts for one phase (moesim_main.cpp:192-201,
// :212-216): phase 0 = prefill (iteration 0), 1 = decode (iterations 1..;
// requests with fewer than 2 iterations are skipped, as `eamc save` does).
// counts gets [n][L][E] u64 in file order.  On a bad line returns false
// with the reference's TraceIngestError text ("line N: Kind: detail").
bool ingest_request_eams(const char* path, uint32_t L, uint32_t E, int phase,
                         std::vector<uint64_t>* counts, uint64_t* n, std::string* err);

// Persistent worker pool for host-side marshalling of the host-pointer entry
// points (the reference's API hands over u64 count matrices; narrowing them
// to the device storage width on the host cuts the PCIe bytes 8x).  Workers
// are created once per process; run() executes fn(0..n-1) on the pool plus
// the calling thread and returns when all are done.  MOE_HOST_THREADS
// overrides the size (default: hardware_concurrency, at most 64).
int pool_threads();
void pool_run(int n, void (*fn)(void*, int), void* ctx);
// Asynchronous variant: fn(0..n-1) on the workers only; the caller continues
// and must call pool_wait() before the next job (jobs are serialised).
void pool_submit(int n, void (*fn)(void*, int), void* ctx);
void pool_wait();

// Narrow n u64 counts to cb (1, 2 or 4) bytes, in parallel on the pool.
// Returns the bitwise OR of all inputs: the caller's width check is
// `or > width_max(cb)` (exactly "some count exceeds the width").
uint64_t pack_counts(const uint64_t* src, uint64_t n, int cb, void* dst);
// The same on the calling thread only (for use inside a pool task).
uint64_t pack_counts_serial(const uint64_t* src, uint64_t n, int cb, void* dst);

}  // namespace host
}  // namespace moe

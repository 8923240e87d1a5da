// abi_internal.hpp -- internals shared by the C ABI translation units
// (abi.cu: single-device collections; sharded.cu: P-sharded collections over
// several shards/devices).  Not part of the public interface.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "host.hpp"
#include "kernels.cuh"

namespace moe::abi {

using moe::DevColl;
using moe::DevProbes;
using moe::MatchGeom;
using moe::MatchWork;

moe_status fail(moe_status s, const char* fmt, ...);
const char* last_error();

#define CK(expr)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(e_ == cudaErrorMemoryAllocation ? MOE_ERR_OOM : MOE_ERR_CUDA, "%s: %s (%s:%d)", \
                  #expr, cudaGetErrorString(e_), __FILE__, __LINE__);                     \
  } while (0)
#define CKS(expr)                    \
  do {                               \
    moe_status s_ = (expr);          \
    if (s_ != MOE_OK) return s_;     \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= n) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    const size_t want = std::max<size_t>(bytes, 256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) n = want;
    return e;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct PinBuf {
  void* p = nullptr;
  size_t n = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= n) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMallocHost(&p, std::max<size_t>(bytes, 64));
    if (e == cudaSuccess) n = std::max<size_t>(bytes, 64);
    return e;
  }
  ~PinBuf() {
    if (p) cudaFreeHost(p);
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};


inline moe_status device_ok(int device, int* n_sm) {
  static int g_n_sm[64] = {0};
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    return fail(MOE_ERR_CUDA, "no CUDA device visible (libmoe_eamc has no CPU fallback)");
  if (device < 0 || device >= n) return fail(MOE_ERR_INVALID_ARGUMENT, "bad device %d", device);
  if (device < 64 && g_n_sm[device]) {
    *n_sm = g_n_sm[device];
    return MOE_OK;
  }
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(MOE_ERR_CUDA, "device %d is sm_%d%d; libmoe_eamc is built for sm_100a only", device,
                prop.major, prop.minor);
  if (device < 64) g_n_sm[device] = prop.multiProcessorCount;
  *n_sm = prop.multiProcessorCount;
  return MOE_OK;
}

// Lock of a (possibly null) handle for the duration of an entry point.
struct HandleLock {
  std::recursive_mutex* m = nullptr;
  explicit HandleLock(const moe_eamc* h);
  ~HandleLock() {
    if (m) m->unlock();
  }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

inline moe_status check_shape(const moe_shape* s) {
  // ModelShape::validate (model.cpp:13-19)
  if (!s) return fail(MOE_ERR_INVALID_ARGUMENT, "null shape");
  if (s->n_layers < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "ModelShape: n_layers must be >= 1");
  if (s->n_experts_per_layer < 1)
    return fail(MOE_ERR_INVALID_ARGUMENT, "ModelShape: n_experts_per_layer must be >= 1");
  if (s->top_k < 1 || s->top_k > s->n_experts_per_layer)
    return fail(MOE_ERR_INVALID_ARGUMENT, "ModelShape: top_k must be in [1, n_experts_per_layer]");
  return MOE_OK;
}

inline uint32_t row_bytes(uint32_t E, int cb) { return (E * cb + 15) / 16 * 16; }


struct Shards;  // sharded.cu

}  // namespace moe::abi

struct moe_eamc {
  // Serialises the host entry points on one handle: the "const reader" calls
  // (match, match_within, prefetch, ...) share the handle's scratch buffers
  // and staging memory, so concurrent readers take turns (recursive: some
  // entry points forward to others).
  std::recursive_mutex mu;
  int device = 0;
  int n_sm = 148;
  moe_shape shape{};
  int phase = 1;
  uint64_t capacity = 0;
  uint64_t next_seq = 0;
  moe::DevColl c;
  cudaStream_t st = nullptr;
  // workspace
  moe::abi::DevBuf raw, packed, ia, sqa, nrm, zq, T, bcnt, bucket, over_list, small, out, partials, wl,
      agg, cand, slots, req, dist, rsim, keys, mem, bdiag;
  moe::abi::PinBuf pin;
  // instrumentation (moe_eamc_set_profiling): a ring of event sets so the
  // asynchronous device path can be timed without synchronising per call
  struct EvSet {
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    bool pending = false;
  };
  bool prof = false;
  std::vector<EvSet> ring;
  size_t ring_i = 0;
  cudaEvent_t* ev = nullptr;  // events of the call in flight
  double ms[3] = {0, 0, 0};
  uint64_t calls[3] = {0, 0, 0};
  moe::abi::DevBuf wide;
  // pipelined host matching: copy stream, double-buffered u64 staging
  cudaStream_t st2 = nullptr;
  moe::abi::DevBuf raw2[2], outall;
  moe::abi::PinBuf hpack;  // host-narrowed probes (moe_eamc_match, match_host_packed)
  // collection version: bumped by every mutation (insert/build/append/widen)
  uint64_t version = 0;
  // decision-path layer-prefix cache (decide_impl / k_dec_dist): pref[p] =
  // the in-order layer sum of rows [0, dec_keep] for the probe rows dec_rows
  moe::abi::PinBuf dpin, cpin;
  moe::abi::DevBuf pref;
  moe::abi::DevBuf rdc, rdx, rocc;  // blocked construction replay: screen matrices, slot occupants
  std::vector<uint8_t> dec_rows;
  std::vector<uint16_t> dec_nz;
  moe::abi::DevBuf dkey, did, drank, dseg, dstate, xdev, tprobe, dmlist;  // fused decision: survivor list, parity state, explicit rows
  moe::abi::PinBuf fpin, xpin;               // n_out / victim (host-mapped), explicit-row staging
  moe::DecisionArgs dargs{};
  uint64_t dec_calls = 0;
  uint32_t bar_base = 0, bar_base2 = 0;  // decision kernel grid-barrier arrivals so far
  int64_t dec_keep = -1;
  uint64_t dec_version = ~0ull;
  int dec_cb = 0;
  moe_status last_status = MOE_OK;
  // persistent decision server (moe_eamc_set_decision_server; decide.cu)
  struct DecServer {
    int G = 0;             // CTAs (0 = off: a launch per decision)
    int cb = 0;            // storage width it was launched for
    bool launched = false;
    bool small = false;    // the launched server is the one-CTA small-collection kernel
    cudaStream_t st = nullptr;
    moe::abi::PinBuf ctl;  // moe::DecServerCtl, device-mapped
    moe::abi::DevBuf dargs, drows, state;  // state: go, done, barrier counter
    uint64_t seq = 0;      // last request posted
    uint32_t k = 0;        // requests completed
    uint32_t gen = 0;      // server launches (tags each launch's exit word)
    size_t smem = 0;
  } srv;
  // P-sharded facade (sharded.cu): when set, this handle owns no collection
  // itself and every entry point forwards to the shards
  moe::abi::Shards* sh = nullptr;
  cudaEvent_t ev_copy[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};

  ~moe_eamc() {
    if (srv.st) {  // ask a resident decision server to exit, then wait for it
      if (srv.ctl.p) reinterpret_cast<volatile int*>(&srv.ctl.as<moe::DecServerCtl>()->stop)[0] = 1;
      cudaStreamSynchronize(srv.st);
      cudaStreamDestroy(srv.st);
    }
    if (c.counts) cudaFree(c.counts);
    if (c.ibT) cudaFree(c.ibT);
    if (c.sqb) cudaFree(c.sqb);
    if (c.seq) cudaFree(c.seq);
    if (c.nrm) cudaFree(c.nrm);
    if (c.zmask) cudaFree(c.zmask);
    for (EvSet& es : ring)
      for (cudaEvent_t e : es.ev)
        if (e) cudaEventDestroy(e);
    for (int i = 0; i < 2; ++i) {
      if (ev_copy[i]) cudaEventDestroy(ev_copy[i]);
      if (ev_free[i]) cudaEventDestroy(ev_free[i]);
    }
    if (st2) cudaStreamDestroy(st2);
    if (st) cudaStreamDestroy(st);
  }
};


namespace moe::abi {
// Shard-level internals (abi.cu) used by the sharded facade (sharded.cu).
// Replace slot `slot` (local) with host u64 counts and the given seq.
moe_status replace_slot(moe_eamc* h, const uint64_t* counts, uint64_t slot, uint64_t seq);
// Entries with d <= d_min + window (fp64 add, eam.cpp:143) from the exact
// distances the last moe_eamc_window_min_device on `h` left; global indices.
moe_status window_list(moe_eamc* h, uint64_t dmin_bits, double window,
                       std::vector<moe::WinEntry>* v);
// Widen the collection so counts up to mx are representable (MOE_ERR_OVERFLOW
// past 2^32 - 1).
moe_status ensure_width(moe_eamc* h, uint64_t mx);
// Sharded facade entry points (sharded.cu), called by the public C ABI when
// h->sh is set.
moe_status sh_create(const moe_shape* shape, moe_phase phase, uint64_t capacity, int count_bytes,
                     int n_shards, const int* device_ids, moe_eamc** out);
moe_status sh_layout(const moe_eamc* h, int* n_shards, int* use_nccl);
moe_status sh_clone(const moe_eamc* h, moe_eamc** out);
moe_status sh_save(const moe_eamc* h, const char* path, bool binary);
moe_status sh_destroy(moe_eamc* h);
moe_status sh_info(const moe_eamc* h, uint64_t* size, int* count_bytes);
moe_status sh_entry(moe_eamc* h, uint64_t index, uint64_t* counts, uint64_t* seq);
moe_status sh_insert(moe_eamc* h, const uint64_t* counts, int64_t* evicted_slot,
                     uint64_t* evicted_counts);
moe_status sh_build(moe_eamc* h, const uint64_t* counts, uint64_t n, int64_t* evicted_slots);
moe_status sh_append(moe_eamc* h, const void* counts, int count_bytes, const uint64_t* seqs,
                     uint64_t n);
moe_status sh_match(moe_eamc* h, const uint64_t* probes, uint64_t n, moe_match* out);
moe_status sh_match_within(moe_eamc* h, const uint64_t* probe, double window, moe_match* out,
                           uint64_t cap, uint64_t* n_out);
moe_status sh_prefetch(moe_eamc* h, const uint64_t* cur_eam, uint32_t cur, int filter,
                       moe_candidate* out, uint64_t cap, uint64_t* n_out);
}  // namespace moe::abi

// expert_cache.cu -- the host consumer of the GPU prefetch order with REAL
// expert-weight movement: the reference simulates it
// (TransferQueue, policy.cpp:43-86; GpuBuffer, memsim.cpp:117-195; the
// engine's dispatch, engine.cpp:306-357, slot acquisition and contention,
// engine.cpp:429-505); here the same rules drive chunked cudaMemcpyAsync of
// expert weights from host memory into a pool of GPU expert slots.
//
//  * queue   TransferQueue semantics: ordered by (priority desc, ExpertId
//            asc), resubmission overwrites, cancel / cancel_all; an on-demand
//            fetch is submitted at kMaxPriority = +inf (policy.hpp:26).
//  * link    one transfer in flight (engine.cpp:306-357), issued as chunks of
//            chunk_bytes (16 MB in MoE-Infinity), two chunks
//            in flight on a copy stream; a cancelled transfer stops at the
//            next chunk boundary (memsim.cpp:73-84).
//  * slots   empty / transferring / resident, prefetch protection, executing
//            (memsim.cpp:117-195).  A slot is acquired free first, else from
//            the eviction victim select_eviction_victim (policy.cpp:143-159,
//            the GPU kernel) priced by cache_priority of the request EAM
//            (engine.cpp:563); a speculative prefetch only displaces a victim
//            it outranks (engine.cpp:438-451); an on-demand fetch always wins
//            and, with every slot protected, displaces the least valuable
//            protected prefetch (engine.cpp:462-495); it also preempts a
//            speculative transfer in flight at a chunk boundary, which goes
//            back to the queue at its old priority (engine.cpp:507-529).
//  * events  execution clears protection and reprices the slot
//            (priority_reset_on_event, policy.cpp:161-167).
#include <cmath>
#include <deque>
#include <limits>
#include <map>
#include <set>
#include <unordered_map>

#include "abi_internal.hpp"

using moe::abi::fail;

namespace {

constexpr double kMaxPriority = std::numeric_limits<double>::infinity();  // policy.hpp:26
constexpr int kChunksInFlight = 2;

struct Cand {
  double pri;
  uint32_t id;  // flat ExpertId (layer * E + expert): orders like ExpertId (model.hpp:35-41)
};
struct CandOrder {  // TransferQueue::Order (policy.hpp:66-71)
  bool operator()(const Cand& a, const Cand& b) const {
    if (a.pri != b.pri) return a.pri > b.pri;
    return a.id < b.id;
  }
};

}  // namespace

struct moe_expert_cache {
  std::recursive_mutex mu;
  int device = 0;
  moe_shape shape{};
  uint64_t bytes = 0, chunk = 0;
  const uint8_t* host = nullptr;
  bool registered = false;
  uint8_t* pool = nullptr;
  cudaStream_t cst = nullptr;
  struct Slot {
    int64_t occ = -1;  // flat ExpertId
    int res = 0;       // 0 empty, 1 transferring, 2 resident
    bool prot = false, exec = false;
    double pri = 0.0;
  };
  std::vector<Slot> slots;
  std::unordered_map<uint32_t, uint32_t> index;  // flat id -> slot
  std::set<Cand, CandOrder> queue;
  std::map<uint32_t, double> by_id;
  struct Link {
    bool busy = false, cancel = false;
    uint32_t id = 0, slot = 0;
    double pri = 0.0;
    uint64_t issued = 0, done = 0;
    std::deque<std::pair<cudaEvent_t, uint64_t>> inflight;
  } link;
  std::vector<cudaEvent_t> free_ev;
  std::vector<uint64_t> req;  // the request's cross-phase EAM (engine.cpp:563)
  moe_expert_cache_stats st{};
  ~moe_expert_cache() {
    if (cst) cudaStreamSynchronize(cst);
    for (auto& e : link.inflight) cudaEventDestroy(e.first);
    for (cudaEvent_t e : free_ev) cudaEventDestroy(e);
    if (cst) cudaStreamDestroy(cst);
    if (pool) cudaFree(pool);
    if (registered) cudaHostUnregister(const_cast<uint8_t*>(host));
  }
};

namespace {

using moe::abi::DeviceGuard;

// ---- TransferQueue (policy.cpp:43-86) ---------------------------------------
void q_submit(moe_expert_cache* c, uint32_t id, double pri) {
  const auto it = c->by_id.find(id);
  if (it != c->by_id.end()) {
    c->queue.erase({it->second, id});
    it->second = pri;
  } else {
    c->by_id.emplace(id, pri);
  }
  c->queue.insert({pri, id});
}
bool q_cancel(moe_expert_cache* c, uint32_t id) {
  const auto it = c->by_id.find(id);
  if (it == c->by_id.end()) return false;
  c->queue.erase({it->second, id});
  c->by_id.erase(it);
  return true;
}

moe_status cache_pri(moe_expert_cache* c, uint32_t id, double* out) {  // policy.cpp:128-141
  const uint32_t E = c->shape.n_experts_per_layer;
  return moe_cache_priority(&c->shape, c->req.data(), id / E, id % E, out);
}

// ---- link: chunked DMA ------------------------------------------------------
moe_status issue_chunks(moe_expert_cache* c) {
  auto& k = c->link;
  while (!k.cancel && k.issued < c->bytes && (int)k.inflight.size() < kChunksInFlight) {
    const uint64_t n = std::min(c->chunk, c->bytes - k.issued);
    cudaEvent_t ev;
    if (!c->free_ev.empty()) {
      ev = c->free_ev.back();
      c->free_ev.pop_back();
    } else {
      CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    CK(cudaMemcpyAsync(c->pool + (uint64_t)k.slot * c->bytes + k.issued,
                       c->host + (uint64_t)k.id * c->bytes + k.issued, n, cudaMemcpyHostToDevice,
                       c->cst));
    CK(cudaEventRecord(ev, c->cst));
    k.inflight.push_back({ev, n});
    k.issued += n;
  }
  return MOE_OK;
}

// Completed chunks retire; a finished transfer makes its slot resident; a
// cancelled one frees its slot once its issued chunks have landed.
moe_status retire(moe_expert_cache* c, bool block) {
  auto& k = c->link;
  while (k.busy && !k.inflight.empty()) {
    cudaError_t q = block ? cudaEventSynchronize(k.inflight.front().first)
                          : cudaEventQuery(k.inflight.front().first);
    if (q == cudaErrorNotReady) break;
    CK(q);
    k.done += k.inflight.front().second;
    c->st.bytes_moved += k.inflight.front().second;
    c->free_ev.push_back(k.inflight.front().first);
    k.inflight.pop_front();
    block = false;
  }
  if (!k.busy) return MOE_OK;
  CKS(issue_chunks(c));  // keep kChunksInFlight chunks on the copy engine
  if (!k.inflight.empty()) return MOE_OK;
  auto& s = c->slots[k.slot];
  if (k.cancel) {  // GpuBuffer::cancel_transfer (memsim.cpp:166-175)
    c->index.erase(k.id);
    s = moe_expert_cache::Slot{};
    ++c->st.transfers_cancelled;
    k = moe_expert_cache::Link{};
  } else if (k.done == c->bytes) {  // GpuBuffer::complete_transfer
    s.res = 2;
    ++c->st.transfers_completed;
    k = moe_expert_cache::Link{};
  }
  return MOE_OK;
}

// Cancel the transfer in flight at the next chunk boundary (memsim.cpp:73-84):
// no further chunks; wait for the issued ones, then free its slot.
moe_status cancel_inflight(moe_expert_cache* c) {
  c->link.cancel = true;
  while (c->link.busy) CKS(retire(c, true));
  return MOE_OK;
}

moe_status evict(moe_expert_cache* c, uint32_t slot) {  // GpuBuffer::evict (memsim.cpp:177-189)
  auto& s = c->slots[slot];
  c->index.erase((uint32_t)s.occ);
  s = moe_expert_cache::Slot{};
  ++c->st.evictions;
  return MOE_OK;
}

// pick_victim (engine.cpp:368-385): resident slots, priced by the GPU kernel.
moe_status pick_victim(moe_expert_cache* c, int64_t* victim) {
  const uint32_t E = c->shape.n_experts_per_layer;
  std::vector<moe_slot_view> v;
  for (uint32_t i = 0; i < c->slots.size(); ++i) {
    const auto& s = c->slots[i];
    if (s.res != 2) continue;  // never evict mid-transfer
    moe_slot_view w{};
    w.slot = i;
    w.layer_idx = (uint32_t)s.occ / E;
    w.expert_idx = (uint32_t)s.occ % E;
    w.prefetch_protected = s.prot;
    w.pinned = s.exec;
    v.push_back(w);
  }
  *victim = -1;
  if (v.empty()) return MOE_OK;
  return moe_select_eviction_victim(&c->shape, c->req.data(), v.data(), v.size(), victim);
}

// force_slot_for_on_demand (engine.cpp:462-505, single GPU, no pending list)
moe_status force_slot(moe_expert_cache* c, int64_t* out) {
  int64_t chosen = -1;
  double chosen_p = 0.0;
  for (uint32_t i = 0; i < c->slots.size(); ++i) {
    const auto& s = c->slots[i];
    if (s.occ < 0 || s.exec || !s.prot) continue;
    double p = 0.0;
    CKS(cache_pri(c, (uint32_t)s.occ, &p));
    if (chosen < 0 || p < chosen_p) {
      chosen = i;
      chosen_p = p;
    }
  }
  if (chosen < 0) return fail(MOE_ERR_LOGIC, "on-demand fetch cannot obtain a buffer slot");
  if (c->slots[chosen].res == 1) {
    CKS(cancel_inflight(c));
  } else {
    c->slots[chosen].prot = false;  // priority_reset_on_event(displaced_from_topk)
    CKS(evict(c, (uint32_t)chosen));
  }
  *out = chosen;
  return MOE_OK;
}

// acquire_slot (engine.cpp:429-455)
moe_status acquire_slot(moe_expert_cache* c, const Cand& cd, int64_t* out) {
  *out = -1;
  for (uint32_t i = 0; i < c->slots.size(); ++i)
    if (c->slots[i].res == 0) {
      *out = i;
      return MOE_OK;
    }
  int64_t victim = -1;
  CKS(pick_victim(c, &victim));
  if (victim >= 0) {
    if (cd.pri != kMaxPriority) {  // contention: displace only what it outranks
      double vp = 0.0;
      CKS(cache_pri(c, (uint32_t)c->slots[victim].occ, &vp));
      if (vp >= cd.pri) return MOE_OK;
    }
    CKS(evict(c, (uint32_t)victim));
    *out = victim;
    return MOE_OK;
  }
  if (cd.pri != kMaxPriority) return MOE_OK;
  return force_slot(c, out);
}

// preempt_for_on_demand (engine.cpp:507-529)
moe_status preempt(moe_expert_cache* c, const Cand& cd, bool* did) {
  *did = false;
  if (cd.pri != kMaxPriority || !c->link.busy || c->link.pri == kMaxPriority) return MOE_OK;
  const uint32_t id = c->link.id;
  const double pri = c->link.pri;
  CKS(cancel_inflight(c));
  ++c->st.preemptions;
  if (!c->by_id.count(id)) q_submit(c, id, pri);
  *did = true;
  return MOE_OK;
}

// try_start_for_gpu (engine.cpp:306-357): at most one transfer started.
moe_status try_start(moe_expert_cache* c, bool* started) {
  *started = false;
restart:
  if (c->link.busy) {
    if (c->queue.empty() || c->queue.begin()->pri != kMaxPriority) return MOE_OK;
  }
  for (auto it = c->queue.begin(); it != c->queue.end(); ++it) {
    const Cand cd = *it;
    if (c->index.count(cd.id)) {  // already resident or in flight: satisfied
      q_cancel(c, cd.id);
      goto restart;
    }
    if (c->link.busy) {
      bool did = false;
      CKS(preempt(c, cd, &did));
      if (did) goto restart;
      continue;
    }
    int64_t slot = -1;
    CKS(acquire_slot(c, cd, &slot));
    if (slot < 0) {
      if (cd.pri == kMaxPriority) continue;
      break;  // lower-priority candidates cannot beat the same victims
    }
    auto& s = c->slots[slot];  // GpuBuffer::begin_transfer(slot, e, protect=true, kMax)
    s.occ = cd.id;
    s.res = 1;
    s.prot = true;
    s.pri = kMaxPriority;
    s.exec = false;
    c->index[cd.id] = (uint32_t)slot;
    c->link = moe_expert_cache::Link{};
    c->link.busy = true;
    c->link.id = cd.id;
    c->link.slot = (uint32_t)slot;
    c->link.pri = cd.pri;
    ++c->st.transfers_started;
    q_cancel(c, cd.id);
    CKS(issue_chunks(c));
    *started = true;
    return MOE_OK;
  }
  return MOE_OK;
}

moe_status pump(moe_expert_cache* c) {
  CKS(retire(c, false));
  for (;;) {
    bool started = false;
    CKS(try_start(c, &started));
    if (!started) break;
  }
  return MOE_OK;
}

moe_status check_id(const moe_expert_cache* c, uint32_t layer, uint32_t expert) {
  if (layer >= c->shape.n_layers || expert >= c->shape.n_experts_per_layer)
    return fail(MOE_ERR_OUT_OF_RANGE, "expert out of range");
  return MOE_OK;
}

}  // namespace

extern "C" {

moe_status moe_expert_cache_create(const moe_shape* shape, uint64_t expert_bytes, uint32_t n_slots,
                                   uint64_t chunk_bytes, const void* host_weights, int device,
                                   moe_expert_cache** out) {
  if (!out || !host_weights) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  CKS(moe::abi::check_shape(shape));
  if (expert_bytes == 0 || n_slots == 0 || chunk_bytes == 0)
    return fail(MOE_ERR_INVALID_ARGUMENT, "expert_bytes, n_slots and chunk_bytes must be > 0");
  int n_sm = 0;
  CKS(moe::abi::device_ok(device, &n_sm));
  DeviceGuard dg(device);
  auto* c = new moe_expert_cache();
  c->device = device;
  c->shape = *shape;
  c->bytes = expert_bytes;
  c->chunk = chunk_bytes;
  c->host = static_cast<const uint8_t*>(host_weights);
  c->slots.resize(n_slots);
  c->req.assign((uint64_t)shape->n_layers * shape->n_experts_per_layer, 0);
  const uint64_t total = (uint64_t)shape->n_layers * shape->n_experts_per_layer * expert_bytes;
  // page-lock the weight store unless the caller did (DMA at PCIe rate)
  cudaPointerAttributes pa{};
  if (cudaPointerGetAttributes(&pa, host_weights) != cudaSuccess || pa.type == cudaMemoryTypeUnregistered) {
    cudaGetLastError();
    if (cudaHostRegister(const_cast<void*>(host_weights), total, cudaHostRegisterReadOnly) ==
        cudaSuccess)
      c->registered = true;
    else
      cudaGetLastError();  // pageable fallback still moves the bytes (staged by the driver)
  }
  if (cudaMalloc(&c->pool, (uint64_t)n_slots * expert_bytes) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->cst, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return fail(MOE_ERR_OOM, "expert cache: device pool allocation failed");
  }
  *out = c;
  return MOE_OK;
}

moe_status moe_expert_cache_destroy(moe_expert_cache* c) {
  if (!c) return MOE_OK;
  DeviceGuard dg(c->device);
  delete c;
  return MOE_OK;
}

moe_status moe_expert_cache_set_request_eam(moe_expert_cache* c, const uint64_t* request_eam) {
  if (!c || !request_eam) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  std::copy(request_eam, request_eam + c->req.size(), c->req.begin());
  return MOE_OK;
}

moe_status moe_expert_cache_submit(moe_expert_cache* c, const moe_candidate* order, uint64_t n) {
  if (!c || (!order && n)) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  const uint32_t E = c->shape.n_experts_per_layer;
  for (uint64_t i = 0; i < n; ++i) CKS(check_id(c, order[i].layer_idx, order[i].expert_idx));
  // recompute_prefetch (engine.cpp:656-678): cancel_all, resubmit the order
  c->queue.clear();
  c->by_id.clear();
  for (uint64_t i = 0; i < n; ++i)
    q_submit(c, order[i].layer_idx * E + order[i].expert_idx, order[i].priority);
  return pump(c);
}

moe_status moe_expert_cache_progress(moe_expert_cache* c, int wait_idle) {
  if (!c) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  CKS(pump(c));
  while (wait_idle && c->link.busy) {
    CKS(retire(c, true));
    CKS(pump(c));
  }
  return MOE_OK;
}

moe_status moe_expert_cache_acquire(moe_expert_cache* c, uint32_t layer, uint32_t expert,
                                    void** device_ptr, int* was_resident) {
  if (!c || !device_ptr) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  CKS(check_id(c, layer, expert));
  const uint32_t id = layer * c->shape.n_experts_per_layer + expert;
  CKS(retire(c, false));
  auto it = c->index.find(id);
  const bool hit = it != c->index.end() && c->slots[it->second].res == 2;
  if (was_resident) *was_resident = hit;
  if (hit) {
    ++c->st.hits;
  } else {
    ++c->st.misses;
    q_submit(c, id, kMaxPriority);  // execute_layer (engine.cpp:689-697)
    for (;;) {
      CKS(pump(c));
      it = c->index.find(id);
      if (it != c->index.end() && c->slots[it->second].res == 2) break;
      if (!c->link.busy)
        return fail(MOE_ERR_LOGIC, "stalled waiting for expert %u/%u with no transfer pending",
                    layer, expert);
      CKS(retire(c, true));
    }
  }
  auto& s = c->slots[it->second];
  s.exec = true;
  *device_ptr = c->pool + (uint64_t)it->second * c->bytes;
  return MOE_OK;
}

moe_status moe_expert_cache_release(moe_expert_cache* c, uint32_t layer, uint32_t expert) {
  if (!c) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  CKS(check_id(c, layer, expert));
  const uint32_t id = layer * c->shape.n_experts_per_layer + expert;
  const auto it = c->index.find(id);
  if (it == c->index.end())
    return fail(MOE_ERR_LOGIC, "priority_reset_on_event: expert not in buffer");
  auto& s = c->slots[it->second];
  s.exec = false;
  s.prot = false;  // priority_reset_on_event(executed), policy.cpp:161-167
  CKS(cache_pri(c, id, &s.pri));
  return pump(c);
}

moe_status moe_expert_cache_slot(const moe_expert_cache* cc, uint32_t slot, int64_t* expert_flat,
                                 int* residency, int* prefetch_protected, double* priority) {
  auto* c = const_cast<moe_expert_cache*>(cc);
  if (!c) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  if (slot >= c->slots.size()) return fail(MOE_ERR_OUT_OF_RANGE, "slot out of range");
  const auto& s = c->slots[slot];
  if (expert_flat) *expert_flat = s.occ;
  if (residency) *residency = s.res;
  if (prefetch_protected) *prefetch_protected = s.prot;
  if (priority) *priority = s.pri;
  return MOE_OK;
}

moe_status moe_expert_cache_read_slot(const moe_expert_cache* cc, uint32_t slot, void* host_dst) {
  auto* c = const_cast<moe_expert_cache*>(cc);
  if (!c || !host_dst) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  if (slot >= c->slots.size()) return fail(MOE_ERR_OUT_OF_RANGE, "slot out of range");
  DeviceGuard dg(c->device);
  CK(cudaStreamSynchronize(c->cst));
  CK(cudaMemcpy(host_dst, c->pool + (uint64_t)slot * c->bytes, c->bytes, cudaMemcpyDeviceToHost));
  return MOE_OK;
}

moe_status moe_expert_cache_stats_get(const moe_expert_cache* cc, moe_expert_cache_stats* out) {
  auto* c = const_cast<moe_expert_cache*>(cc);
  if (!c || !out) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  std::lock_guard<std::recursive_mutex> lk(c->mu);
  *out = c->st;
  out->queued = c->queue.size();
  out->in_flight = c->link.busy ? 1 : 0;
  return MOE_OK;
}

}  // extern "C"

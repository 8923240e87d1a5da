// sharded.cu -- P-sharded EAMCs behind the C ABI.
//
// A sharded collection is a moe_eamc facade (h->sh set) over n shard handles,
// one per entry of device_ids (several shards may share a device).  Shard s
// owns the contiguous global slot range [base_s, base_s + cap_s); slots fill
// in order, as Eamc::insert appends at entries_.size() (eam.cpp:160-163), and
// every shard reports index = base_s + local slot with the entry's global seq,
// so results merge into exactly the unsharded answer:
//
//  match (eam.cpp:118-129)        probes to every shard's device, per-shard
//                                  matching (moe_eamc_match_device), one
//                                  all-gather of the {index, seq, distance}
//                                  rows (24 B per probe per shard, independent
//                                  of P), the lexicographic (distance, seq)
//                                  merge kernel on shard 0.
//  prefetch (policy.cpp:88-126)   per-shard exact distances + local minimum,
//                                  MIN all-reduce of the minimum's bits
//                                  (non-negative doubles order like their bit
//                                  patterns), per-shard u64 window aggregate,
//                                  SUM all-reduce, order phases on shard 0.
//                                  Min and integer sums are order-independent:
//                                  bit-identical to the unsharded call.
//  match_within (eam.cpp:131-150) per-shard exact distances, global minimum,
//                                  per-shard window lists, (distance, seq) sort.
//  insert (eam.cpp:152-178)       below capacity: append to the shard owning
//                                  slot `size`; at capacity: the sharded match
//                                  of the incoming EAM picks the victim (the
//                                  same lexicographic argmin), replaced in place
//                                  on its shard with seq = next_seq++.
//
// Collectives: with shards on distinct devices and NCCL present (libnccl.so.2,
// loaded at run time; the one torch already mapped when present), the
// all-gather and the two all-reduces are NCCL collectives over one
// communicator clique (ncclCommInitAll), and their failures are
// MOE_ERR_NCCL.  Shards sharing a device (e.g. a single-GPU box) or
// MOE_SHARD_NCCL=0 use stream-ordered device copies into shard 0 plus the
// same reductions as small kernels -- the same arithmetic, so the one-GPU
// tests exercise the full sharded logic.
#include <dlfcn.h>
#include <nccl.h>  // types and enums only: the library is resolved with dlopen

#include <atomic>
#include <limits>

#include "abi_internal.hpp"

namespace moe::abi {

namespace {

// ---- NCCL, resolved at run time -------------------------------------------
struct NcclApi {
  bool ok = false;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!so) so = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!so) return a;
    a.CommInitAll = reinterpret_cast<decltype(a.CommInitAll)>(dlsym(so, "ncclCommInitAll"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(so, "ncclCommDestroy"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(so, "ncclAllGather"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(so, "ncclAllReduce"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(so, "ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(so, "ncclGroupEnd"));
    a.GetErrorString =
        reinterpret_cast<decltype(a.GetErrorString)>(dlsym(so, "ncclGetErrorString"));
    a.ok = a.CommInitAll && a.CommDestroy && a.AllGather && a.AllReduce && a.GroupStart &&
           a.GroupEnd && a.GetErrorString;
    return a;
  }();
  return api;
}

#define CKN(expr)                                                                       \
  do {                                                                                  \
    ncclResult_t r_ = (expr);                                                           \
    if (r_ != ncclSuccess)                                                              \
      return fail(MOE_ERR_NCCL, "%s: %s (%s:%d)", #expr, nccl().GetErrorString(r_),     \
                  __FILE__, __LINE__);                                                  \
  } while (0)

// ---- small kernels of the copy path ----------------------------------------
__global__ void k_fill_none(moe_match* m, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    m[i] = moe_match{~0ull, ~0ull, __longlong_as_double(0x7ff0000000000000ll)};
}

__global__ void k_min_u64(const unsigned long long* parts, uint32_t n, unsigned long long* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long m = ~0ull;
    for (uint32_t i = 0; i < n; ++i) m = min(m, parts[i]);
    *out = m;
  }
}

__global__ void k_sum_u64(const unsigned long long* parts, uint32_t n, uint64_t cells,
                          unsigned long long* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cells;
       i += (uint64_t)gridDim.x * blockDim.x) {
    unsigned long long s = 0;
    for (uint32_t p = 0; p < n; ++p) s += parts[(uint64_t)p * cells + i];
    out[i] = s;
  }
}

}  // namespace

struct Shards {
  int n = 0;
  std::vector<moe_eamc*> s;
  std::vector<uint64_t> base, cap;
  std::vector<int> dev;
  uint64_t size = 0;
  bool use_nccl = false;
  std::vector<ncclComm_t> comm;
  // per shard (allocated on the shard's device)
  std::vector<DevBuf> probes, part, gath, dmin, agg;
  std::vector<cudaEvent_t> ev;
  // on shard 0's device
  DevBuf merged, cands, nout, dmin_all, agg_all;
  PinBuf hpack, hres;
  ~Shards() {
    for (size_t i = 0; i < comm.size(); ++i)
      if (comm[i]) nccl().CommDestroy(comm[i]);
    for (size_t i = 0; i < ev.size(); ++i) {
      DeviceGuard dg(dev[i]);
      if (ev[i]) cudaEventDestroy(ev[i]);
    }
    for (moe_eamc* h : s) moe_eamc_destroy(h);
  }
  int owner(uint64_t slot) const {  // shard owning a global slot
    int i = 0;
    while (i + 1 < n && slot >= base[i + 1]) ++i;
    return i;
  }
};

namespace {

uint64_t cells_of(const moe_eamc* h) {
  return (uint64_t)h->shape.n_layers * h->shape.n_experts_per_layer;
}

// Make every shard's event follow its stream's work, then shard 0's stream wait.
moe_status join_into_first(Shards& S) {
  for (int i = 1; i < S.n; ++i) {
    DeviceGuard dg(S.dev[i]);
    CK(cudaEventRecord(S.ev[i], S.s[i]->st));
    DeviceGuard d0(S.dev[0]);
    CK(cudaStreamWaitEvent(S.s[0]->st, S.ev[i], 0));
  }
  return MOE_OK;
}

// parts (n_parts x bytes, one per shard, on each shard's device) -> shard 0's
// `all` buffer [n][bytes]: NCCL all-gather, or stream-ordered device copies.
moe_status gather_to_first(Shards& S, std::vector<DevBuf>& parts, std::vector<DevBuf>& gath,
                           DevBuf& all, size_t bytes, void** all_p) {
  if (S.use_nccl) {
    for (int i = 0; i < S.n; ++i) {
      DeviceGuard dg(S.dev[i]);
      CK(gath[i].ensure(bytes * S.n));
    }
    CKN(nccl().GroupStart());
    for (int i = 0; i < S.n; ++i)
      CKN(nccl().AllGather(parts[i].p, gath[i].p, bytes, ncclUint8, S.comm[i], S.s[i]->st));
    CKN(nccl().GroupEnd());
    *all_p = gath[0].p;
    return MOE_OK;
  }
  {
    DeviceGuard dg(S.dev[0]);
    CK(all.ensure(bytes * S.n));
  }
  CKS(join_into_first(S));
  DeviceGuard d0(S.dev[0]);
  for (int i = 0; i < S.n; ++i)
    CK(cudaMemcpyPeerAsync(static_cast<uint8_t*>(all.p) + bytes * i, S.dev[0], parts[i].p,
                           S.dev[i], bytes, S.s[0]->st));
  *all_p = all.p;
  return MOE_OK;
}

// The global minimum of the shards' d_min bits, left in every S.dmin[i].
moe_status all_min(Shards& S) {
  if (S.use_nccl) {
    CKN(nccl().GroupStart());
    for (int i = 0; i < S.n; ++i)
      CKN(nccl().AllReduce(S.dmin[i].p, S.dmin[i].p, 1, ncclUint64, ncclMin, S.comm[i],
                           S.s[i]->st));
    CKN(nccl().GroupEnd());
    return MOE_OK;
  }
  void* all = nullptr;
  std::vector<DevBuf> none;
  CKS(gather_to_first(S, S.dmin, none, S.dmin_all, 8, &all));
  DeviceGuard d0(S.dev[0]);
  k_min_u64<<<1, 32, 0, S.s[0]->st>>>(static_cast<unsigned long long*>(all), (uint32_t)S.n,
                                      S.dmin[0].as<unsigned long long>());
  CK(cudaGetLastError());
  CK(cudaEventRecord(S.ev[0], S.s[0]->st));
  for (int i = 1; i < S.n; ++i) {
    DeviceGuard dg(S.dev[i]);
    CK(cudaStreamWaitEvent(S.s[i]->st, S.ev[0], 0));
    CK(cudaMemcpyPeerAsync(S.dmin[i].p, S.dev[i], S.dmin[0].p, S.dev[0], 8, S.s[i]->st));
  }
  return MOE_OK;
}

// Packed host probes of the smallest width holding them (1, 2, 4; 8 when a
// count needs it), every shard widened to match; returns the width.
moe_status pack_probes(moe_eamc* h, const uint64_t* probes, uint64_t n, int* wb) {
  Shards& S = *h->sh;
  const uint64_t cells = cells_of(h);
  CK(S.hpack.ensure(n * cells * 8));
  uint64_t o = moe::host::pack_counts(probes, n * cells, 1, S.hpack.p);
  int w = 1;
  if (o > 255ull) {
    w = o > 0xffffffffull ? 8 : o > 65535ull ? 4 : 2;
    if (w == 8)
      std::memcpy(S.hpack.p, probes, n * cells * 8);
    else
      moe::host::pack_counts(probes, n * cells, w, S.hpack.p);
  }
  for (int i = 0; i < S.n; ++i) CKS(ensure_width(S.s[i], std::min<uint64_t>(o, 0xffffffffull)));
  *wb = w;
  return MOE_OK;
}

}  // namespace

// ---- facade entry points ----------------------------------------------------

moe_status sh_create(const moe_shape* shape, moe_phase phase, uint64_t capacity, int count_bytes,
                     int n_shards, const int* device_ids, moe_eamc** out) {
  if (!out || !device_ids) return fail(MOE_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  CKS(check_shape(shape));
  if (n_shards < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "n_shards must be >= 1");
  if (capacity < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "Eamc: capacity must be >= 1");
  if ((uint64_t)n_shards > capacity)
    return fail(MOE_ERR_INVALID_ARGUMENT, "more shards than capacity");
  auto* S = new Shards();
  S->n = n_shards;
  uint64_t b = 0;
  for (int i = 0; i < n_shards; ++i) {
    const uint64_t c = capacity / n_shards + ((uint64_t)i < capacity % n_shards);
    moe_eamc* sh = nullptr;
    moe_status st = moe_eamc_create(shape, phase, c, count_bytes, device_ids[i], &sh);
    if (st != MOE_OK) {
      delete S;
      return st;
    }
    moe_eamc_set_index_base(sh, b);
    S->s.push_back(sh);
    S->base.push_back(b);
    S->cap.push_back(c);
    S->dev.push_back(device_ids[i]);
    b += c;
  }
  S->ev.assign(n_shards, nullptr);
  S->probes.resize(n_shards);
  S->part.resize(n_shards);
  S->gath.resize(n_shards);
  S->dmin.resize(n_shards);
  S->agg.resize(n_shards);
  for (int i = 0; i < n_shards; ++i) {
    DeviceGuard dg(S->dev[i]);
    if (cudaEventCreateWithFlags(&S->ev[i], cudaEventDisableTiming) != cudaSuccess) {
      delete S;
      return fail(MOE_ERR_CUDA, "event create failed");
    }
  }
  // NCCL clique when every shard has its own device
  bool distinct = n_shards > 1;
  for (int i = 0; i < n_shards && distinct; ++i)
    for (int j = 0; j < i; ++j)
      if (S->dev[i] == S->dev[j]) distinct = false;
  const char* env = getenv("MOE_SHARD_NCCL");
  if (distinct && !(env && env[0] == '0') && nccl().ok) {
    S->comm.assign(n_shards, nullptr);
    const ncclResult_t r = nccl().CommInitAll(S->comm.data(), n_shards, S->dev.data());
    if (r != ncclSuccess) {
      const char* msg = nccl().GetErrorString(r);
      S->comm.assign(n_shards, nullptr);
      delete S;
      return fail(MOE_ERR_NCCL, "ncclCommInitAll: %s", msg);
    }
    S->use_nccl = true;
  }
  auto* h = new moe_eamc();
  h->device = device_ids[0];
  h->shape = *shape;
  h->phase = phase;
  h->capacity = capacity;
  h->c.L = shape->n_layers;
  h->c.E = shape->n_experts_per_layer;
  h->c.cb = count_bytes ? count_bytes : 1;
  h->sh = S;
  *out = h;
  return MOE_OK;
}

moe_status sh_destroy(moe_eamc* h) {
  delete h->sh;
  h->sh = nullptr;
  delete h;
  return MOE_OK;
}

moe_status sh_layout(const moe_eamc* h, int* n_shards, int* use_nccl) {
  if (n_shards) *n_shards = h->sh->n;
  if (use_nccl) *use_nccl = h->sh->use_nccl;
  return MOE_OK;
}

moe_status sh_info(const moe_eamc* h, uint64_t* size, int* count_bytes) {
  const Shards& S = *h->sh;
  if (size) *size = S.size;
  if (count_bytes) {
    int cb = 1;
    for (moe_eamc* s : S.s) cb = std::max(cb, s->c.cb);
    *count_bytes = cb;
  }
  return MOE_OK;
}

moe_status sh_entry(moe_eamc* h, uint64_t index, uint64_t* counts, uint64_t* seq) {
  Shards& S = *h->sh;
  if (index >= S.size) return fail(MOE_ERR_OUT_OF_RANGE, "entry index out of range");
  const int i = S.owner(index);
  return moe_eamc_entry(S.s[i], index - S.base[i], counts, seq);
}

moe_status sh_append(moe_eamc* h, const void* counts, int count_bytes, const uint64_t* seqs,
                     uint64_t n) {
  Shards& S = *h->sh;
  if (S.size + n > h->capacity)
    return fail(MOE_ERR_SNAPSHOT, "snapshot holds more entries than its capacity");
  const uint64_t cells = cells_of(h);
  uint64_t off = 0;
  while (off < n) {
    const int i = S.owner(S.size);
    const uint64_t room = S.base[i] + S.cap[i] - S.size;
    const uint64_t m = std::min(room, n - off);
    CKS(moe_eamc_append_packed(S.s[i], static_cast<const uint8_t*>(counts) +
                                           off * cells * count_bytes,
                               count_bytes, seqs + off, m));
    S.size += m;
    off += m;
    for (uint64_t k = 0; k < m; ++k) h->next_seq = std::max(h->next_seq, seqs[off - m + k] + 1);
  }
  return MOE_OK;
}

moe_status sh_match(moe_eamc* h, const uint64_t* probes, uint64_t n, moe_match* out) {
  Shards& S = *h->sh;
  if (n == 0) return MOE_OK;
  if (S.size == 0) {
    for (uint64_t q = 0; q < n; ++q)
      out[q] = moe_match{~0ull, ~0ull, std::numeric_limits<double>::infinity()};
    return MOE_OK;
  }
  int wb = 1;
  CKS(pack_probes(h, probes, n, &wb));
  const uint64_t cells = cells_of(h);
  const size_t pbytes = n * cells * wb, rbytes = n * sizeof(moe_match);
  // the batch once per device, then every shard's matcher on its stream
  for (int i = 0; i < S.n; ++i) {
    DeviceGuard dg(S.dev[i]);
    int first = i;
    for (int j = 0; j < i; ++j)
      if (S.dev[j] == S.dev[i]) {
        first = j;
        break;
      }
    if (first == i) {
      CK(S.probes[i].ensure(pbytes + 16));
      CK(cudaMemcpyAsync(S.probes[i].p, S.hpack.p, pbytes, cudaMemcpyHostToDevice, S.s[i]->st));
    } else {  // same device as an earlier shard: wait for that shard's upload
      CK(cudaEventRecord(S.ev[first], S.s[first]->st));
      CK(cudaStreamWaitEvent(S.s[i]->st, S.ev[first], 0));
    }
    CK(S.part[i].ensure(rbytes));
    if (S.s[i]->c.size == 0) {
      k_fill_none<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 1024), 256, 0, S.s[i]->st>>>(
          S.part[i].as<moe_match>(), n);
      CK(cudaGetLastError());
    } else {
      CKS(moe_eamc_match_device(S.s[i], S.probes[first].p, wb, n, S.part[i].as<moe_match>(),
                                S.s[i]->st));
    }
  }
  void* all = nullptr;
  CKS(gather_to_first(S, S.part, S.gath, S.merged, rbytes, &all));
  DeviceGuard d0(S.dev[0]);
  CK(S.cands.ensure(rbytes));
  CKS(moe_match_merge_device(static_cast<moe_match*>(all), S.n, n, S.cands.as<moe_match>(),
                             S.s[0]->st));
  CK(S.hres.ensure(rbytes));
  CK(cudaMemcpyAsync(S.hres.p, S.cands.p, rbytes, cudaMemcpyDeviceToHost, S.s[0]->st));
  CK(cudaStreamSynchronize(S.s[0]->st));
  std::memcpy(out, S.hres.p, rbytes);
  for (uint64_t q = 0; q < n; ++q)
    if (out[q].index == MOE_MATCH_WIDTH_SENTINEL)
      return fail(MOE_ERR_OVERFLOW,
                  "probe %llu: a row's sum of squared counts reaches 2^53, beyond the range "
                  "where the reference's fp64 arithmetic (eam.cpp:75-87) is exact",
                  (unsigned long long)q);
  return MOE_OK;
}

moe_status sh_insert(moe_eamc* h, const uint64_t* counts, int64_t* evicted_slot,
                     uint64_t* evicted_counts) {
  Shards& S = *h->sh;
  if (S.size < h->capacity) {  // append at slot `size` (eam.cpp:160-163)
    const int i = S.owner(S.size);
    const uint64_t seq = h->next_seq;
    CKS(moe_eamc_append(S.s[i], counts, &seq, 1));
    ++S.size;
    h->next_seq = seq + 1;
    if (evicted_slot) *evicted_slot = -1;
    return MOE_OK;
  }
  // at capacity: the lexicographic (distance, seq) argmin over all shards
  moe_match v;
  CKS(sh_match(h, counts, 1, &v));
  const int i = S.owner(v.index);
  if (evicted_counts) CKS(moe_eamc_entry(S.s[i], v.index - S.base[i], evicted_counts, nullptr));
  CKS(replace_slot(S.s[i], counts, v.index - S.base[i], h->next_seq));
  ++h->next_seq;
  if (evicted_slot) *evicted_slot = (int64_t)v.index;
  return MOE_OK;
}

moe_status sh_build(moe_eamc* h, const uint64_t* counts, uint64_t n, int64_t* evicted_slots) {
  // construction does not shard (the victim chain is sequential):
  // n ordered inserts, each victim found by the sharded matcher
  const uint64_t cells = cells_of(h);
  for (uint64_t k = 0; k < n; ++k) {
    int64_t slot = -1;
    CKS(sh_insert(h, counts + k * cells, &slot, nullptr));
    if (evicted_slots) evicted_slots[k] = slot;
  }
  return MOE_OK;
}

moe_status sh_prefetch(moe_eamc* h, const uint64_t* cur_eam, uint32_t cur, int filter,
                       moe_candidate* out, uint64_t cap, uint64_t* n_out) {
  Shards& S = *h->sh;
  *n_out = 0;
  if (S.size == 0) return MOE_OK;  // policy.cpp:91-93
  const uint64_t cells = cells_of(h);
  for (int i = 0; i < S.n; ++i) {  // local exact distances and minimum
    DeviceGuard dg(S.dev[i]);
    CK(S.dmin[i].ensure(8));
    CK(S.agg[i].ensure(cells * 8));
    CKS(moe_eamc_window_min_device(S.s[i], cur_eam, S.dmin[i].as<uint64_t>(), S.s[i]->st));
  }
  CKS(all_min(S));
  for (int i = 0; i < S.n; ++i) {  // local window aggregates (kMatchWindow, policy.hpp:30)
    DeviceGuard dg(S.dev[i]);
    CKS(moe_eamc_window_aggregate_device(S.s[i], cur, 0.01, S.dmin[i].as<uint64_t>(),
                                         S.agg[i].as<uint64_t>(), S.s[i]->st));
  }
  unsigned long long* agg = nullptr;
  if (S.use_nccl) {
    CKN(nccl().GroupStart());
    for (int i = 0; i < S.n; ++i)
      CKN(nccl().AllReduce(S.agg[i].p, S.agg[i].p, cells, ncclUint64, ncclSum, S.comm[i],
                           S.s[i]->st));
    CKN(nccl().GroupEnd());
    agg = S.agg[0].as<unsigned long long>();
  } else {
    void* all = nullptr;
    std::vector<DevBuf> none;
    CKS(gather_to_first(S, S.agg, none, S.agg_all, cells * 8, &all));
    DeviceGuard d0(S.dev[0]);
    k_sum_u64<<<(unsigned)std::min<uint64_t>((cells + 255) / 256, 1024), 256, 0, S.s[0]->st>>>(
        static_cast<unsigned long long*>(all), (uint32_t)S.n, cells,
        S.agg[0].as<unsigned long long>());
    CK(cudaGetLastError());
    agg = S.agg[0].as<unsigned long long>();
  }
  DeviceGuard d0(S.dev[0]);
  CK(S.cands.ensure(std::max<uint64_t>(cells, 1) * sizeof(moe_candidate)));
  CK(S.nout.ensure(8));
  CKS(moe_eamc_prefetch_order_device(S.s[0], reinterpret_cast<const uint64_t*>(agg), cur, filter,
                                     S.cands.as<moe_candidate>(), S.nout.as<uint32_t>(),
                                     S.s[0]->st));
  CK(S.hres.ensure(8 + cells * sizeof(moe_candidate)));
  CK(cudaMemcpyAsync(S.hres.p, S.nout.p, 4, cudaMemcpyDeviceToHost, S.s[0]->st));
  CK(cudaStreamSynchronize(S.s[0]->st));
  const uint32_t n = *S.hres.as<uint32_t>();
  *n_out = n;
  const uint64_t m = std::min<uint64_t>(n, cap);
  if (m && out)
    CK(cudaMemcpy(out, S.cands.p, m * sizeof(moe_candidate), cudaMemcpyDeviceToHost));
  return MOE_OK;
}

moe_status sh_match_within(moe_eamc* h, const uint64_t* probe, double window, moe_match* out,
                           uint64_t cap, uint64_t* n_out) {
  Shards& S = *h->sh;
  *n_out = 0;
  if (S.size == 0) return MOE_OK;
  for (int i = 0; i < S.n; ++i) {
    DeviceGuard dg(S.dev[i]);
    CK(S.dmin[i].ensure(8));
    CKS(moe_eamc_window_min_device(S.s[i], probe, S.dmin[i].as<uint64_t>(), S.s[i]->st));
  }
  CKS(all_min(S));
  uint64_t bits = 0;
  {
    DeviceGuard d0(S.dev[0]);
    CK(cudaMemcpyAsync(&bits, S.dmin[0].p, 8, cudaMemcpyDeviceToHost, S.s[0]->st));
    CK(cudaStreamSynchronize(S.s[0]->st));
  }
  std::vector<moe::WinEntry> all, v;
  for (int i = 0; i < S.n; ++i) {
    CKS(window_list(S.s[i], bits, window, &v));
    all.insert(all.end(), v.begin(), v.end());
  }
  // (distance, seq) order of the result list (eam.cpp:145-148)
  std::sort(all.begin(), all.end(), [](const moe::WinEntry& a, const moe::WinEntry& b) {
    return a.d != b.d ? a.d < b.d : a.seq < b.seq;
  });
  for (uint64_t k = 0; k < all.size() && k < cap; ++k)
    out[k] = moe_match{all[k].p, all[k].seq, all[k].d};
  *n_out = all.size();
  return MOE_OK;
}

moe_status sh_clone(const moe_eamc* h, moe_eamc** out) {
  const Shards& S = *h->sh;
  moe_eamc* c = nullptr;
  int cb = 1;
  sh_info(h, nullptr, &cb);
  CKS(sh_create(&h->shape, (moe_phase)h->phase, h->capacity, cb, S.n, S.dev.data(), &c));
  const uint64_t cells = cells_of(h);
  std::vector<uint64_t> counts, seqs;
  for (int i = 0; i < S.n; ++i) {  // slot order preserved shard by shard
    const uint64_t m = S.s[i]->c.size;
    counts.resize(m * cells);
    seqs.resize(m);
    for (uint64_t k = 0; k < m; ++k) {
      moe_status st = moe_eamc_entry(S.s[i], k, counts.data() + k * cells, &seqs[k]);
      if (st != MOE_OK) {
        sh_destroy(c);
        return st;
      }
    }
    moe_status st = sh_append(c, counts.data(), 8, seqs.data(), m);
    if (st != MOE_OK) {
      sh_destroy(c);
      return st;
    }
  }
  c->next_seq = h->next_seq;
  *out = c;
  return MOE_OK;
}

moe_status sh_save(const moe_eamc* h, const char* path, bool binary) {
  // the snapshot of the equivalent single collection: entries in global slot
  // order with their seqs and next_seq (JSON v1, eam.cpp:184-205)
  const Shards& S = *h->sh;
  int cb = 1;
  sh_info(h, nullptr, &cb);
  moe_eamc* one = nullptr;
  CKS(moe_eamc_create(&h->shape, (moe_phase)h->phase, h->capacity, cb, S.dev[0], &one));
  const uint64_t cells = cells_of(h);
  std::vector<uint64_t> counts, seqs;
  moe_status st = MOE_OK;
  for (int i = 0; i < S.n && st == MOE_OK; ++i) {
    const uint64_t m = S.s[i]->c.size;
    counts.resize(m * cells);
    seqs.resize(m);
    for (uint64_t k = 0; k < m && st == MOE_OK; ++k)
      st = moe_eamc_entry(S.s[i], k, counts.data() + k * cells, &seqs[k]);
    if (st == MOE_OK && m) st = moe_eamc_append(one, counts.data(), seqs.data(), m);
  }
  if (st == MOE_OK) {
    one->next_seq = h->next_seq;
    st = binary ? moe_eamc_save_binary(one, path) : moe_eamc_save(one, path);
  }
  moe_eamc_destroy(one);
  return st;
}

}  // namespace moe::abi

/*
 * moe_eamc.h -- C ABI of the B200-native EAM/EAMC decision path
 * (MoE-Infinity, arXiv 2401.14361).  libmoe_eamc.so implements every entry
 * point below with hand-written sm_100a CUDA kernels; there is no CPU
 * fallback: a missing or unusable GPU is reported as MOE_ERR_CUDA.
 *
 * The reference boundary is the C++ library API of moesim::core
 * (/root/reference/proj/core/include/moesim/{eam,policy}.hpp).  Each entry
 * point cites the reference symbol it replaces.  Reference C++ exceptions
 * map to status codes; the C++ wrapper include/moesim_b200/eamc.hpp maps
 * them back so the reference's callers compile unchanged.
 *
 * Conventions
 *  - Count matrices are row-major L x E uint64 (eam.hpp:55), exactly the
 *    reference Eam storage.  Batches are [n][L][E].
 *  - Functions without a `_device` suffix take HOST pointers and are
 *    synchronous.  `_device` variants take device pointers and a
 *    cudaStream_t (passed as void*) and are stream-ordered.
 *  - Threading: one handle per writer.  match/match_within/prefetch are
 *    const readers (eam.hpp:89-94) and may be called from
 *    several host threads on one handle: the host entry points of a handle
 *    serialise on its lock (they share its scratch and staging memory).
 *    `_device` calls on one handle must be ordered on one stream (they share
 *    device scratch); insert needs exclusivity.
 *  - Errors: the status code, plus a thread-local message from
 *    moe_last_error().
 */
#ifndef MOE_EAMC_H_
#define MOE_EAMC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MOE_EAMC_ABI_VERSION 1

typedef enum moe_status {
  MOE_OK = 0,
  MOE_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument (eam.cpp:55-58,:109,:114,:153-158) */
  MOE_ERR_OUT_OF_RANGE = 2,     /* std::out_of_range (eam.cpp:43-46,:66; policy.cpp:91,:130) */
  MOE_ERR_SNAPSHOT = 3,         /* EamcSnapshotError (eam.hpp:63-65) */
  MOE_ERR_LOGIC = 4,            /* std::logic_error (policy.cpp:164) */
  MOE_ERR_CUDA = 5,             /* no usable sm_100 device / kernel failure */
  MOE_ERR_NCCL = 6,
  MOE_ERR_OOM = 7,
  MOE_ERR_OVERFLOW = 8, /* a count outside the range where the reference's fp64
                          arithmetic is exact (row sum of squares >= 2^53) */
  MOE_ERR_TRACE = 9     /* TraceIngestError (workload.hpp:55-59): a bad trace line;
                           moe_last_error() holds the reference's "line N: ..." text */
} moe_status;

/* ModelShape (model.hpp:19-29) */
typedef struct moe_shape {
  uint32_t n_layers;
  uint32_t n_experts_per_layer;
  uint32_t top_k;
} moe_shape;

typedef enum moe_phase { MOE_PHASE_PREFILL = 0, MOE_PHASE_DECODE = 1 } moe_phase; /* eam.hpp:17 */
typedef enum moe_eam_kind { MOE_KIND_ITERATION = 0, MOE_KIND_REQUEST = 1 } moe_eam_kind; /* eam.hpp:16 */

/* EamcMatch (eam.hpp:67-71).  A "none" result (empty collection / shard) is
 * index = seq = UINT64_MAX, distance = +inf. */
typedef struct moe_match {
  uint64_t index;
  uint64_t seq;
  double distance;
} moe_match;

/* PrefetchCandidate (policy.hpp:46-50) */
typedef struct moe_candidate {
  uint32_t layer_idx;
  uint32_t expert_idx;
  double priority;
} moe_candidate;

/* SlotView (policy.hpp:96-101) */
typedef struct moe_slot_view {
  uint64_t slot;
  uint32_t layer_idx;
  uint32_t expert_idx;
  uint8_t prefetch_protected;
  uint8_t pinned;
  uint8_t pad_[6];
} moe_slot_view;

typedef struct moe_eamc moe_eamc; /* opaque device-resident Eamc */

int moe_abi_version(void);
/* Host threads of the marshalling pool used by the host-pointer entry points
 * (u64 -> storage-width narrowing; MOE_HOST_THREADS overrides). */
int moe_host_threads(void);
const char* moe_last_error(void);
/* Device properties the library keys its launch geometry on. */
moe_status moe_device_info(int device, int* sm_count, int* cc_major, int* cc_minor,
                           size_t* l2_bytes);
/* Creates the device's CUDA context (the cost of the first call otherwise). */
moe_status moe_device_warmup(int device);

/* ---- collection lifecycle: Eamc(ModelShape, Phase, capacity) eam.cpp:106-111 ---- */
/* count_bytes: storage width of one count on the device, 1, 2 or 4 (0 = 1).
 * The collection widens itself (1 -> 2 -> 4 bytes) when an inserted EAM or
 * a probe needs it.  Any u64 count the reference answers EXACTLY is
 * accepted: its fp64 sums (eam.cpp:75-87) are exact integers while every
 * row's sum of squared counts is below 2^53, and the device computes those
 * sums exactly in integers.  A row at or past that bound (so also any count
 * >= 2^27) is MOE_ERR_OVERFLOW: there the reference rounds, and this library
 * refuses rather than answer differently. */
moe_status moe_eamc_create(const moe_shape* shape, moe_phase phase, uint64_t capacity,
                           int count_bytes, int device, moe_eamc** out);
moe_status moe_eamc_destroy(moe_eamc* h);
/* shape()/phase()/capacity()/size()/next_seq (eam.hpp:80-87) */
moe_status moe_eamc_info(const moe_eamc* h, moe_shape* shape, int* phase, uint64_t* capacity,
                         uint64_t* size, uint64_t* next_seq, int* count_bytes);
/* Deep copy (Eamc's implicit copy constructor, eam.hpp:76-116): same slots,
 * seqs, next_seq, capacity and device. */
moe_status moe_eamc_clone(const moe_eamc* h, moe_eamc** out);
/* entry(i) / entry_seq(i) (eam.hpp:86-87); counts may be NULL. */
moe_status moe_eamc_entry(const moe_eamc* h, uint64_t index, uint64_t* counts, uint64_t* seq);

/* ---- construction: Eamc::insert (eam.cpp:152-178) ---- */
/* *evicted_slot = slot replaced (-1 when appended); evicted_counts (nullable)
 * receives the evicted Eam. */
moe_status moe_eamc_insert(moe_eamc* h, const uint64_t* counts, moe_eam_kind kind,
                           moe_phase phase, int64_t* evicted_slot, uint64_t* evicted_counts);
/* Batched construction (K7): n request-level EAMs inserted in order with the
 * exact semantics of n sequential Eamc::insert calls (as driven by
 * moesim_main.cpp:212-216).  evicted_slots[n] (nullable). */
moe_status moe_eamc_build(moe_eamc* h, const uint64_t* counts, uint64_t n,
                          int64_t* evicted_slots);
/* Clustering construction (north-star item 3; OPT-IN and PARITY-UNPINNED:
 * the reference defers clustering).  Picks
 * capacity representatives from the n request EAMs: iteration 0 is exactly
 * moe_eamc_build (n ordered Eamc::insert calls); each further iteration
 * assigns every EAM to its nearest representative (the exact matcher),
 * proposes per cluster the member closest to the u64 sum of the cluster's
 * counts, and replaces the representative when the cluster's total exact
 * distance to the proposal is strictly lower -- so representatives stay
 * real request EAMs and the objective sum_i min_p d(eam_i, rep_p) never
 * increases.  Stops after `iterations` or when nothing changes.  The
 * collection must start empty.  objective[iterations+1] (nullable): the
 * objective after each iteration (index 0 = the reference construction);
 * rep_index[capacity] (nullable): the input index of every slot's EAM, which
 * is also its seq; *iterations_run (nullable): refinement iterations done. */
moe_status moe_eamc_build_clustered(moe_eamc* h, const uint64_t* counts, uint64_t n,
                                    uint32_t iterations, double* objective, uint64_t* rep_index,
                                    uint32_t* iterations_run);
/* Bulk append with caller-given seqs (Eamc::load semantics, eam.cpp:229-244);
 * used for snapshots and for P-sharded collections where the global
 * insertion number of every entry is assigned by the caller.  Entries are
 * u64 [n][L][E]; next_seq becomes max(next_seq, max(seqs)+1). */
moe_status moe_eamc_append(moe_eamc* h, const uint64_t* counts, const uint64_t* seqs, uint64_t n);
/* Same, with counts already narrow on the host ([n][L][E] of count_bytes:
 * 1, 2, 4 or 8). */
moe_status moe_eamc_append_packed(moe_eamc* h, const void* counts, int count_bytes,
                                  const uint64_t* seqs, uint64_t n);

/* ---- matching: Eamc::match (eam.cpp:118-129) over a probe batch ---- */
/* probes [n][L][E] u64 host; out[n]; found[n] (nullable). */
moe_status moe_eamc_match(const moe_eamc* h, const uint64_t* probes, uint64_t n_probes,
                          moe_match* out, uint8_t* found);
/* Same, with host probes already narrow: [n][L][E] of probe_bytes (1, 2, 4
 * or 8) bytes per count (e.g. counts traced as u8/u16/u32).  Results are identical
 * to moe_eamc_match on the widened counts; one H2D of the narrow batch. */
moe_status moe_eamc_match_packed(const moe_eamc* h, const void* probes, int probe_bytes,
                                 uint64_t n_probes, moe_match* out, uint8_t* found);
/* Device variant: probes are device [n][L][E] of probe_bytes (1, 2, 4 or 8)
 * bytes per count, out is device moe_match[n].  stream NULL = the handle's
 * internal stream (NOT the legacy default stream); pass the caller's stream
 * to order the work with the caller's kernels and events.  Nothing waits on
 * the host, so the collection is never widened here: a probe with a count
 * above the collection's current storage width gets the WIDTH SENTINEL
 * {index = MOE_MATCH_WIDTH_SENTINEL, seq = UINT64_MAX, distance = NaN}; redo
 * such probes with moe_eamc_match / moe_eamc_match_packed (which widen). */
#define MOE_MATCH_WIDTH_SENTINEL 0xFFFFFFFFFFFFFFFEull
moe_status moe_eamc_match_device(const moe_eamc* h, const void* probes, int probe_bytes,
                                 uint64_t n_probes, moe_match* out, void* stream);
/* Eamc::match_within (eam.cpp:131-150): every entry within `window` of the
 * best distance, sorted by (distance, seq).  *n_out = total number; at most
 * cap are written. */
moe_status moe_eamc_match_within(const moe_eamc* h, const uint64_t* probe, double window,
                                 moe_match* out, uint64_t cap, uint64_t* n_out);
/* Lexicographic (distance, seq) merge of per-shard results (P-sharded
 * matching): parts is [n_parts][n] -> out[n].  A width
 * sentinel in any part makes the merged result the sentinel (never hidden
 * behind another shard's answer). */
moe_status moe_match_merge(const moe_match* parts, uint64_t n_parts, uint64_t n, moe_match* out);
moe_status moe_match_merge_device(const moe_match* parts, uint64_t n_parts, uint64_t n,
                                  moe_match* out, void* stream);

/* P-sharded collections: results report index = base + local slot, so the
 * per-shard outputs merge into global slot numbers. */
moe_status moe_eamc_set_index_base(moe_eamc* h, uint64_t base);

/* A P-sharded Eamc(ModelShape, Phase, capacity) (eam.cpp:106-111; SURVEY.md
 * 8e) behind the same handle type: n_shards shards, shard s on device
 * device_ids[s] (ids may repeat: shards sharing one GPU), owning the
 * contiguous global slot range of its share of the capacity.  Every entry
 * point of this header that takes host pointers (insert, build, append,
 * match, match_packed, match_within, prefetch_priorities, decide, entry,
 * info, clone, save, destroy, build_from_traces) works on it with exactly the
 * unsharded semantics and results: matching = per-shard matcher + all-gather
 * of the per-shard {index, seq, distance} (24 B per probe per shard) + the
 * lexicographic (distance, seq) merge; prefetch = per-shard exact distances,
 * MIN all-reduce, per-shard u64 window aggregates, SUM all-reduce, order on
 * shard 0; insert at capacity = the sharded match of the incoming EAM picks
 * the victim.  With every shard on its own device the collectives are NCCL
 * (libnccl.so.2, loaded at run time; failures are MOE_ERR_NCCL); shards that
 * share a device (or MOE_SHARD_NCCL=0) use stream-ordered device copies and
 * reduction kernels.  The `_device` entry points and set_index_base apply to
 * single-device handles only (MOE_ERR_INVALID_ARGUMENT here). */
moe_status moe_eamc_create_sharded(const moe_shape* shape, moe_phase phase, uint64_t capacity,
                                   int count_bytes, int n_shards, const int* device_ids,
                                   moe_eamc** out);
/* Eamc::load (eam.cpp:207-256) into a sharded collection (same snapshot
 * semantics as moe_eamc_load; a snapshot whose capacity is below n_shards
 * loads as a single-device collection on device_ids[0]). */
moe_status moe_eamc_load_sharded(const char* path, const moe_shape* expected, int n_shards,
                                 const int* device_ids, moe_eamc** out);
/* n_shards (1 for a single-device handle) and whether NCCL carries its collectives. */
moe_status moe_eamc_shard_layout(const moe_eamc* h, int* n_shards, int* uses_nccl);

/* Persistent decision server (0 = off, the default: one kernel launch per
 * decision).  With n_ctas > 0 (capped at half the SMs), prefetch_priorities
 * on this handle is served by a decision kernel resident on n_ctas SMs and
 * fed through a pinned-memory mailbox: no launch and no stream
 * synchronisation per call.  It exits after 50 ms without requests and is
 * relaunched on the next one.  While enabled, other decision launches in the
 * process size their grids to the remaining SMs. */
moe_status moe_eamc_set_decision_server(moe_eamc* h, int n_ctas);

/* Instrumentation: when enabled, matching records CUDA events around its
 * kernels on the launching stream; ms[0..2] = accumulated device time of
 * probe packing, the screen pass and the refine pass, calls[0..2] their
 * launch counts (reset by moe_eamc_set_profiling). */
moe_status moe_eamc_set_profiling(moe_eamc* h, int enable);
moe_status moe_eamc_kernel_times(const moe_eamc* h, double* ms, uint64_t* calls);

/* eam_distance (eam.cpp:91-104), evaluated on the device. */
moe_status moe_eam_distance(const moe_shape* shape, const uint64_t* a, const uint64_t* b,
                            double* out);

/* ---- policy (policy.cpp) ---- */
/* prefetch_priorities (policy.cpp:88-126) and, if apply_floor_filter, the
 * engine's floor filter (engine.cpp:663-668).  Candidates in the reference
 * order (priority desc, ExpertId asc); *n_out total, at most cap written. */
moe_status moe_prefetch_priorities(const moe_eamc* h, const uint64_t* cur_eam,
                                   uint32_t current_layer, int apply_floor_filter,
                                   moe_candidate* out, uint64_t cap, uint64_t* n_out);
/* Fused decision (K5+K6): the prefetch order above and the eviction victim
 * over `slots` priced from request_eam, in one launch. */
moe_status moe_decide(const moe_eamc* h, const uint64_t* cur_eam, uint32_t current_layer,
                      const uint64_t* request_eam, const moe_slot_view* slots, uint64_t n_slots,
                      moe_candidate* out, uint64_t cap, uint64_t* n_out, int64_t* victim);
/* P-sharded prefetch_priorities (policy.cpp:88-126 split at its two
 * reductions).  Per rank, on the rank's shard:
 *   1. moe_eamc_window_min_device: exact distances of cur_eam to every entry
 *      (kept in the handle) and *d_min_bits = bits of the shard's minimum
 *      distance (+inf for an empty shard) -- the d_min of eam.cpp:132-141.
 *      Synchronises once (count-width check).
 *   2. MIN all-reduce of d_min_bits across ranks (non-negative doubles order
 *      like their bit patterns).
 *   3. moe_eamc_window_aggregate_device: agg [L][E] u64 (overwritten) = sum of
 *      the rows > current_layer of the shard's entries with
 *      d <= d_min + window (eam.cpp:143; policy.cpp:96-104 uses window 0.01,
 *      policy.hpp:30).  Must follow step 1 on the same handle.
 *   4. SUM all-reduce of agg.
 *   5. moe_eamc_prefetch_order_device: priorities, floor filter
 *      (engine.cpp:663-668) and order from the summed agg; out needs
 *      (L-current_layer-1)*E slots, *n_out (device) = count.
 * All pointers except cur_eam are device pointers; work runs on `stream`
 * (NULL: the handle's stream). */
moe_status moe_eamc_window_min_device(const moe_eamc* h, const uint64_t* cur_eam,
                                      uint64_t* d_min_bits, void* stream);
moe_status moe_eamc_window_aggregate_device(const moe_eamc* h, uint32_t current_layer,
                                            double window, const uint64_t* d_min_bits,
                                            uint64_t* agg, void* stream);
moe_status moe_eamc_prefetch_order_device(const moe_eamc* h, const uint64_t* agg,
                                          uint32_t current_layer, int apply_floor_filter,
                                          moe_candidate* out, uint32_t* n_out, void* stream);
/* cache_priority (policy.cpp:128-141) */
moe_status moe_cache_priority(const moe_shape* shape, const uint64_t* request_eam,
                              uint32_t layer, uint32_t expert, double* out);
/* select_eviction_victim (policy.cpp:143-159); *victim = slot or -1. */
moe_status moe_select_eviction_victim(const moe_shape* shape, const uint64_t* request_eam,
                                      const moe_slot_view* slots, uint64_t n_slots,
                                      int64_t* victim);

/* ---- expert weights: the host consumer of the prefetch order ----
 * A pool of n_slots GPU expert slots filled from host expert weights
 * ([L][E][expert_bytes], page-locked here unless already) by chunked
 * cudaMemcpyAsync, driven by the engine's rules for the reference's simulated
 * transfers: TransferQueue (policy.cpp:43-86), one transfer in flight cut at
 * chunk boundaries (memsim.cpp:73-84), slot acquisition -- free slot, else the
 * select_eviction_victim victim priced by cache_priority of the request EAM,
 * displaced by a speculative prefetch only when it outranks it -- and
 * on-demand fetches at +inf priority that preempt speculative transfers and
 * displace the least valuable protected prefetch when nothing else is free
 * (engine.cpp:306-357, :429-529), execution resets protection
 * (policy.cpp:161-167). */
typedef struct moe_expert_cache moe_expert_cache;
typedef struct moe_expert_cache_stats {
  uint64_t transfers_started, transfers_completed, transfers_cancelled, preemptions, evictions;
  uint64_t hits, misses, bytes_moved, queued, in_flight;
} moe_expert_cache_stats;
moe_status moe_expert_cache_create(const moe_shape* shape, uint64_t expert_bytes, uint32_t n_slots,
                                   uint64_t chunk_bytes, const void* host_weights, int device,
                                   moe_expert_cache** out);
moe_status moe_expert_cache_destroy(moe_expert_cache* c);
/* The request's cross-phase EAM [L][E] that prices cache_priority (engine.cpp:563). */
moe_status moe_expert_cache_set_request_eam(moe_expert_cache* c, const uint64_t* request_eam);
/* recompute_prefetch (engine.cpp:656-678): cancel_all, submit the order (e.g. the
 * output of moe_prefetch_priorities with the floor filter), start transfers. */
moe_status moe_expert_cache_submit(moe_expert_cache* c, const moe_candidate* order, uint64_t n);
/* Retire finished chunks/transfers and start the next ones; wait_idle: until
 * nothing is in flight and nothing startable remains. */
moe_status moe_expert_cache_progress(moe_expert_cache* c, int wait_idle);
/* execute_layer's fetch (engine.cpp:681-712): the expert's device weights,
 * on demand when not resident (blocks until resident); marks it executing. */
moe_status moe_expert_cache_acquire(moe_expert_cache* c, uint32_t layer, uint32_t expert,
                                    void** device_ptr, int* was_resident);
/* Execution done: not executing, protection cleared, repriced (policy.cpp:161-167). */
moe_status moe_expert_cache_release(moe_expert_cache* c, uint32_t layer, uint32_t expert);
/* Slot state: occupant (flat layer*E+expert, -1 empty), residency (0 empty,
 * 1 transferring, 2 resident), protection, cache priority. */
moe_status moe_expert_cache_slot(const moe_expert_cache* c, uint32_t slot, int64_t* expert_flat,
                                 int* residency, int* prefetch_protected, double* priority);
moe_status moe_expert_cache_stats_get(const moe_expert_cache* c, moe_expert_cache_stats* out);
/* The bytes a slot holds (D2H; for verification). */
moe_status moe_expert_cache_read_slot(const moe_expert_cache* c, uint32_t slot, void* host_dst);

/* ---- tracing: Eam::record (eam.cpp:41-52) from router top-k ids ---- */
/* topk_idx [n_tokens][L][top_k] with idx_bytes in {1,2,4}; request r owns
 * tokens [offsets[r], offsets[r+1]).  counts [R][L][E] u64 are ACCUMULATED
 * (Eam::record adds).  All-or-nothing: any index >= E returns
 * MOE_ERR_OUT_OF_RANGE with counts untouched (eam.cpp:42-47). */
moe_status moe_eam_trace(const moe_shape* shape, const void* topk_idx, int idx_bytes,
                         uint64_t n_tokens, const uint64_t* offsets, uint64_t n_requests,
                         uint64_t* counts);
/* Device variant: all pointers device, stream-ordered on `stream`; counts_u32
 * [R][L][E] accumulated.  *bad_index_flag must be 0 on entry; an index >= E
 * leaves it 1 and counts_u32 as it was (the call's additions are rolled back
 * on the device).  Calls on different streams share no scratch memory.
 * Request offsets must lie within [0, n_tokens].  u8 ids are read in aligned
 * 16-byte granules, so up to 15 bytes past either end of the id buffer (in
 * the granules holding its first and last byte, never another page) may be
 * read; they are never counted. */
moe_status moe_eam_trace_device(const moe_shape* shape, const void* topk_idx, int idx_bytes,
                                uint64_t n_tokens, const uint64_t* offsets, uint64_t n_requests,
                                uint32_t* counts_u32, int* bad_index_flag, void* stream);

/* ---- trace ingest: ingest_traces (workload.cpp:209-232) + validate_trace
 * (model.cpp:32-71) + request_level_eam (moesim_main.cpp:192-201) ---- */
/* Request-level EAMs of one phase from a JSONL trace file (model.hpp:103-114):
 * prefill = iteration 0, decode = iterations 1.. (requests with < 2
 * iterations skipped, moesim_main.cpp:212-214).  Writes up to cap EAMs
 * [n][L][E] u64 (counts may be NULL with cap 0); *n_eams = total. */
moe_status moe_traces_request_eams(const char* path, const moe_shape* shape, moe_phase phase,
                                   uint64_t* counts, uint64_t cap, uint64_t* n_eams);
/* `moesim eamc save` (moesim_main.cpp:203-221) minus the file write: the
 * request EAMs of the collection's phase inserted in file order (K7). */
moe_status moe_eamc_build_from_traces(moe_eamc* h, const char* path, uint64_t* n_inserted);

/* eamc_capacity_bound (eam.cpp:258-268) */
moe_status moe_eamc_capacity_bound(const moe_shape* shape, double similarity, uint64_t* out);

/* ---- snapshots: Eamc::save / Eamc::load (eam.cpp:184-256), JSON v1 ---- */
moe_status moe_eamc_save(const moe_eamc* h, const char* path);
/* Binary fast path (same contents: slot order, seqs, next_seq): a 64-byte
 * header, seq[size] u64 and the counts at the storage width, written from one
 * D2H copy (layout in abi.cu).  moe_eamc_load reads either format (by its
 * magic "MOEEAMCB"). */
moe_status moe_eamc_save_binary(const moe_eamc* h, const char* path);
/* expected may be NULL (load(path)) or the configured shape (load(path, shape)). */
moe_status moe_eamc_load(const char* path, const moe_shape* expected, int device,
                         moe_eamc** out);

/* ---- synthetic input families (host, bit-identical to the reference) ---- */
/* bench_match's random_request_eam stream (bench.cpp:44-54,60-66): skips
 * `skip` EAMs of Rng::stream(seed, 0x6265636E), then writes n EAMs as
 * count_bytes-wide counts (1, 2 or 8) into out [n][L][E]. */
moe_status moe_gen_bench_family(uint64_t seed, uint32_t L, uint32_t E, uint64_t skip, uint64_t n,
                                int count_bytes, void* out);

#ifdef __cplusplus
}
#endif
#endif /* MOE_EAMC_H_ */

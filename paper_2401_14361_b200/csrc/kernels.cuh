// kernels.cuh -- host-visible launch interface of the sm_100a kernels.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "../../include/moe_eamc.h"

namespace moe {

// Device-resident collection (AoS counts [cap][L][RB], SoA metadata).
struct DevColl {
  uint32_t L = 0, E = 0, RB = 0, C = 0;
  int cb = 1;              // bytes per stored count (1, 2 or 4)
  uint64_t cap = 0;
  uint32_t size = 0;
  uint64_t index_base = 0;    // reported index = index_base + slot (P-sharding)
  uint8_t* counts = nullptr;  // [cap][L][RB]
  float* ibT = nullptr;       // [L][cap] fp32 1/sqrt(sum c^2) (0 on zero rows)
  double* sqb = nullptr;      // [cap][L] sqrt(sum c^2)
  uint64_t* seq = nullptr;    // [cap]
  // tensor-core screen operands (L <= 64): rows normalised to unit length,
  // fp16, K-major [cap][Kp] with Kp = roundup(L*E, 64); zero-row bitmasks
  uint32_t Kp = 0;
  __half* nrm = nullptr;
  uint64_t* zmask = nullptr;
};

// Packed probe batch.
struct DevProbes {
  uint32_t Q = 0;
  uint8_t* packed = nullptr;  // [Q][L][RB]
  float* ia = nullptr;        // [Q][L]
  double* sqa = nullptr;      // [Q][L]
  __half* nrm = nullptr;      // [Q][Kp] (tensor-core screen operand) or null
  uint64_t* zmask = nullptr;  // [Q]
  uint8_t* wide = nullptr;    // [Q] 1 = a count exceeds the collection's storage width
};

struct MatchGeom {
  uint32_t G = 1, S = 2, QT = 1, n_groups = 1, n_pt = 0, grid = 1, blocks_per_sm = 1;
  size_t smem = 0;
};

struct MatchWork {  // scratch for one match pipeline
  uint32_t* T = nullptr;       // [Q]
  uint32_t* bcnt = nullptr;    // [Q]
  uint2* bucket = nullptr;     // [Q][bcap]
  uint32_t bcap = 0;
  uint32_t* over_list = nullptr;  // [Q]
  uint32_t* over_n = nullptr;     // [1]
  moe_match* partials = nullptr;  // [chunk][grid]
  uint32_t part_chunk = 0;
  float eps2 = 0.f;               // screen band the refine pass must honour
};

struct WinEntry {
  uint64_t p;
  uint64_t seq;
  double d;
};

float screen_eps2(uint32_t L);

// Geometry for a matcher launch (mode 0 screen with QT probes / tile, or
// QT=1 exact modes).  Returns false if the shape does not fit shared memory.
bool plan_match(const DevColl& c, int n_sm, int mode, uint32_t QT, MatchGeom* g);

cudaError_t encode_tmap(const DevColl& c, uint32_t G, CUtensorMap* map);

// Matcher state that the probe-prep kernel initialises for the screen pass
// that follows it (instead of separate memset launches): T[q] = +huge,
// bcnt[q] = 0, *over_n = 0.  Null members are left alone.
struct MatchInit {
  uint32_t* T = nullptr;
  uint32_t* bcnt = nullptr;
  uint32_t* over_n = nullptr;
  unsigned long long* dmin = nullptr;  // single-probe exact pass: running minimum <- ~0
};

// u64/u16/u8 counts -> packed rows + norms.  rows = n*L.  When ibT != null
// the row norms are written as collection metadata at slots base..base+n.
// *max_count (if given) is reset and receives the largest count that does not
// fit the storage width.
cudaError_t launch_prep(const void* src, int src_bytes, uint64_t n, uint32_t L, uint32_t E,
                        uint32_t RB, int cb, uint8_t* dst, float* ia, double* sq, float* ibT,
                        uint64_t ib_cap, uint64_t ib_base, unsigned long long* max_count,
                        __half* nrm, uint32_t Kp, uint64_t* zmask, uint8_t* wide,
                        cudaStream_t st, MatchInit init = MatchInit{});

// Tensor-core (tcgen05 kind::f16) screen pass for large probe batches.
float tc_eps2(uint32_t L, uint32_t E, uint32_t Kp);
bool tc_supported(const DevColl& c);
// dmat != null: matrix mode, every screen distance -> dmat[q * ldd + p]
// (no threshold / buckets; ldd a multiple of 4).
cudaError_t launch_tc_screen(const DevColl& c, const DevProbes& pr, const MatchWork& w, int n_sm,
                             cudaStream_t st, float* dmat = nullptr, uint32_t ldd = 0);
// Blocked construction replay of staged entries [first, first+nb): screen
// matrices dc [nb][c.size] and dx [nb][nb] -> victims vic[nb] (slot +
// index_base, evicted seq, exact distance), collection updated; occ[c.size]
// must be all -1 (it is again on return).
size_t replay_block_smem(const DevColl& c);  // must be <= 220 KB for the blocked replay
cudaError_t launch_replay_block(const DevColl& c, const DevProbes& staged, uint32_t first,
                                uint32_t nb, const float* dc, uint32_t ldc, const float* dx,
                                uint32_t ldx, float eps2, int* occ, uint64_t seq0,
                                moe_match* vic, cudaStream_t st,
                                unsigned long long* prof = nullptr);
// Exact-integer tensor-core (tcgen05 kind::i8) screen for small probe batches
// (u8 collections, L <= 32); blockdiag is scratch of i8_blockdiag_bytes().
bool i8_supported(const DevColl& c);
size_t i8_blockdiag_bytes(const DevColl& c, uint32_t Q);
cudaError_t launch_tci8_screen(const DevColl& c, const DevProbes& pr, const MatchWork& w,
                               uint8_t* blockdiag, int n_sm, cudaStream_t st);

// mode 0: screen all Q probes; then refine.
cudaError_t launch_screen(const CUtensorMap& map, const DevColl& c, const DevProbes& pr,
                          const MatchGeom& g, const MatchWork& w, cudaStream_t st);
cudaError_t launch_refine(const DevColl& c, const DevProbes& pr, const MatchWork& w,
                          moe_match* out, const int* halt, int* halt_set, uint32_t halt_value,
                          cudaStream_t st);
// mode 1: exact argmin for the probes listed in qlist[0..*qlist_n) (at most
// chunk of them starting at qlist_off); T may be null (evaluate all).
cudaError_t launch_exact(const CUtensorMap& map, const DevColl& c, const DevProbes& pr,
                         const MatchGeom& g, const MatchWork& w, const uint32_t* qlist,
                         uint32_t qlist_n, const uint32_t* T, moe_match* out, cudaStream_t st,
                         const uint32_t* nq_dev = nullptr);
// Exact argmin for listed probes without the TMA pipeline (any shape); parts
// is scratch of chunk * exact_warp_blocks(n_sm) moe_match.
uint32_t exact_warp_blocks(int n_sm);
cudaError_t launch_exact_warp(const DevColl& c, const DevProbes& pr, const uint32_t* qlist,
                              uint32_t qlist_n, moe_match* out, moe_match* parts,
                              uint32_t chunk, int n_sm, cudaStream_t st,
                              const uint32_t* nq_dev = nullptr);
cudaError_t launch_window_list(const DevColl& c, const double* dist,
                               const unsigned long long* dmin, double window, WinEntry* wl,
                               uint32_t* wl_n, cudaStream_t st);

// Single-probe exact distances, row-parallel: r[p][l] for l in [l0, l1), then
// the in-order layer sum of all L rows -> dist[p] and atomic min -> *dmin.
cudaError_t launch_exact_rows(const DevColl& c, const DevProbes& pr, uint32_t q0, uint32_t l0,
                              uint32_t l1, double* r, double* dist, unsigned long long* dmin,
                              int n_sm, cudaStream_t st);
// Window members (dist <= d_min + window) -> mem list; agg[L][E] += their
// rows > cur (u64).
cudaError_t launch_member_agg(const DevColl& c, const double* dist,
                              const unsigned long long* dmin, double window, uint32_t cur,
                              uint32_t* mem, uint32_t* n_mem, unsigned long long* agg, int n_sm,
                              cudaStream_t st, bool n_mem_zeroed = false);
// ---- fused single-probe decision (decide.cu, K4 + K5 [+ K6]) -------------
constexpr uint32_t kDecMaxNz = 1024;        // explicit probe rows per call (else the old path)
constexpr uint32_t kDecInlineBytes = 512;   // explicit rows passed inside the launch parameters
constexpr uint32_t kDecInlineNz = 32;
constexpr uint32_t kDecBarriers = 5;        // grid barriers per decision launch
constexpr uint32_t kDecListWords = 4096;    // member row words of a 256-entry batch above which members are listed
constexpr uint32_t kDecStagedMin = 2048;    // survivors above which every CTA stages the whole list (C2)
constexpr size_t kDecStageCap = 92 * 1024;  // its shared memory bound (two CTAs per SM)
constexpr uint32_t kDecMaxLayers = 2048;    // layers above the current one (order phases)
constexpr uint32_t kDecMaxExperts = 8192;   // experts per layer (a layer's segment in shared memory)

struct DecisionArgs {
  // phases: do_dist = distances + minimum (else dist[] and *dmin_ext are
  // given); do_agg = window aggregation (else agg[] is given); the order is
  // always computed
  int do_dist, do_agg;
  const unsigned long long* dmin_ext;
  // collection
  const uint8_t* counts;
  const double* sqb;
  const uint64_t* zm;  // zero-row bitmasks (L <= 64) or null
  uint32_t size, L, E, RB;
  // the probe's explicit rows (its nonzero rows in [j0, hi], ascending), at
  // the storage width, RB bytes each: inline below or at `rows`/`nz`
  uint32_t n_nz, j0, hi, keep;
  int rows_inline;
  const uint8_t* rows;
  const uint16_t* nz;
  double* pref;  // [size] in-order layer sum through row `keep` (reused when j0 > 0)
  double* dist;  // [size]
  // window + aggregation
  uint32_t cur;
  double window;
  unsigned long long* dmin2;  // [2] by call parity, ~0 before first use
  unsigned long long* agg;    // [L*E]
  uint32_t* mcount;           // listed window members (0 between calls; null: never list)
  uint32_t* mlist;            // [size] listed window members (wide windows)
  // order
  int filter;
  unsigned long long* ckey;  // [(L-cur-1)*E] per-layer sorted survivor keys (~bits(priority))
  uint32_t* cid;             // [(L-cur-1)*E] their flat ExpertIds
  uint32_t* crank;           // [(L-cur-1)*E] their output positions
  uint32_t* nseg;            // [L-cur-1] survivors per layer
  uint32_t parity;
  moe_candidate* out;  // [(L-cur-1)*E] (host-mapped or device)
  uint32_t* n_out;
  // eviction (optional)
  const unsigned long long* req;  // request EAM [L*E]
  const moe_slot_view* slots;
  uint32_t n_slots;
  double* slot_pri;  // [n_slots] scratch
  long long* victim;
  unsigned long long* tprobe;  // optional [8] phase timestamps of CTA 0 (MOE_DEC_TIMING)
  uint32_t* bar;      // grid-barrier arrival counter (never reset)
  uint32_t bar_base;  // arrivals before this launch (kDecBarriers * grid per launch)
  alignas(16) uint8_t inline_rows[kDecInlineBytes];
  uint16_t inline_nz[kDecInlineNz];
};
size_t decision_smem(uint32_t L, uint32_t E, uint32_t RB, uint32_t n_nz, uint32_t cur,
                     uint32_t grid);
int decision_grid(int n_sm, uint32_t size, uint32_t L, uint32_t cur);
// One cooperative launch (grid <= co-resident CTAs; decision_grid picks it).
cudaError_t launch_decision(const DecisionArgs& a, int cb, int grid, size_t smem,
                            cudaStream_t st);
// Small collections: the whole decision in one CTA (decide.cu).
size_t decision_small_smem(uint32_t size, uint32_t L, uint32_t E, uint32_t RB, uint32_t n_nz,
                           uint32_t cur);
cudaError_t launch_decision_small(const DecisionArgs& a, int cb, size_t smem, cudaStream_t st);
// Shared memory of the small-path kernel for any request it takes (size <= kSmallMaxP,
// rows above x E <= kSmallMaxCells, all L probe rows explicit).
size_t decision_small_smem_max(uint32_t L, uint32_t RB);
constexpr uint32_t kSmallMaxP = 512;        // entries (one per thread)
constexpr uint32_t kSmallMaxCells = 1024;   // (L - cur - 1) * E candidates
// The persistent decision server's mailbox (pinned host memory, device-mapped).
struct DecServerCtl {
  uint64_t seq_req;   // host: the request number being posted
  uint64_t seq_done;  // device: the last request completed
  int stop;           // host: ask the server to exit
  int pad_;
  DecisionArgs args;  // the request (host-side pointers for rows/nz when not inline)
};
// One-CTA persistent server for small collections (moe_eamc_set_decision_server).
cudaError_t launch_decision_small_server(DecServerCtl* ctl, uint64_t seq0, uint64_t idle_ns, int cb,
                                        size_t smem, cudaStream_t st);
cudaError_t launch_decision_server(DecServerCtl* ctl, DecisionArgs* dargs, uint8_t* drows,
                                   uint32_t* go, uint32_t* done, uint32_t* bar, uint64_t seq0,
                                   uint32_t k0, uint64_t idle_ns, uint32_t gen, int cb, int grid,
                                   size_t smem, cudaStream_t st);

cudaError_t launch_merge(const moe_match* parts, uint64_t n_parts, uint64_t n, moe_match* out,
                         cudaStream_t st);
cudaError_t launch_pair_distance(const uint8_t* a, const double* sqa, const uint8_t* b,
                                 const double* sqb, uint32_t L, uint32_t C, uint32_t RB, int cb,
                                 double* out, cudaStream_t st);

// Build replay step: copy staged probe i into the slot chosen by out->index
// (or append slot), seq = seq_value.  Skips when *halt != 0.
cudaError_t launch_replace(const DevColl& c, const DevProbes& staged, uint32_t i,
                           const moe_match* victim, uint64_t seq_value, const int* halt,
                           cudaStream_t st);
// Bulk copy staged probes [first, first+n) into slots [base, base+n).
cudaError_t launch_append_staged(const DevColl& c, const DevProbes& staged, uint32_t first,
                                 uint32_t n, uint64_t base, cudaStream_t st);

// Eviction scoring (K6): cache priorities and the victim over slot views; the
// prefetch half of this kernel is superseded by the fused decision kernel
// (launch_decision); it serves cache_priority / select_eviction_victim.
cudaError_t launch_decide(const unsigned long long* agg, uint32_t L, uint32_t E, uint32_t cur,
                          int filter, int do_prefetch, const unsigned long long* req,
                          const moe_slot_view* slots, uint64_t n_slots, moe_candidate* out,
                          uint32_t* n_out, long long* victim, double* slot_pri,
                          cudaStream_t st);

// K1 tracing (trace.cu): counts[R][L][E] (count_bytes 4 = u32, 8 = u64) +=
// the per-request histograms of the ids; an out-of-range id sets *bad and
// the call's additions are rolled back on the device (all-or-nothing).
cudaError_t launch_trace(const void* topk, int idx_bytes, uint64_t T, uint32_t L, uint32_t E,
                         uint32_t k, const uint64_t* offsets, uint64_t R, void* counts,
                         int count_bytes, int* bad, int n_sm, cudaStream_t st);

// Clustering construction (cluster.cu): one refinement step's device work --
// centroids of the assignment m, per-cluster proposals cidx (trace index),
// fixed-point totals of the current and proposed representatives' distances.
cudaError_t launch_cluster_step(const uint8_t* packed, const double* sq, uint64_t n, uint32_t L,
                                uint32_t E, uint32_t RB, int cb, const moe_match* m,
                                uint64_t base, uint64_t P, unsigned long long* cent, double* dc,
                                unsigned long long* cmin, unsigned long long* cidx,
                                unsigned long long* tot_cur, unsigned long long* tot_cand,
                                cudaStream_t st);

cudaError_t launch_widen(const uint8_t* src, uint8_t* dst, uint64_t rows, uint32_t RB_old,
                         uint32_t RB_new, int cb_old, int cb_new, cudaStream_t st);

}  // namespace moe
